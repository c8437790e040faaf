# tcgen05 reduce routing tests + phase profile of the warp-pair LS kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_units.py -x -q -p no:cacheprovider > gpurun_out/r2b_units.txt 2>&1; echo "rc=$?" >> gpurun_out/r2b_units.txt
MDR_LIB_PATH=paper_2410_10447_b200/variants/prof/libmdr_b200.so PHASE_OUT=r2b_phase.json timeout 300 python tools/phase_profile.py > gpurun_out/r2b_phase.txt 2>&1
tail -5 gpurun_out/r2b_units.txt; cat gpurun_out/r2b_phase.txt
