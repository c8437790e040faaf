mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dock.py tests/test_gpu_headline_parity.py -x -q -p no:cacheprovider > gpurun_out/r2l_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2l_tests.txt
tail -3 gpurun_out/r2l_tests.txt
MDR_LIB_PATH=paper_2410_10447_b200/variants/prof/libmdr_b200.so PHASE_OUT=r2l_phase.json timeout 300 python tools/phase_profile.py > gpurun_out/r2l_phase.txt 2>&1; cat gpurun_out/r2l_phase.txt
AB_OUT=r2l_ab.json timeout 900 python tools/ls_ab.py "MDR_LS_WARPS=0" "MDR_LS_SLOTS=6" "MDR_LS_SLOTS=7" "MDR_LS_SLOTS=5" "MDR_LS_SLOTS=4"
