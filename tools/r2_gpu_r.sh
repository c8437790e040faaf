mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dock.py tests/test_gpu_headline_parity.py -x -q -p no:cacheprovider > gpurun_out/r2r_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2r_tests.txt
tail -3 gpurun_out/r2r_tests.txt
AB_OUT=r2r_ab.json timeout 900 python tools/ls_ab.py "MDR_LS_WARPS=2" "MDR_LS_WARPS=0"
