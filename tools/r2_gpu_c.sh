mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dock.py -x -q -p no:cacheprovider -k "multi_warp or sqrt or warp_pair or chunked" > gpurun_out/r2c_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2c_tests.txt
tail -5 gpurun_out/r2c_tests.txt
AB_OUT=r2c_ab.json timeout 900 python tools/ls_ab.py "MDR_LS_WARPS=1" "MDR_LS_WARPS=0" "MDR_LS_WARPS=2" "MDR_LS_WARPS=3" "MDR_LS_WARPS=3 MDR_LS_CHUNK_LEN=16" "MDR_LS_WARPS=4" "MDR_LS_WARPS=4 MDR_LS_CHUNK_LEN=16" "MDR_LS_WARPS=2 MDR_LS_CHUNK_LEN=16"
