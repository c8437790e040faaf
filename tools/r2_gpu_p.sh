mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_units.py tests/test_gpu_headline_parity.py -q -p no:cacheprovider -k "c2 or c4_analytic or tcgen05" > gpurun_out/r2p_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2p_tests.txt
tail -4 gpurun_out/r2p_tests.txt
timeout 1200 python -m paper_2410_10447_b200.microbench --cpu > gpurun_out/r2p_microbench.json 2> gpurun_out/r2p_microbench.err
tail -3 gpurun_out/r2p_microbench.err; head -c 400 gpurun_out/r2p_microbench.json
