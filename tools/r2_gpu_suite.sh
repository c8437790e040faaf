# Round-2 GPU check: full -m gpu suite, default bench, reference arm, lscpu.  Output under gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt
lscpu > gpurun_out/r2_lscpu.txt
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_pytest.txt
timeout 600 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err
tail -5 gpurun_out/r2_pytest.txt; cat gpurun_out/r2_bench.json gpurun_out/r2_bench_ref.json
