set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2a_pytest.txt
timeout 600 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
lscpu | head -20 > gpurun_out/r2a_lscpu.txt
cat gpurun_out/r2a_pytest.txt gpurun_out/r2a_bench.json
