# Round-2 GPU evidence in one call (run on the box: gpurun -- 'TAG=r2 bash tools/r2_full.sh'):
# the -m gpu suite, the default bench line and the reference arm, the launch list, one ncu
# --set full capture of the dominant kernel (+ its DRAM traffic), and the per-phase cycle split
# of the search (a -DMDR_PHASE_PROF=1 build, variants/prof, built beforehand:
#   python -m paper_2410_10447_b200.build --variant prof -DMDR_PHASE_PROF=1).
mkdir -p gpurun_out
TAG=${TAG:-r2}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.txt
tail -3 gpurun_out/${TAG}_pytest.txt
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-extra > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:lga_ls_multi -s 2 -c 1 -o gpurun_out/${TAG}_ls_kernel -f python bench.py --steps 1 --warmup 1 --no-cpu --no-extra > gpurun_out/${TAG}_ncu.log 2>&1
python tools/ncu_traffic.py gpurun_out/${TAG}_ls_kernel.ncu-rep > gpurun_out/${TAG}_ls_kernel_traffic.json 2>&1
if [ -f paper_2410_10447_b200/variants/prof/libmdr_b200.so ]; then
  MDR_LIB_PATH=paper_2410_10447_b200/variants/prof/libmdr_b200.so PHASE_OUT=${TAG}_phase_profile.json timeout 300 python tools/phase_profile.py > /dev/null 2>&1
fi
head -c 1500 gpurun_out/${TAG}_bench.json; echo; head -c 600 gpurun_out/${TAG}_bench_ref.json
