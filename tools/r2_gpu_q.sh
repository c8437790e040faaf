mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_headline_parity.py -q -p no:cacheprovider -k "c4_analytic" -s > gpurun_out/r2q_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/r2q_tests.txt
grep -h "c4 analytic\|passed\|failed" gpurun_out/r2q_tests.txt | tail -3
# ncu stall tables of the C2 kernels: K1c (5), paper f16 MMA (2), K2s (4), K2t (7), every B, chain and stream launches
for B in 64 128 256; do
  timeout 600 ncu --set full --clock-control none -k regex:"chain_kernel|stream_kernel|reduce_tc05" -c 8 -o gpurun_out/r2q_c2_b${B} -f \
    bash -c "for k in 5 2 4 7; do python -m paper_2410_10447_b200.microbench --kernel \$k --blocks $B --n 1000000; done" > gpurun_out/r2q_ncu_b${B}.log 2>&1
done
ls -la gpurun_out/r2q_c2_b*.ncu-rep
