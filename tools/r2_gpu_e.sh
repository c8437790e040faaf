mkdir -p gpurun_out
./tools/probes/sincos_probe > gpurun_out/r2e_sincos.txt 2>&1; cat gpurun_out/r2e_sincos.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lga_ls -s 2 -c 1 -o gpurun_out/r2e_ls_multi -f python bench.py --steps 1 --warmup 1 --no-cpu --no-extra > gpurun_out/r2e_ncu.log 2>&1
tail -3 gpurun_out/r2e_ncu.log
