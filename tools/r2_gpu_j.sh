mkdir -p gpurun_out
PARITY_MODES=fp64fast PARITY_OUT=r2j_parity_default.json timeout 900 python tools/parity_scale.py > gpurun_out/r2j_parity_default.txt 2>&1
MDR_LIB_PATH=paper_2410_10447_b200/variants/rcp1/libmdr_b200.so PARITY_MODES=fp64fast PARITY_OUT=r2j_parity_rcp1.json timeout 900 python tools/parity_scale.py > gpurun_out/r2j_parity_rcp1.txt 2>&1
grep -h "fp64fast" gpurun_out/r2j_parity_default.txt gpurun_out/r2j_parity_rcp1.txt | cut -c1-200
AB_OUT=r2j_ab.json timeout 900 python tools/ls_ab.py "MDR_LS_WARPS=2" "MDR_LIB_PATH=paper_2410_10447_b200/variants/rcp1/libmdr_b200.so"
