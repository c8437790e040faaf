mkdir -p gpurun_out
PARITY_OUT=r2n_report_default.json timeout 900 python tools/parity_report.py > gpurun_out/r2n_report_default.txt 2>&1
MDR_LIB_PATH=paper_2410_10447_b200/variants/rcp1/libmdr_b200.so PARITY_OUT=r2n_report_rcp1.json timeout 900 python tools/parity_report.py > gpurun_out/r2n_report_rcp1.txt 2>&1
grep -h "fp64fast" gpurun_out/r2n_report_default.txt gpurun_out/r2n_report_rcp1.txt | cut -c1-150
AB_OUT=r2n_ab.json timeout 900 python tools/ls_ab.py "MDR_LS_WARPS=2" "MDR_LIB_PATH=paper_2410_10447_b200/variants/rcp1/libmdr_b200.so"
