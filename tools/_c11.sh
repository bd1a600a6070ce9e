export LS=16,32,48,64,96,128,192
O=SP_LIB_OVERRIDE=paper_2408_12526_b200/_lib/old/libstudentpar_b200.so
timeout 1200 bash tools/knob_sweep.sh "$O" "X=0" "$O" "X=0" "SP_GEMM_EPI4_MAXBN=0" > gpurun_out/c11_sweep.txt 2>&1
