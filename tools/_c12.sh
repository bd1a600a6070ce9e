timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_configs.py -q -x 2>&1 | tail -2 > gpurun_out/c12_tests.txt
export LS=16,32,64,128,192,256,320,384,448,512
O=SP_LIB_OVERRIDE=paper_2408_12526_b200/_lib/old/libstudentpar_b200.so
timeout 1200 bash tools/knob_sweep.sh "$O" "X=0" "$O" "X=0" > gpurun_out/c12_sweep.txt 2>&1
