timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x -k "gemm or not opt_in" 2>&1 | tail -2 > gpurun_out/c44_tests.txt
export LS=16,32,64,80,96,112,128,160,192,256,320,384,448,512
timeout 2400 bash tools/knob_sweep.sh "X=0" "SP_GEMM_MAXBN=128" "SP_PERSIST_WPOL=0" "SP_GEMM_SMEM_KB=110" "SP_GEMM_WKEEP=1" > gpurun_out/c44_sweep.txt 2>&1
