timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q --timeout 300 -x 2>&1 | tail -3
for cfg in "SP_GEMM_PERSIST_MIN_ROWS=100000" "SP_GEMM_PERSIST_MIN_ROWS=129" "SP_GEMM_PERSIST_MIN_ROWS=200"; do
  echo "== $cfg"; env $cfg timeout 200 python tools/graph_probe.py 2>&1 | grep -E "L=|Error"
done
