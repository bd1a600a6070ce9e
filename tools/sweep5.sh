for cfg in "SP_GEMM_L2PREFETCH=0" "SP_GEMM_L2PREFETCH=1"; do
  echo "== $cfg"; env $cfg timeout 200 python tools/graph_probe.py 2>&1 | grep -E "L=|Error"
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
