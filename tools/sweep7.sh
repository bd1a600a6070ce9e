timeout 300 python -m pytest tests/test_gpu_kernels.py -q -k attention --timeout 120 2>&1 | tail -15
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 2>&1 | tail -3
for cfg in "SP_ATTN_TC=0" "SP_ATTN_TC=1"; do
  echo "== $cfg"; env $cfg timeout 200 python tools/graph_probe.py 2>&1 | grep -E "L=|Error"
done
