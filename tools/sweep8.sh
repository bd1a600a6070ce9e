for cfg in "SP_ATTN_NW=4" "SP_ATTN_NW=6" "SP_ATTN_NW=8"; do
  echo "== $cfg"; env $cfg timeout 200 python tools/graph_probe.py 2>&1 | grep -E "L=|Error"
done
SP_ATTN_NW=6 timeout 300 python -m pytest tests/test_gpu_kernels.py -q -k attention 2>&1 | tail -1
