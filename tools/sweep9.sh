timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -3
for cfg in "SP_LN_FUSE=0" "SP_LN_FUSE=1 SP_LN_FUSE_MIN_CTAS=96" "SP_LN_FUSE=1 SP_LN_FUSE_MIN_CTAS=1" "SP_LN_FUSE=1 SP_LN_FUSE_MIN_CTAS=100000"; do
  echo "== $cfg"; env $cfg timeout 200 python tools/graph_probe.py 2>&1 | grep -E "L=|Error"
done
