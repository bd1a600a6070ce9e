for cfg in "SP_GEMM_WKEEP=0" "SP_GEMM_WKEEP=1"; do
  echo "== $cfg"; env $cfg timeout 200 python tools/trace_gemm.py 256 2>&1 | grep -E "event|mma0|commit_last|epi0|end|entry"
  env $cfg timeout 200 python tools/graph_probe.py 2>&1 | grep -E "L=|Error"
done
