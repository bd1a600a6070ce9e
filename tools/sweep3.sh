for cfg in "SP_GEMM_MAXBN=128" "SP_GEMM_MAXBN=256" "SP_GEMM_MAXBN=256 SP_GEMM_SMEM_KB=110" "SP_GEMM_MAXBN=192"; do
  echo "== $cfg"; env $cfg timeout 200 python tools/graph_probe.py 2>&1 | grep -E "L=|Error"
done
