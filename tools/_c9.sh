LS=256,320,384,416,448,480,512
for cfg in "SP_ATTN_TC=1" "SP_ATTN_TC=0" "SP_ATTN_TC=0 SP_ATTN_NW=4 SP_ATTN_MINB=3" "SP_ATTN_TC=0 SP_ATTN_NW=4 SP_ATTN_MINB=4" "SP_ATTN_TC=0 SP_ATTN_NW=6 SP_ATTN_MINB=2" "SP_ATTN_TC=0 SP_ATTN_NW=6 SP_ATTN_MINB=3" "SP_ATTN_TC=0 SP_ATTN_NW=8 SP_ATTN_MINB=2"; do
  echo "== $cfg"; env $cfg timeout 120 python tools/attn_bench.py $LS 2>&1 | tr '\n' ' '; echo
done > gpurun_out/c9_attn.txt
