# Per-length batch-1 latency and the L~U{16..512} mean for each engine configuration:
#   bash tools/knob_sweep.sh "X=0" "SP_ATTN_NW=6" ...
LS=${LS:-16,64,128,160,192,224,256,288,320,352,384,416,448,480,512}
for cfg in "$@"; do
  r=$(env $cfg timeout 300 python tools/len_probe.py $LS 2>/dev/null)
  python - "$cfg" "$r" <<'PY'
import sys
cfg, r = sys.argv[1], sys.argv[2].split()
pts = sorted((int(a), float(b)) for a, b in (x.split(":") for x in r))
# trapezoid mean over L in [16, 512] (bench distribution U{16..512})
area = sum((x1 - x0) * (y0 + y1) / 2 for (x0, y0), (x1, y1) in zip(pts, pts[1:]))
print(f"{cfg:45s} mean {area / (pts[-1][0] - pts[0][0]):6.1f}  " + " ".join(f"{a}:{b:.1f}" for a, b in pts))
PY
done
