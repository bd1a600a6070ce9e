# latency probes (run under gpurun): per-length graph latency, per-launch breakdown, GEMM CTA timeline
set -x
P=${1:-p}
timeout 600 python tools/len_probe.py 16,32,64,96,128,160,192,256,320,384,448,512 > gpurun_out/${P}_len.txt 2>&1; echo "len rc=$?"
timeout 600 python tools/kind_profile.py 16,128,256,512 > gpurun_out/${P}_kinds.txt 2>&1; echo "kinds rc=$?"
timeout 600 python tools/trace_forward.py 16,64,128 > gpurun_out/${P}_trace.txt 2>&1; echo "trace rc=$?"
cat gpurun_out/${P}_len.txt
