# quick GPU check (run under gpurun): smoke, GPU tests, latency probes
set -x
P=${1:-q}
timeout 300 python __graft_entry__.py smoke > gpurun_out/${P}_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/${P}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -x > gpurun_out/${P}_tests.log 2>&1; echo "tests rc=$?"
tail -8 gpurun_out/${P}_tests.log
timeout 600 python tools/len_probe.py 16,32,64,96,128,160,192,256,320,384,448,512 > gpurun_out/${P}_len.txt 2>&1; echo "len rc=$?"
cat gpurun_out/${P}_len.txt
timeout 600 python tools/kind_profile.py 16,512 > gpurun_out/${P}_kinds.txt 2>&1; echo "kinds rc=$?"
