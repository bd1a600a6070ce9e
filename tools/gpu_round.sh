# full GPU pass (run under gpurun): tests, smoke, bench (driver-sized + long), reference arm,
# bursty serving, length probe; logs under gpurun_out/<prefix>_*
set -x
P=${1:-g}
timeout 300 python __graft_entry__.py smoke > gpurun_out/${P}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${P}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${P}_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/${P}_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${P}_bench20.json 2> gpurun_out/${P}_bench20.err; echo "bench20 rc=$?"
timeout 900 python bench.py --steps 500 --warmup 20 --no-cpu-baseline > gpurun_out/${P}_bench500.json 2> gpurun_out/${P}_bench500.err; echo "bench500 rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/${P}_ref.json 2> gpurun_out/${P}_ref.err; echo "ref rc=$?"
timeout 900 python tools/serve_bursty.py --out gpurun_out/${P}_serve.json > gpurun_out/${P}_serve.log 2>&1; echo "serve rc=$?"; tail -3 gpurun_out/${P}_serve.log
timeout 600 python tools/len_probe.py 16,32,64,96,128,160,192,256,320,384,448,512 > gpurun_out/${P}_len.txt 2>&1; cat gpurun_out/${P}_len.txt
