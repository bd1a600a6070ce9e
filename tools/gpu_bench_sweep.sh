# bench (engine arm + reference arm, driver-sized and long) then the parity seed sweep; logs in gpurun_out/
set -x
P=${1:-b}
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${P}_bench20.json 2> gpurun_out/${P}_bench20.err; echo "bench20 rc=$?"
timeout 900 python bench.py --steps 500 --warmup 20 --no-cpu-baseline > gpurun_out/${P}_bench500.json 2> gpurun_out/${P}_bench500.err; echo "bench500 rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/${P}_ref.json 2> gpurun_out/${P}_ref.err; echo "ref rc=$?"
timeout 2400 python tools/parity_sweep.py > gpurun_out/${P}_sweep.txt 2> gpurun_out/${P}_sweep.err; echo "sweep rc=$?"
tail -3 gpurun_out/${P}_sweep.txt
