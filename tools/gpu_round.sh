set -x
timeout 900 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -15
timeout 600 python bench.py > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_r1.err
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --profile-steps 2"
timeout 300 $B > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 200 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 30 -c 4 -o gpurun_out/prof_gemm $B > gpurun_out/ncu2.log 2>&1; echo "ncu2 rc=$?"
