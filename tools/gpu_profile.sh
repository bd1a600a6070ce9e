# Round profile: bench lines + ncu launch list + full captures of the top kernels.
set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k opt_in 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench_b8.json 2> gpurun_out/bench_b8.err; echo "bench b8 rc=$?"
timeout 900 python bench.py --config large --batch 16 --steps 40 --warmup 4 --no-cpu-baseline --profile-steps 10 > gpurun_out/bench_l12_b16.json 2> gpurun_out/bench_l12_b16.err; echo "bench l12 rc=$?"
S="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --profile-steps 2"
timeout 300 $S > gpurun_out/plain_s.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 180 --csv --log-file gpurun_out/launches_b8.csv $S > gpurun_out/ncu_l.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 40 -c 4 -o gpurun_out/prof_gemm_b8 $S > gpurun_out/ncu_f1.log 2>&1; echo "ncu gemm b8 rc=$?"
L="python bench.py --config large --batch 16 --steps 3 --warmup 2 --no-cpu-baseline --profile-steps 1"
timeout 600 $L > gpurun_out/plain_l.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_persistent -s 4 -c 2 -o gpurun_out/prof_gemm_l12 $L > gpurun_out/ncu_f2.log 2>&1; echo "ncu gemm l12 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 4 -c 1 -o gpurun_out/prof_attn_l12 $L > gpurun_out/ncu_f3.log 2>&1; echo "ncu attn rc=$?"
