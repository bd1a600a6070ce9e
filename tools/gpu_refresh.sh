# Round evidence refresh: GPU tests, bench lines (all configs + reference arm), serving trace,
# ncu launch list of the default bench and full captures of the top kernels. Outputs in gpurun_out/.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_b8.json 2> gpurun_out/bench_b8.err; echo "b8 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 python bench.py --config large --batch 16 --steps 200 --warmup 10 > gpurun_out/bench_l12_b16.json 2> gpurun_out/bench_l12.err; echo "l12 rc=$?"
timeout 900 python bench.py --config k32 --steps 500 --warmup 20 --no-cpu-baseline > gpurun_out/bench_k32.json 2> gpurun_out/bench_k32.err; echo "k32 rc=$?"
timeout 900 python tools/serve_bursty.py > gpurun_out/serve_bursty.json 2> gpurun_out/serve.err; echo "serve rc=$?"
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --profile-steps 2"
timeout 300 $B > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 200 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_l.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 30 -c 4 -o gpurun_out/prof_gemm_b8 $B > gpurun_out/ncu_g.log 2>&1; echo "gemm rc=$?"
timeout 300 python tools/one_request.py 512 base 2 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 2 -c 1 -o gpurun_out/prof_attn512 python tools/one_request.py 512 base 2 > gpurun_out/ncu_a.log 2>&1; echo "attn rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_persistent -s 4 -c 4 -o gpurun_out/prof_persist512 python tools/one_request.py 512 base 2 > gpurun_out/ncu_p.log 2>&1; echo "persist rc=$?"
