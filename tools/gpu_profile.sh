# Profiles for profiles/ (run under gpurun, one GPU): the ncu launch list of the default bench, full
# captures of the main kernels at batch-1 L=16 / L=512 and the BERT-large batched pair GEMM, and the
# batched bench line. Every ncu run follows the same command's plain run (exit 0).
set -x
P=${1:-u}
S="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --profile-steps 2"
timeout 300 $S > gpurun_out/${P}_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 200 --csv --log-file gpurun_out/${P}_launches_b8.csv $S > gpurun_out/${P}_ncu_l.log 2>&1; echo "launch list rc=$?"
timeout 120 python tools/one_request.py 16 base 4 > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel|reduce_ln|attn" -s 17 -c 8 -o gpurun_out/${P}_L16 python tools/one_request.py 16 base 4 > gpurun_out/${P}_ncu_a.log 2>&1; echo "ncu L16 rc=$?"
timeout 120 python tools/one_request.py 512 base 4 > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_persistent|mlp_persistent|attn_tc3|reduce_ln|embed_ln" -s 12 -c 10 -o gpurun_out/${P}_L512 python tools/one_request.py 512 base 4 > gpurun_out/${P}_ncu_b.log 2>&1; echo "ncu L512 rc=$?"
timeout 900 python bench.py --config large --batch 16 --steps 40 --warmup 4 --no-cpu-baseline --profile-steps 10 > gpurun_out/${P}_bench_l12_b16.json 2> gpurun_out/${P}_bench_l12.err; echo "bench l12 rc=$?"
L="python bench.py --config large --batch 16 --steps 3 --warmup 2 --no-cpu-baseline --profile-steps 1"
timeout 600 $L > gpurun_out/${P}_plain_l.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_persistent -s 4 -c 3 -o gpurun_out/${P}_l12 $L > gpurun_out/${P}_ncu_c.log 2>&1; echo "ncu l12 rc=$?"
