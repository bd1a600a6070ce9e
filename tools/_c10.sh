export LS=384,400,416,432,448,464,480
timeout 900 bash tools/knob_sweep.sh "X=0" "SP_ATTN_TC=1" > gpurun_out/c10_sweep.txt 2>&1
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/c10_bench.json 2> gpurun_out/c10_bench.err
