# Compare engine knobs on the batch-1 latency probe (and optionally the batched L12 bench):
#   bash tools/sweep_env.sh "SP_PERSIST_PAIR=0" "SP_PERSIST_PAIR=1" ...
# Each argument is one set of environment assignments (knobs are read once per process).
for cfg in "$@"; do
  echo "== $cfg"
  env $cfg timeout 200 python tools/graph_probe.py 2>&1 | grep -E "L=|Error"
  if [ -n "$SWEEP_L12" ]; then
    env $cfg timeout 600 python bench.py --config large --batch 16 --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('L12 b16', round(d['value'],1), round(d['roofline']['frac'],3))"
  fi
done
