timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -2
for v in 0 1; do echo "== SP_PERSIST_PAIR=$v"; SP_PERSIST_PAIR=$v timeout 200 python tools/graph_probe.py 2>&1 | grep -E "L=|Error"
SP_PERSIST_PAIR=$v timeout 600 python bench.py --config large --batch 16 --steps 20 --warmup 3 --no-cpu-baseline --profile-steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('L12 b16', round(d['value'],1), round(d['roofline']['frac'],3))"; done
