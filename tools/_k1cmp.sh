timeout 900 python -m pytest tests -m gpu -x -q -k "not full_size" 2>&1 | tail -2
for i in 1 2 3; do python bench.py --no-cpu-baseline --steps 10 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['phases_ms'])"; done
