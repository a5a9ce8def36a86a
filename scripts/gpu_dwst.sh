#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout -s KILL 900 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -2
for i in 1 2; do timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-baseline --no-nockpt 2>&1 | tail -n 1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('C2', j['ms_per_step'])"; done
for i in 1 2; do timeout -s KILL 400 python bench.py --model lstm --steps 3 --no-baseline --no-nockpt 2>&1 | tail -n 1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('C3', j['ms_per_step'])"; done
