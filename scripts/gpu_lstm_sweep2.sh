#!/bin/bash
cd "$GRAFT_REPO_ROOT"
TAG=${1:-lw}
mkdir -p gpurun_out
: > gpurun_out/${TAG}_sweep.txt
run() {
  timeout -s KILL 400 python bench.py --model lstm --steps 3 --warmup 3 --no-baseline --no-nockpt "$@" > gpurun_out/${TAG}_tmp.txt 2>&1
  echo "$* :: $(tail -n 1 gpurun_out/${TAG}_tmp.txt | python -c "
import json,sys
try:
  j=json.loads(sys.stdin.read()); print(j['ms_per_step'])
except Exception as e: print('ERR', e)")" >> gpurun_out/${TAG}_sweep.txt
}
run
run --opt lstm_fuse_cell=1
run --opt lstm_early_trigger=0
run --opt lstm_grid=0
run --opt prio=1
run --opt lstm_skx=3
cat gpurun_out/${TAG}_sweep.txt
