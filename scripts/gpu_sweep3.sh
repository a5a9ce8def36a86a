#!/bin/bash
cd "$GRAFT_REPO_ROOT"
TAG=${1:-s3}
mkdir -p gpurun_out
: > gpurun_out/${TAG}_sweep.txt
run() {
  timeout -s KILL 400 python bench.py --steps 6 --warmup 3 --no-baseline --no-nockpt "$@" > gpurun_out/${TAG}_tmp.txt 2>&1
  echo "$* :: $(tail -n 2 gpurun_out/${TAG}_tmp.txt | head -n 1 | python -c "
import json,sys
try:
  j=json.loads(sys.stdin.read()); print(j['ms_per_step'])
except Exception as e: print('ERR', e)")" >> gpurun_out/${TAG}_sweep.txt
}
run --opt fused_bn=64
run --opt fused_bn=64 --opt sk_fwd=1
run --opt fused_bn=64 --opt sk_dx=1
run --model lstm --steps 3 --opt lstm_skx=2
run --model lstm --steps 3 --opt lstm_skx=8
run --model lstm --steps 3 --opt lstm_sk=2
run --model lstm --steps 3 --seg 32
run --model lstm --steps 3 --seg 128
cat gpurun_out/${TAG}_sweep.txt
