#!/bin/bash
# overlap variants: stream priorities, split-K / tile options (C2 bench, no baseline/no-ckpt legs)
cd "$GRAFT_REPO_ROOT"
TAG=${1:-sw}
mkdir -p gpurun_out
: > gpurun_out/${TAG}_sweep.txt
run() {
  timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-baseline --no-nockpt "$@" > gpurun_out/${TAG}_tmp.txt 2>&1
  echo "$* :: $(tail -n 2 gpurun_out/${TAG}_tmp.txt | head -n 1 | python -c "
import json,sys
try:
  j=json.loads(sys.stdin.read()); r=j['roofline']['per_kind']; print(j['ms_per_step'], j['config'].get('recompute','')[:10], {k: v['avg_us'] for k, v in r.items()})
except Exception as e: print('ERR', e)")" >> gpurun_out/${TAG}_sweep.txt
}
run
run --opt prio=1
run --opt s3_prio=2
run --opt prio=1 --opt s3_prio=2
run --opt prio=1 --opt s3_prio=5
run --opt sk_fwd=4
run --opt sk_dx=4
run --opt sk_fwd=1
run --opt fused_bn=256
cat gpurun_out/${TAG}_sweep.txt
