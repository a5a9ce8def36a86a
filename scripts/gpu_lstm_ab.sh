#!/bin/bash
# LSTM option A/B at full C3 size (bench --model lstm, short runs)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
TAG=${1:-ab}
shift
for o in "$@"; do
  timeout 600 python bench.py --model lstm --steps 2 --warmup 3 --no-baseline --no-nockpt --opt $o 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$o', d['ms_per_step'], d['roofline']['per_kind'])" >> gpurun_out/${TAG}.txt
done
cat gpurun_out/${TAG}.txt
