#!/bin/bash
# A/B sweep of model options on the full bench config (headline timing only)
cd "$GRAFT_REPO_ROOT"
TAG=${1:-sw}
mkdir -p gpurun_out
: > gpurun_out/${TAG}_sweep.txt
while read -r OPTS; do
  ARGS=""
  for o in $OPTS; do ARGS="$ARGS --opt $o"; done
  R=$(timeout -s KILL 240 python bench.py --steps 6 --warmup 3 --no-baseline --no-nockpt $ARGS 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'])")
  echo "[$OPTS] $R" >> gpurun_out/${TAG}_sweep.txt
done < ${2:-scripts/sweep2.txt}
cat gpurun_out/${TAG}_sweep.txt
