#!/bin/bash
# ncu --set full of one launch of each top kernel in the bench configuration (warm caches)
cd "$GRAFT_REPO_ROOT"
TAG=${1:-r1}
LAYERS=${2:-64}
mkdir -p gpurun_out
timeout -s KILL 900 /usr/local/cuda/bin/ncu --set full --cache-control none --clock-control none --import-source on \
  -k regex:"tc_gemm|bn_act|bn_bwd" -s 400 -c 8 -o gpurun_out/${TAG}_full -f \
  python bench.py --layers $LAYERS --steps 1 --warmup 3 --no-baseline --no-nockpt > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/${TAG}_ncu_full.log
