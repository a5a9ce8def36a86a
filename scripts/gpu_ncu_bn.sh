#!/bin/bash
cd "$GRAFT_REPO_ROOT"
TAG=${1:-it}
mkdir -p gpurun_out
timeout -s KILL 300 python scripts/gemm_phases.py 0,256,8 1,256,8 0,256,4 0,128,8 0,256,2 > gpurun_out/${TAG}_phases.txt 2>&1
timeout -s KILL 900 /usr/local/cuda/bin/ncu --set full --cache-control none --clock-control none --import-source on \
  -k regex:"bn_act_rk|bn_bwd_rk|EpiPartial" -s 300 -c 6 -o gpurun_out/${TAG}_bnfull -f \
  python bench.py --layers 32 --steps 1 --warmup 3 --no-baseline --no-nockpt > gpurun_out/${TAG}_bnfull.log 2>&1
