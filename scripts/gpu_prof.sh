#!/bin/bash
# usage: bash scripts/gpu_prof.sh TAG   (runs on the GPU box; outputs in gpurun_out/)
cd "$GRAFT_REPO_ROOT"
TAG=${1:-r1}
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
# 1) launch list (device time per launch) of the bench command, one full step after warm-up
timeout -s KILL 1200 $NCU --metrics gpu__time_duration.sum --clock-control none -s 31000 -c 10200 --csv \
  --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-baseline --no-nockpt > gpurun_out/${TAG}_ncu_bench.log 2>&1
echo "launches rc=$?" >> gpurun_out/${TAG}_ncu_bench.log
# 2) full sets of the top kernels (GEMM kinds + the SIMT kernels)
timeout -s KILL 900 $NCU --set full --clock-control none --import-source on -k regex:"tc_gemm|bn_act|bn_bwd" \
  -s 300 -c 8 -o gpurun_out/${TAG}_full -f \
  python bench.py --layers 64 --steps 1 --warmup 3 --no-baseline --no-nockpt > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/${TAG}_ncu_full.log
tail -3 gpurun_out/${TAG}_ncu_bench.log gpurun_out/${TAG}_ncu_full.log
