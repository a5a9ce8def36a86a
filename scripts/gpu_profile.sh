#!/bin/bash
# Round-2 profile pass (GPU box): device-clock phase timeline of the C2 step, the ncu launch list of
# the bench command, and ncu --set full of the fused Block kernels on a 64-layer chain.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r2}
NCU=/usr/local/cuda/bin/ncu
PHASES=1 timeout -s KILL 300 python scripts/chain_timeline.py > gpurun_out/${TAG}_timeline.txt 2>&1
timeout -s KILL 1200 $NCU --metrics gpu__time_duration.sum --clock-control none -s 16500 -c 8300 --csv \
  --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-baseline --no-nockpt --no-lstm > gpurun_out/${TAG}_ncu_bench.log 2>&1
echo "launches rc=$?" >> gpurun_out/${TAG}_ncu_bench.log
timeout -s KILL 900 $NCU --set full --clock-control none --import-source on -k regex:"blk_kernel|tc_gemm" \
  -s 400 -c 6 -o gpurun_out/${TAG}_full -f \
  python bench.py --layers 64 --steps 1 --warmup 3 --no-baseline --no-nockpt --no-lstm > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/${TAG}_ncu_full.log
