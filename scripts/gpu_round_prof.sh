#!/bin/bash
# Round profile set (runs on the GPU box; outputs in gpurun_out/):
#   1) the default bench line (C2) and the LSTM bench line (C3)
#   2) ncu launch list (gpu__time_duration, clock-control none) of the default bench command
#   3) ncu --set full of the top kernels on a 64-layer chain
# usage: bash scripts/gpu_round_prof.sh TAG
cd "$GRAFT_REPO_ROOT"
TAG=${1:-r1}
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout -s KILL 900 python bench.py > gpurun_out/${TAG}_bench.txt 2>&1
timeout -s KILL 900 python bench.py --model lstm --steps 3 > gpurun_out/${TAG}_bench_lstm.txt 2>&1
echo "bench rc=$?" >> gpurun_out/${TAG}_bench.txt
timeout -s KILL 1500 $NCU --metrics gpu__time_duration.sum --clock-control none -s 31000 -c 10200 --csv \
  --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-baseline --no-nockpt --no-lstm > gpurun_out/${TAG}_ncu_bench.log 2>&1
echo "launches rc=$?" >> gpurun_out/${TAG}_ncu_bench.log
timeout -s KILL 900 $NCU --set full --clock-control none --import-source on -k regex:"tc_gemm|bn_act|bn_bwd" \
  -s 300 -c 8 -o gpurun_out/${TAG}_full -f \
  python bench.py --layers 64 --steps 1 --warmup 3 --no-baseline --no-nockpt --no-lstm > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/${TAG}_ncu_full.log
tail -n 2 gpurun_out/${TAG}_bench.txt gpurun_out/${TAG}_ncu_bench.log gpurun_out/${TAG}_ncu_full.log | cut -c1-400
