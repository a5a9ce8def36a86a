#!/bin/bash
# LSTM profile set (GPU box): launch list of one T=64 step (after 2 warm-up steps) and
# ncu --set full of its main kernels.  usage: bash scripts/gpu_lstm_prof.sh TAG
cd "$GRAFT_REPO_ROOT"
TAG=${1:-r1}
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout -s KILL 900 $NCU --metrics gpu__time_duration.sum --clock-control none -s 3200 -c 1600 --csv \
  --log-file gpurun_out/${TAG}_lstm_launches.csv python scripts/lstm_step.py 64 2 > gpurun_out/${TAG}_lstm_ncu.log 2>&1
echo "launches rc=$?" >> gpurun_out/${TAG}_lstm_ncu.log
timeout -s KILL 900 $NCU --set full --clock-control none --import-source on \
  -k regex:"tc_gemm|lstm_gates_cell|lstm_cell_bwd_dpre|lstm_head_ce" -s 200 -c 10 -o gpurun_out/${TAG}_lstm_full -f \
  python scripts/lstm_step.py 64 1 > gpurun_out/${TAG}_lstm_full.log 2>&1
echo "full rc=$?" >> gpurun_out/${TAG}_lstm_full.log
tail -n 2 gpurun_out/${TAG}_lstm_ncu.log gpurun_out/${TAG}_lstm_full.log
