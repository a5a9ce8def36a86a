#!/bin/bash
# ncu --set full of the LSTM's persistent forward / backward runs and its launch list (T = 64)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout -s KILL 900 $NCU --set full --clock-control none --import-source on -k regex:"lstm_(fwd|bwd)_run_kernel|tc_gemm" \
  -s 200 -c 8 -o gpurun_out/r2_lstm_full -f \
  python bench.py --model lstm --unroll 64 --steps 1 --warmup 2 --no-baseline --no-nockpt > gpurun_out/r2_lstm_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r2_lstm_ncu.log
timeout -s KILL 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_lstm_launches.csv \
  python bench.py --model lstm --unroll 64 --steps 1 --warmup 2 --no-baseline --no-nockpt > gpurun_out/r2_lstm_ncu2.log 2>&1
echo "rc=$?" >> gpurun_out/r2_lstm_ncu2.log
