#!/bin/bash
# LSTM recompute scheduling A/B: A24 plan + mirror streams (default) vs mirror units on the layer
# streams vs the plain grouped plan (sequential recompute)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for cfg in "" "--opt lstm_streams=1" "--lstm-parity 0" "--lstm-parity 0 --opt lstm_streams=1"; do
  echo "== $cfg" >> gpurun_out/ls_bench.txt
  timeout -s KILL 600 python bench.py --model lstm --steps 3 --no-baseline --no-nockpt $cfg 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['activation_gb'])" >> gpurun_out/ls_bench.txt 2>&1
done
