#!/bin/bash
# LSTM: overlapped segment recompute (mirror-run parity plan + mirror streams) vs default
cd "$GRAFT_REPO_ROOT"
TAG=${1:-lo1}
mkdir -p gpurun_out
: > gpurun_out/${TAG}_lstm.txt
run() {
  timeout -s KILL 400 python bench.py --model lstm --steps 3 --warmup 3 --no-baseline --no-nockpt "$@" > gpurun_out/${TAG}_tmp.txt 2>&1
  echo "$* :: $(tail -n 2 gpurun_out/${TAG}_tmp.txt | head -n 1 | python -c "
import json,sys
try:
  j=json.loads(sys.stdin.read()); print(j['ms_per_step'], j.get('activation_gb'))
except Exception as e: print('ERR', e)")" >> gpurun_out/${TAG}_lstm.txt
}
run
run --lstm-parity 1
run --lstm-parity 1 --opt lstm_streams=2
run --opt lstm_streams=2
cat gpurun_out/${TAG}_lstm.txt
timeout -s KILL 600 python -m pytest tests/test_gpu_lstm.py -x -q --timeout 300 > gpurun_out/${TAG}_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_tests.txt
tail -n 2 gpurun_out/${TAG}_tests.txt
