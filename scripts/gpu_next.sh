#!/bin/bash
cd "$GRAFT_REPO_ROOT"
TAG=${1:-nx}
mkdir -p gpurun_out
: > gpurun_out/${TAG}_sweep.txt
run() {
  timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-baseline --no-nockpt "$@" > gpurun_out/${TAG}_tmp.txt 2>&1
  echo "$* :: $(tail -n 2 gpurun_out/${TAG}_tmp.txt | head -n 1 | python -c "
import json,sys
try:
  j=json.loads(sys.stdin.read()); r=j['roofline']['per_kind']; print(j['ms_per_step'], {k: v['avg_us'] for k, v in r.items()})
except Exception as e: print('ERR', e)")" >> gpurun_out/${TAG}_sweep.txt
}
run
run --opt dw_lag=4
run --opt dw_lag=8
cat gpurun_out/${TAG}_sweep.txt
timeout -s KILL 600 python -m pytest tests/test_gpu_chain.py -x -q --timeout 300 > gpurun_out/${TAG}_chain.txt 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_chain.txt
tail -n 2 gpurun_out/${TAG}_chain.txt
bash scripts/gpu_lstm_ov.sh ${TAG}
