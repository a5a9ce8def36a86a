#!/bin/bash
cd "$GRAFT_REPO_ROOT"
TAG=${1:-ov1}
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_chain.py -x -q --timeout 300 -k "overlap or bitwise" > gpurun_out/${TAG}_chain.txt 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_chain.txt
tail -n 5 gpurun_out/${TAG}_chain.txt
for MP in 1 0; do
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-baseline --mirror-parity $MP > gpurun_out/${TAG}_bench_mp$MP.txt 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_bench_mp$MP.txt
tail -n 2 gpurun_out/${TAG}_bench_mp$MP.txt | head -n 1 | python -c "
import json,sys; j=json.loads(sys.stdin.read()); r=j['roofline']; print(j['ms_per_step'], j['config']['recompute'], j['activation_gb'], j['ckpt_over_nockpt_time'], r['per_kind'])"
done
