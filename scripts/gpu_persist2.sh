#!/bin/bash
cd "$GRAFT_REPO_ROOT"
TAG=${1:-p2}
mkdir -p gpurun_out
timeout -s KILL 120 python scripts/persist_phases.py > gpurun_out/${TAG}_phases.txt 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_phases.txt
cat gpurun_out/${TAG}_phases.txt | tail -n 12
timeout -s KILL 600 python -m pytest tests/test_gpu_chain.py -x -q --timeout 200 > gpurun_out/${TAG}_chain.txt 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_chain.txt
tail -n 3 gpurun_out/${TAG}_chain.txt
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-baseline > gpurun_out/${TAG}_bench_on.txt 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_bench_on.txt
tail -n 2 gpurun_out/${TAG}_bench_on.txt | head -n 1 | python -c "
import json,sys; j=json.loads(sys.stdin.read()); r=j['roofline']; print(j['ms_per_step'], r['per_kind'], r.get('gemm_share_of_step'), j.get('no_ckpt',{}))"
