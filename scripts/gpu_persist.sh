#!/bin/bash
# persistent forward kernel: chain GPU tests, then bench A/B (persist on / off)
cd "$GRAFT_REPO_ROOT"
TAG=${1:-p1}
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_chain.py -x -q --timeout 200 > gpurun_out/${TAG}_chain.txt 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_chain.txt
tail -n 30 gpurun_out/${TAG}_chain.txt
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-baseline > gpurun_out/${TAG}_bench_on.txt 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_bench_on.txt
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-baseline --no-nockpt --opt persist=0 > gpurun_out/${TAG}_bench_off.txt 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_bench_off.txt
for f in gpurun_out/${TAG}_bench_*.txt; do echo $f; tail -n 2 $f | cut -c1-600; done
