#!/bin/bash
cd "$GRAFT_REPO_ROOT"
TAG=${1:-ep}
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/${TAG}_t.txt 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_t.txt
tail -n 3 gpurun_out/${TAG}_t.txt
python scripts/gemm_phases.py 0,128,2 1,128,2 2,256,1,256,0,2048,2048 2>&1 | tail -3
timeout -s KILL 200 python scripts/chain_timeline.py 2>&1 | head -5
timeout -s KILL 400 python bench.py --model lstm --steps 3 --no-baseline --no-nockpt 2>&1 | tail -n 1 | cut -c 1-200
