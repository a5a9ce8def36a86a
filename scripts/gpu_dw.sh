#!/bin/bash
cd "$GRAFT_REPO_ROOT"
TAG=${1:-dw1}
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_chain.py -x -q --timeout 300 > gpurun_out/${TAG}_chain.txt 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_chain.txt
tail -n 3 gpurun_out/${TAG}_chain.txt
python scripts/chain_timeline.py > gpurun_out/${TAG}_tl.txt 2>&1
python scripts/chain_timeline.py dw_tma=0 >> gpurun_out/${TAG}_tl.txt 2>&1
cat gpurun_out/${TAG}_tl.txt
