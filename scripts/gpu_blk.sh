#!/bin/bash
cd "$GRAFT_REPO_ROOT"
TAG=${1:-bk}
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_chain.py -q --timeout 120 -k "cluster_block" > gpurun_out/${TAG}_t.txt 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_t.txt
grep -E "passed|failed|Error|assert" gpurun_out/${TAG}_t.txt | head -20
for o in blk_cluster=4 blk_cluster=2; do timeout -s KILL 200 python scripts/chain_timeline.py $o 2>&1 | head -6; done
