#!/bin/bash
cd "$GRAFT_REPO_ROOT"
TAG=${1:-bv}
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_chain.py -q --timeout 120 -k "bn_vec or overlapped" > gpurun_out/${TAG}_t.txt 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_t.txt
grep -E "passed|failed|Error|assert" gpurun_out/${TAG}_t.txt | head -10
for o in "" bn_vec=1 "bn_vec=1 sk_fwd=4" "bn_vec=1 sk_fwd=4 sk_dx=4"; do timeout -s KILL 200 python scripts/chain_timeline.py $o 2>&1 | head -4; done
