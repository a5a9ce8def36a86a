#!/bin/bash
cd "$GRAFT_REPO_ROOT"
TAG=${1:-tl}
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_chain.py -q --timeout 120 -k "overlapped" > gpurun_out/${TAG}_t.txt 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_t.txt
grep -E "passed|failed|Error|assert" gpurun_out/${TAG}_t.txt | head -10
for o in "" tile_mir=256 tile_dx=256 "tile_mir=256 tile_dx=256"; do timeout -s KILL 200 python scripts/chain_timeline.py $o 2>&1 | head -3; done
