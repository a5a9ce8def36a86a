#!/bin/bash
# flag-chained forward Blocks: chain GPU tests, timeline A/B, bench line
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
PHASES=1 timeout -s KILL 300 python scripts/chain_timeline.py > gpurun_out/f_timeline_on.txt 2>&1
PHASES=1 timeout -s KILL 300 python scripts/chain_timeline.py blk_flags=0 > gpurun_out/f_timeline_off.txt 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_chain.py tests/test_gpu_block.py tests/test_gpu_dp.py -x -q > gpurun_out/f_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/f_tests.txt
timeout -s KILL 600 python bench.py --no-baseline > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
