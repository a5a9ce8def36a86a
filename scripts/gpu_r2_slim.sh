#!/bin/bash
# slim mirror Blocks: chain GPU tests (bitwise ckpt == no-ckpt with slim mirrors), timeline A/B, bench
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_chain.py tests/test_gpu_dp.py -x -q > gpurun_out/s_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/s_tests.txt
PHASES=1 timeout -s KILL 300 python scripts/chain_timeline.py > gpurun_out/s_tl_on.txt 2>&1
PHASES=1 timeout -s KILL 300 python scripts/chain_timeline.py slim_mirror=0 > gpurun_out/s_tl_off.txt 2>&1
timeout -s KILL 600 python bench.py --no-baseline > gpurun_out/s_bench.json 2> gpurun_out/s_bench.err
