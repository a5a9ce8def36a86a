cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_block.py -q --timeout 300 > gpurun_out/r2_blk_test.txt 2>&1
echo "rc=$?" >> gpurun_out/r2_blk_test.txt
timeout -s KILL 200 python scripts/blk_phases.py > gpurun_out/r2_blk_phases.txt 2>&1
PHASES=1 timeout -s KILL 300 python scripts/chain_timeline.py > gpurun_out/r2_timeline.txt 2>&1
