cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_block.py -q --timeout 300 > gpurun_out/r2_blk_test.txt 2>&1
echo "rc=$?" >> gpurun_out/r2_blk_test.txt
timeout -s KILL 200 python scripts/blk_phases.py 2 1 > gpurun_out/r2_blk_phases_exp.txt 2>&1
for c in 2 1; do timeout -s KILL 300 python scripts/chain_timeline.py block_cfg=$c >> gpurun_out/r2_timeline_exp.txt 2>&1; done
