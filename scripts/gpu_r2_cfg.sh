cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_block.py -q --timeout 300 > gpurun_out/r2_blk_test.txt 2>&1
echo "rc=$?" >> gpurun_out/r2_blk_test.txt
for c in 1 2; do
  PHASES=1 timeout -s KILL 300 python scripts/chain_timeline.py block_cfg=$c > gpurun_out/r2_timeline_cfg$c.txt 2>&1
  timeout -s KILL 300 python scripts/chain_timeline.py block_cfg=$c >> gpurun_out/r2_timeline_cfg$c.txt 2>&1
done
