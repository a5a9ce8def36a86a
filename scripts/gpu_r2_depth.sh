cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 900 python scripts/diag_block.py depth 256 2048 1 2 4 8 16 > gpurun_out/r2_depth.txt 2>&1
timeout -s KILL 600 python scripts/diag_block.py depth 64 256 1 2 4 8 16 32 >> gpurun_out/r2_depth.txt 2>&1
