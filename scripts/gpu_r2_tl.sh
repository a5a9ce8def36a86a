cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
PHASES=1 timeout -s KILL 300 python scripts/chain_timeline.py > gpurun_out/r2_timeline.txt 2>&1
STRATEGY=none MP=0 PHASES=1 timeout -s KILL 300 python scripts/chain_timeline.py >> gpurun_out/r2_timeline.txt 2>&1
