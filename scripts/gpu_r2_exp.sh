cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 300 python scripts/chain_timeline.py > gpurun_out/r2_timeline_exp.txt 2>&1
SLM_LIB=libslm_nb4.so timeout -s KILL 300 python scripts/chain_timeline.py >> gpurun_out/r2_timeline_exp.txt 2>&1
