cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
N=64 timeout -s KILL 900 ncu -k regex:blk_kernel --launch-skip 10 -c 30 --section SourceCounters --section WarpStateStats --import-source on -o /tmp/r2_blk_src -f python scripts/chain_timeline.py > gpurun_out/r2_ncu_log3.txt 2>&1
ncu -i /tmp/r2_blk_src.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_blk_sass3.csv 2>&1
