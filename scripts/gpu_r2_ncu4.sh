cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
if [ ! -f /tmp/r2_blk_iso.ncu-rep ]; then
timeout -s KILL 900 ncu -k regex:blk_kernel -c 10 --section SourceCounters --section WarpStateStats --import-source on -o /tmp/r2_blk_iso -f python scripts/blk_phases.py 2 > gpurun_out/r2_ncu_log4.txt 2>&1
fi
ncu -i /tmp/r2_blk_iso.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r2_blk_cudasass4.csv 2>&1
