cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 600 ncu -k regex:blk_kernel -c 4 --set full --import-source on -o gpurun_out/r2_blk_full2 -f python scripts/blk_phases.py > gpurun_out/r2_ncu_log2.txt 2>&1
ncu -i gpurun_out/r2_blk_full2.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_blk_sass2.csv 2>&1
ncu -i gpurun_out/r2_blk_full2.ncu-rep --page details --csv > gpurun_out/r2_blk_details2.csv 2>&1
