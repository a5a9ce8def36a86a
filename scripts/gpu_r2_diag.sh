cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 300 python scripts/diag_block.py parity 8 64 256 8 > gpurun_out/r2_diag_parity.txt 2>&1
timeout -s KILL 300 python scripts/diag_block.py parity 4 256 512 12 >> gpurun_out/r2_diag_parity.txt 2>&1
timeout -s KILL 600 ncu -k regex:blk_kernel --launch-skip 8 -c 3 --set full --import-source on -o gpurun_out/r2_blk_full -f python scripts/diag_block.py prof 8 256 2048 > gpurun_out/r2_ncu_log.txt 2>&1
ncu -i gpurun_out/r2_blk_full.ncu-rep --page details --csv > gpurun_out/r2_blk_details.csv 2>&1
ncu -i gpurun_out/r2_blk_full.ncu-rep --page raw --csv > gpurun_out/r2_blk_raw.csv 2>&1
