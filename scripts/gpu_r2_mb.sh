cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 120 ./scripts/mb_tc > gpurun_out/r2_mb_tc.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_mb_tc.txt
timeout -s KILL 300 python scripts/mb_cublas.py > gpurun_out/r2_mb_cublas.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_mb_cublas.txt
