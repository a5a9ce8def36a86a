cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt 2>&1
timeout -s KILL 120 ./scripts/mb_cluster > gpurun_out/r2_mb_cluster.txt 2>&1
echo "rc=$?" >> gpurun_out/r2_mb_cluster.txt
timeout -s KILL 400 python bench.py --steps 10 --warmup 3 --no-baseline > gpurun_out/r2_bench0.txt 2>&1
echo "bench rc=$?" >> gpurun_out/r2_bench0.txt
