cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 2400 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/r2_gpu_all.txt 2>&1
echo "rc=$?" >> gpurun_out/r2_gpu_all.txt
timeout -s KILL 600 python bench.py --steps 20 --warmup 5 --no-baseline > gpurun_out/r2_bench2.txt 2>&1
echo "bench rc=$?" >> gpurun_out/r2_bench2.txt
