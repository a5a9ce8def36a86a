cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_chain.py -x -q --timeout 300 -k "not c2_full" > gpurun_out/r2_chain.txt 2>&1
echo "chain rc=$?" >> gpurun_out/r2_chain.txt
timeout -s KILL 400 python bench.py --steps 10 --warmup 3 --no-baseline > gpurun_out/r2_bench1.txt 2>&1
echo "bench rc=$?" >> gpurun_out/r2_bench1.txt
