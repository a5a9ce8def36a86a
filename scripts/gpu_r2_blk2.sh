cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_block.py -q --timeout 120 > gpurun_out/r2_blk_test.txt 2>&1
echo "rc=$?" >> gpurun_out/r2_blk_test.txt
timeout -s KILL 200 python scripts/blk_phases.py > gpurun_out/r2_blk_phases.txt 2>&1
echo "rc=$?" >> gpurun_out/r2_blk_phases.txt
timeout -s KILL 300 python scripts/diag_block.py parity 8 64 256 8 > gpurun_out/r2_diag_parity.txt 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_chain.py -q --timeout 300 -k "not c2_full" > gpurun_out/r2_chain.txt 2>&1
echo "chain rc=$?" >> gpurun_out/r2_chain.txt
timeout -s KILL 400 python bench.py --steps 10 --warmup 3 --no-baseline > gpurun_out/r2_bench1.txt 2>&1
echo "bench rc=$?" >> gpurun_out/r2_bench1.txt
