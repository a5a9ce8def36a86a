cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_lstm.py -x -q -s --timeout 600 > gpurun_out/r2_ops_test.txt 2>&1
echo "rc=$?" >> gpurun_out/r2_ops_test.txt
timeout -s KILL 600 python scripts/ops_strategies.py > gpurun_out/r2_ops_strategies.json 2> gpurun_out/r2_ops_strategies.err
