cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests/test_gpu_lstm.py -q -s --timeout 900 > gpurun_out/r2_lstm_test.txt 2>&1
echo "rc=$?" >> gpurun_out/r2_lstm_test.txt
