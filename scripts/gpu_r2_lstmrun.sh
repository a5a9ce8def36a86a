cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 600 python scripts/lstm_bitdiff.py > gpurun_out/r2_bitdiff.txt 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_lstm.py -x -q -s --timeout 600 > gpurun_out/r2_lstmrun_test.txt 2>&1
echo "rc=$?" >> gpurun_out/r2_lstmrun_test.txt
T=1024 timeout -s KILL 300 python scripts/lstm_timeline.py lstm_streams=2 > gpurun_out/r2_lstmrun_tl.txt 2>&1
T=1024 AF=23 SEG=64 timeout -s KILL 300 python scripts/lstm_timeline.py lstm_streams=2 >> gpurun_out/r2_lstmrun_tl.txt 2>&1
T=4096 timeout -s KILL 400 python scripts/lstm_time.py lstm_streams=2 > gpurun_out/r2_lstmrun_time.txt 2>&1
