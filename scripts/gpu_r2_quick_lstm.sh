cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=4096 timeout -s KILL 400 python scripts/lstm_time.py lstm_streams=2 > gpurun_out/r2_lstm_rm.txt 2>&1
T=1024 AF=23 SEG=64 timeout -s KILL 300 python scripts/lstm_timeline.py lstm_streams=2 >> gpurun_out/r2_lstm_rm.txt 2>&1
