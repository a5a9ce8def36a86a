cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=256 AF=23 SEG=64 DUMP=0 DUMPN=3000 timeout -s KILL 300 python scripts/lstm_timeline.py lstm_streams=2 > gpurun_out/r2_lstm_tl5.txt 2>&1
