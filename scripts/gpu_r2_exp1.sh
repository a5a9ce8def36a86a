#!/bin/bash
# experiment batch: isolated Block phases per shape, chain timeline with CTA pairs, LSTM timeline
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout -s KILL 300 python scripts/blk_phases.py 0 4 1 > gpurun_out/e1_blk_phases.txt 2>&1
PHASES=1 timeout -s KILL 300 python scripts/chain_timeline.py block_cfg=4 > gpurun_out/e1_timeline_cfg4.txt 2>&1
PHASES=1 timeout -s KILL 300 python scripts/chain_timeline.py pdl=0 > gpurun_out/e1_timeline_nopdl.txt 2>&1
T=1024 SEG=64 AF=23 timeout -s KILL 300 python scripts/lstm_timeline.py > gpurun_out/e1_lstm_tl.txt 2>&1
T=1024 SEG=64 AF=23 timeout -s KILL 300 python scripts/lstm_timeline.py lstm_streams=1 > gpurun_out/e1_lstm_tl_s1.txt 2>&1
