#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
T=512 PLAN=none AF=7 DUMP=20 DUMPN=400 timeout -s KILL 300 python scripts/lstm_timeline.py > gpurun_out/lt_none.txt 2>&1
T=512 SEG=64 AF=7 DUMP=30 DUMPN=400 timeout -s KILL 300 python scripts/lstm_timeline.py > gpurun_out/lt_seg.txt 2>&1
