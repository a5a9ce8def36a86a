#!/bin/bash
# a lowering option (KEY=V): bitwise A/B against the default, then the C2 timeline with it
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout -s KILL 90 python scripts/opt_ab_check.py $1 > gpurun_out/ab_check.txt 2>&1
PHASES=1 timeout -s KILL 90 python scripts/chain_timeline.py $1 > gpurun_out/ab_tl.txt 2>&1
PHASES=1 timeout -s KILL 90 python scripts/chain_timeline.py > gpurun_out/ab_tl0.txt 2>&1
