#!/bin/bash
# C2 A/B over in-tree library variants (SLM_LIB): bitwise loss check + device-clock timeline
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for lib in "$@"; do
  echo "== $lib" >> gpurun_out/lib_ab.txt
  SLM_LIB=$lib timeout -s KILL 90 python scripts/chain_timeline.py 2>/dev/null | grep -v phases | head -6 >> gpurun_out/lib_ab.txt
done
