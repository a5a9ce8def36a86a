#!/bin/bash
# chain backward-phase diagnosis: dW lag 4, dW on the main stream, sequential recompute
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for v in "" "SLM_LIB=libslm_kna4.so" ; do
  echo "== $v default" >> gpurun_out/bx.txt
  env $v timeout -s KILL 300 python scripts/chain_timeline.py 2>/dev/null | grep -v phases >> gpurun_out/bx.txt
done
echo "== dw_stream=0" >> gpurun_out/bx.txt
timeout -s KILL 300 python scripts/chain_timeline.py dw_stream=0 2>/dev/null >> gpurun_out/bx.txt
echo "== overlap=0" >> gpurun_out/bx.txt
timeout -s KILL 300 python scripts/chain_timeline.py overlap=0 2>/dev/null >> gpurun_out/bx.txt
