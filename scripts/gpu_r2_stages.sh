#!/bin/bash
# GEMM pipeline-depth variants on C3 (LSTM) and C2 (chain)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for lib in libslm.so libslm_dw4.so libslm_dw4dx6.so; do
  echo "== $lib" >> gpurun_out/st.txt
  SLM_LIB=$lib timeout -s KILL 600 python bench.py --model lstm --steps 3 --no-baseline --no-nockpt 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', d['ms_per_step'], {k: v['tflops'] for k, v in d['roofline']['per_kind'].items()})" >> gpurun_out/st.txt 2>&1
  SLM_LIB=$lib timeout -s KILL 600 python bench.py --steps 5 --no-baseline --no-nockpt 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2', d['ms_per_step'])" >> gpurun_out/st.txt 2>&1
done
