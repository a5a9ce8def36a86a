#!/bin/bash
# C3 A/B over in-tree library variants (SLM_LIB): ms/step and per-kind GEMM throughput
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for lib in "$@"; do
  echo "== $lib" >> gpurun_out/lab.txt
  SLM_LIB=$lib timeout -s KILL 600 python bench.py --model lstm --steps 3 --no-baseline --no-nockpt 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], {k: (v['avg_us'], v['tflops']) for k, v in d['roofline']['per_kind'].items()})" >> gpurun_out/lab.txt 2>&1
done
