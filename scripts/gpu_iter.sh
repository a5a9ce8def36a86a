#!/bin/bash
# quick iteration on the GPU box: tests, bench variants, small ncu launch list
cd "$GRAFT_REPO_ROOT"
TAG=${1:-it}
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/${TAG}_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_gpu.txt
for BN in "" "32,32,256" "128,128,128"; do
  timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-baseline ${BN:+--bn $BN} >> gpurun_out/${TAG}_bench.txt 2>&1
done
timeout -s KILL 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -s 1100 -c 330 --csv \
  --log-file gpurun_out/${TAG}_launches32.csv python bench.py --layers 32 --steps 1 --warmup 3 --no-baseline --no-nockpt \
  > gpurun_out/${TAG}_ncu.log 2>&1
tail -n 3 gpurun_out/${TAG}_gpu.txt
