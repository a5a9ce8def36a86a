#!/bin/bash
# small ncu launch list (32 layers) + phase stamps of the GEMMs
cd "$GRAFT_REPO_ROOT"
TAG=${1:-it}
mkdir -p gpurun_out
timeout -s KILL 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum --cache-control none --clock-control none -s 1100 -c 330 --csv \
  --log-file gpurun_out/${TAG}_launches32.csv python bench.py --layers 32 --steps 1 --warmup 3 --no-baseline --no-nockpt \
  > gpurun_out/${TAG}_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_ncu.log
