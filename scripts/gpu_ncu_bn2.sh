#!/bin/bash
# ncu --set full of the forward BN kernel (bn_act_rk) at split-K 2 and 4 (64-layer chain)
cd "$GRAFT_REPO_ROOT"
TAG=${1:-bn}
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
for SK in 2 4; do
timeout -s KILL 600 $NCU --set full --clock-control none --import-source on -k regex:"bn_act_rk" -s 40 -c 3 \
  -o gpurun_out/${TAG}_sk${SK} -f python bench.py --layers 64 --steps 1 --warmup 3 --no-baseline --no-nockpt --mirror-parity 0 --opt sk_fwd=$SK > gpurun_out/${TAG}_sk${SK}.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_sk${SK}.log
tail -n 2 gpurun_out/${TAG}_sk${SK}.log
done
