#!/bin/bash
# f4 conv ResNet (D = 3): ncu --set full of the implicit-GEMM conv kernels (weight-gradient and
# flipped-kernel input-gradient GEMMs; the forward capture used -k regex:"EpiBiasF32" -s 200 -c 10)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
export CONV=1 HW=32 DEPTHS=3,3,3 WIDTHS=128,256,512 B=64 STEPS=1
timeout -s KILL 900 $NCU --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"EpiPartial|EpiStoreF32" -s 0 -c 6 -o gpurun_out/conv_full_bwd -f \
  python scripts/ops_strategies.py > gpurun_out/conv_ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/conv_ncu_full.log
