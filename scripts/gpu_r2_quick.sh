cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests/test_gpu_chain.py -q --timeout 600 -k "poison or bf16_vs_oracle or edge" > gpurun_out/r2_quick.txt 2>&1
echo "rc=$?" >> gpurun_out/r2_quick.txt
