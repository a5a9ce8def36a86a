cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_dp.py -q --timeout 600 > gpurun_out/r2_dp_test.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_dp_test.txt
for tool in memcheck racecheck synccheck; do
  for cfg in c1 bf16; do
    timeout -s KILL 600 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_chain.py $cfg > gpurun_out/r2_san_${tool}_${cfg}.txt 2>&1
    echo "rc=$?" >> gpurun_out/r2_san_${tool}_${cfg}.txt
  done
done
