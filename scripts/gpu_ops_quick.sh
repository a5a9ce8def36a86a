cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_conv.py -x -q > gpurun_out/f1_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/f1_tests.txt
timeout -s KILL 600 python scripts/ops_strategies.py > gpurun_out/f1_strat.json 2>&1
STEPS=2 timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/f1_launches.csv python scripts/ops_strategies.py > gpurun_out/f1_ncu.log 2>&1
