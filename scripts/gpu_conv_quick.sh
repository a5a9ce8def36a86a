cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_conv.py tests/test_gpu_ops.py -x -q > gpurun_out/c3_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/c3_tests.txt
CONV=1 HW=32 DEPTHS=3,3,3 WIDTHS=128,256,512 B=64 timeout -s KILL 600 python scripts/ops_strategies.py > gpurun_out/c3_strat_333.json 2>&1
CONV=1 HW=32 DEPTHS=3,3,3 WIDTHS=128,256,512 B=64 STEPS=2 timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/conv_launches2.csv python scripts/ops_strategies.py > gpurun_out/c3_ncu.log 2>&1
