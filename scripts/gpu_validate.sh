#!/bin/bash
# full GPU validation + bench lines (round-2 artifacts)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${1:-r2}
timeout -s KILL 1800 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gpu_tests.txt 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_gpu_tests.txt
timeout -s KILL 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_smoke.txt
timeout -s KILL 1500 python bench.py > gpurun_out/${TAG}_bench_c2.json 2> gpurun_out/${TAG}_bench_c2.err
timeout -s KILL 900 python bench.py --model lstm --steps 3 > gpurun_out/${TAG}_bench_c3.json 2> gpurun_out/${TAG}_bench_c3.err
timeout -s KILL 600 python bench.py --impl reference --steps 1 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
