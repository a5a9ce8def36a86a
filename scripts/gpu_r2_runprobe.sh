cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lstm_fwd_run|tc_gemm" --csv --log-file gpurun_out/r2_runprobe.csv python scripts/lstm_runprobe.py > gpurun_out/r2_runprobe.txt 2>&1
L=1 timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:"lstm_fwd_run" -c 1 -o /tmp/runfull python scripts/lstm_runprobe.py >> gpurun_out/r2_runprobe.txt 2>&1
ncu -i /tmp/runfull.ncu-rep --page raw --csv > gpurun_out/r2_run_raw.csv 2>&1
ncu -i /tmp/runfull.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r2_run_src.csv 2>&1
ls -la gpurun_out/r2_run* >> gpurun_out/r2_runprobe.txt
