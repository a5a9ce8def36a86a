cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for o in "late_trigger=1" "late_trigger=0" "late_trigger=1 pdl=0"; do
  timeout -s KILL 300 python scripts/chain_timeline.py $o >> gpurun_out/r2_timeline_lt.txt 2>&1
done
