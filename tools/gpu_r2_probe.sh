# Round-2 first call: host facts, GPU suite, sanitizers on small grids, classify timing.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2probe
O=gpurun_out/r2probe
(nproc; free -g; lscpu | head -20; nvidia-smi) > $O/host.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/gputests.txt 2>&1; tail -3 $O/gputests.txt
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_run.py > $O/san_$t.txt 2>&1
  echo "$t rc=$?"; tail -4 $O/san_$t.txt
done
