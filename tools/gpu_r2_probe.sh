# Round-2 probe: host facts, full GPU suite, sanitizers on small grids, per-config quick bench in two orders.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2probe
O=gpurun_out/r2probe
(nproc; free -g; lscpu | head -20; nvidia-smi) > $O/host.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/gputests.txt 2>&1; tail -3 $O/gputests.txt
bash tools/quick_bench.sh C2 C1 C3 C5 TS C4 2>&1 | tee $O/quick_order1.log
bash tools/quick_bench.sh TS C4 C5 TS C2 2>&1 | tee $O/quick_order2.log
for t in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_run.py > $O/san_$t.txt 2>&1
  echo "$t rc=$?"; tail -4 $O/san_$t.txt
done
