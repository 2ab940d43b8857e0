# GPU suite (config-parity tests included) + default bench line.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
O=gpurun_out/r2
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > $O/gputests.txt 2>&1; echo "tests rc=$?"; tail -25 $O/gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err; cat $O/bench.json | head -c 1500
