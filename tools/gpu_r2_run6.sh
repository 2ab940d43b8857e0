cd $GRAFT_REPO_ROOT
O=gpurun_out/run6; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -x --durations=8 > $O/gputests.txt 2>&1; tail -25 $O/gputests.txt
