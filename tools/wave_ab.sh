cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_edge.py -m gpu -x -q -k waves 2>&1 | tail -5
for w in 0 2 4 6 8 12; do echo "WAVE $w"; EIK_WAVE=$w bash tools/quick_bench.sh C5; done
