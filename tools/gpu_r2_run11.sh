cd $GRAFT_REPO_ROOT
O=gpurun_out/run11; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -m gpu -q -x > $O/tests_quick.txt 2>&1; tail -4 $O/tests_quick.txt
echo "== tstore (default)"; bash tools/quick_bench.sh C2 TS 2>&1 | tee $O/quick_tstore.log
echo "== EIK_TSTORE=0"; EIK_TSTORE=0 bash tools/quick_bench.sh C2 TS 2>&1 | tee $O/quick_notstore.log
echo "== tstore again"; bash tools/quick_bench.sh C2 2>&1 | tee -a $O/quick_tstore.log
timeout 2400 python -m pytest tests -m gpu -q -x > $O/gputests.txt 2>&1; tail -4 $O/gputests.txt
