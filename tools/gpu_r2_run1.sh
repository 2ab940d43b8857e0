# Round-2 run 1: default suite + bench, E=8 / IL=1 column-kernel variants (bench + parity subset), evidence refresh.
cd $GRAFT_REPO_ROOT
O=gpurun_out/run1; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x > $O/gputests.txt 2>&1; tail -3 $O/gputests.txt
echo "== default"; bash tools/quick_bench.sh C2 C5 C3 C1 2>&1 | tee $O/quick_default.log
for v in e8 il1 e8l9; do
  echo "== $v"
  EIK_LIB=$PWD/altv/$v/libeikfld_b200.so bash tools/quick_bench.sh C2 C5 C3 2>&1 | tee $O/quick_$v.log
  EIK_LIB=$PWD/altv/$v/libeikfld_b200.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py -m gpu -q -x > $O/tests_$v.txt 2>&1; tail -2 $O/tests_$v.txt
done
echo "== default again"; bash tools/quick_bench.sh C2 C5 2>&1 | tee -a $O/quick_default.log
bash tools/profile_round.sh > $O/profile_round.log 2>&1
