cd $GRAFT_REPO_ROOT
O=gpurun_out/run3; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/gputests.txt 2>&1; tail -3 $O/gputests.txt
echo "== persistent (default)"; bash tools/quick_bench.sh C2 C5 C3 C1 TS 2>&1 | tee $O/quick_persist.log
echo "== EIK_PERSIST=0"; EIK_PERSIST=0 bash tools/quick_bench.sh C2 C5 C3 C1 TS 2>&1 | tee $O/quick_nopersist.log
echo "== nonextpf"; EIK_LIB=$PWD/altv/nonextpf/libeikfld_b200.so bash tools/quick_bench.sh C2 C5 C3 2>&1 | tee $O/quick_nonextpf.log
echo "== persistent again"; bash tools/quick_bench.sh C2 C5 2>&1 | tee -a $O/quick_persist.log
