# Timing-only ablation (results are wrong): quick_bench of the default library and of every variant under altv/
cd $GRAFT_REPO_ROOT
CFGS=${1:-C2}
O=gpurun_out/ablate; mkdir -p $O
echo "== default"; bash tools/quick_bench.sh $CFGS 2>&1 | tee $O/default.log
for d in altv/*/; do v=$(basename $d); echo "== $v"; EIK_LIB=$PWD/altv/$v/libeikfld_b200.so bash tools/quick_bench.sh $CFGS 2>&1 | tee $O/$v.log; done
