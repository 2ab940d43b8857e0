# quick_bench of several library variants (dirs holding libeikfld_b200.so) against the default:
#   ab_multi.sh "C2 C5" altv/a altv/b ...
cd $GRAFT_REPO_ROOT
cfgs=$1; shift
for round in 1 2; do
  echo "== default"; unset EIK_LIB; bash tools/quick_bench.sh $cfgs
  for d in "$@"; do echo "== $d"; EIK_LIB=$PWD/$d/libeikfld_b200.so bash tools/quick_bench.sh $cfgs; done
done
