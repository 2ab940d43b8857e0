# quick_bench A/B of altbuild/ against the default library: ab_quick.sh CONFIG...
cd $GRAFT_REPO_ROOT
for lib in default alt default alt; do
  if [ $lib = alt ]; then export EIK_LIB=$PWD/altbuild/libeikfld_b200.so; else unset EIK_LIB; fi
  echo "== $lib"; bash tools/quick_bench.sh "$@"
done
