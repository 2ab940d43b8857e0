# A/B: default library vs build/alt (EIK_LIB) on the given configs
for c in "$@"; do
  for lib in default alt; do
    if [ $lib = alt ]; then export EIK_LIB=$PWD/altbuild/libeikfld_b200.so; else unset EIK_LIB; fi
    echo -n "$lib "; bash tools/quick_bench.sh $c
  done
done
