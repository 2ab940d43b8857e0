# Build an A/B variant that recompiles only the given translation units with extra flags and links the
# rest from the default build (build/obj must be up to date):
#   bash tools/build_var_units.sh nofp "launch_col_dense" -DEIK_DBG_NODFT=1 -DEIK_DBG_NOTW=1
name=$1; units=$2; shift 2
set -e
D=altv/$name; rm -rf $D; mkdir -p $D/obj
ARCH="-gencode arch=compute_100a,code=sm_100a"
ALL="pipeline launch_col_sparse launch_col_dense launch_col_spec launch_lines launch_rows classify dd_pipeline spectral"
OBJS=""
for u in $ALL; do
  if [[ " $units " == *" $u "* ]]; then
    nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v "$@" -c paper_1112_3010_b200/csrc/$u.cu -o $D/obj/$u.o > $D/obj/$u.o.ptxas.log 2>&1 || { cat $D/obj/$u.o.ptxas.log; exit 1; }
    OBJS="$OBJS $D/obj/$u.o"
  else
    OBJS="$OBJS build/obj/$u.o"
  fi
done
nvcc $ARCH -shared -o $D/libeikfld_b200.so $OBJS build/obj/dd_twiddle.o -Xlinker -Bstatic -lquadmath -Xlinker -Bdynamic
echo "$D: [$units] $*"
