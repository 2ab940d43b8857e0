# A/B of an altbuild/ library against the default on C2/C5 (quick_bench), then
# an ncu --set full capture of the C5 column and row kernels (one step)
cd $GRAFT_REPO_ROOT
for lib in default alt; do
  if [ $lib = alt ]; then export EIK_LIB=$PWD/altbuild/libeikfld_b200.so; else unset EIK_LIB; fi
  echo "== $lib"; bash tools/quick_bench.sh C2 C5
done
unset EIK_LIB
OUT=gpurun_out/prof
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:col_tmem_kernel|row_kernel' -c 2 -o $OUT/c5_full -f \
  python tools/prof_step.py C5 1 > $OUT/ncu_full_c5.log 2>&1
python tools/ncu_summary.py $OUT/c5_full.ncu-rep > $OUT/ncu_full_c5.txt 2>&1
ncu -i $OUT/c5_full.ncu-rep --page source --csv --print-kernel-base demangled > $OUT/c5_sass_src.csv 2>/dev/null
gzip -f $OUT/c5_sass_src.csv
ls -la $OUT
