# A/B kernel durations (ncu gpu__time_duration, one device-resident step after
# the plan) for the default library vs build/alt: ab_kernels.sh REGEX CONFIG...
re=$1; shift
for c in "$@"; do
  for lib in default alt; do
    if [ $lib = alt ]; then export EIK_LIB=$PWD/altbuild/libeikfld_b200.so; else unset EIK_LIB; fi
    timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k "regex:$re" \
      python tools/prof_step.py $c 2 2>/dev/null | grep '"gpu__time' | awk -F'","' -v l=$lib -v c=$c '{print c, l, $5, $NF}'
  done
done
