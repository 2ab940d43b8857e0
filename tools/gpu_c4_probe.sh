#!/bin/bash
# C4 at 1024^3: memory counters of the axis-0 column kernel, and the LPC=4 variant of it
O=gpurun_out/c4prof; mkdir -p $O
M=dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum,l1tex__t_requests_pipe_lsu_mem_global_op_st.sum,gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active
timeout 1500 ncu --replay-mode application --metrics $M --clock-control none -k regex:"col_tmem|lines_kernel|row_kernel" -c 6 --launch-skip 7 --csv --log-file $O/mem_c4_1024.csv python tools/prof_c4.py 1024 1 > $O/ncu_mem.log 2>&1; tail -3 $O/ncu_mem.log
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/c4prof/mem_c4_1024.csv')) if len(r)>10]
h=rows[0]; ki,mi,vi,ii=h.index('Kernel Name'),h.index('Metric Name'),h.index('Metric Value'),h.index('ID')
for r in rows[1:]:
    print(r[ii], r[ki][:40], r[mi], r[vi])
PY
for v in default lpc4; do
  echo "== $v"
  L=""; [ $v != default ] && L=$PWD/altv/$v/libeikfld_b200.so
  EIK_LIB=$L timeout 900 python bench.py --config C4 --steps 2 --warmup 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['pass_ms'], d['config']['inside_fraction'])"
done
