# Round-2 evidence run (one GPU): smoke, default bench + reference arm, per-config quick bench,
# launch lists, ncu --set full of C2 / C3 / C5 steps, FP64 instruction counts.
cd $GRAFT_REPO_ROOT
O=gpurun_out/final; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 900 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; tail -c 400 $O/bench_c2.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_c2_reference.json 2> $O/bench_ref.err; tail -c 300 $O/bench_c2_reference.json
bash tools/quick_bench.sh C2 C1 C3 C5 TS 2>&1 | tee $O/quick_bench.txt
bash tools/quick_bench.sh TS C5 C2 2>&1 | tee $O/quick_bench_order2.txt
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 > $O/bench_c4_1024.json 2> $O/bench_c4.err; tail -c 300 $O/bench_c4_1024.json
bash tools/profile_round.sh > $O/profile_round.log 2>&1
OUT=gpurun_out/prof
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:col_tmem_kernel|row_kernel|impulse_rows' -c 3 -o $OUT/c5_full -f \
  python tools/prof_step.py C5 1 > $OUT/ncu_full_c5.log 2>&1
python tools/ncu_summary.py $OUT/c5_full.ncu-rep > $OUT/ncu_full_c5.txt 2>&1
rm -f $OUT/c5_full.ncu-rep
timeout 600 ncu --metrics smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__inst_executed_pipe_fp64.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,sm__cycles_elapsed.avg \
  --clock-control none -k 'regex:col_tmem_kernel|row_kernel' -c 3 python tools/prof_step.py C2 1 > $OUT/fp64_counts_c2.txt 2>&1
python tools/ncu_sass.py $OUT/c2_sass_src.csv.gz > $OUT/sass_stalls.txt 2>&1
ls -la $OUT $O
