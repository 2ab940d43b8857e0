cd $GRAFT_REPO_ROOT
O=gpurun_out/c4_1024; mkdir -p $O
nvidia-smi --query-gpu=memory.total,memory.free --format=csv > $O/mem.txt; free -g >> $O/mem.txt; cat $O/mem.txt
timeout 1500 python bench.py --config C4 --steps 3 --warmup 3 > $O/c4_1024.json 2> $O/c4_1024.err; echo rc=$?; tail -c 1500 $O/c4_1024.json; tail -5 $O/c4_1024.err
