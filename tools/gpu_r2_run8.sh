cd $GRAFT_REPO_ROOT
O=gpurun_out/run8; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -x > $O/gputests.txt 2>&1; tail -4 $O/gputests.txt
bash tools/quick_bench.sh C2 C5 C3 2>&1 | tee $O/quick.log
EIK_C4_SLAB=1 EIK_C4_STREAMED=1 timeout 600 python bench.py --config C4 --c4-size 512 --steps 3 --warmup 2 > $O/c4_512_slab_streamed.json 2> $O/c4s.err; tail -c 700 $O/c4_512_slab_streamed.json; tail -3 $O/c4s.err
EIK_C4_SLAB=1 timeout 600 python bench.py --config C4 --c4-size 512 --steps 3 --warmup 2 > $O/c4_512_slab_p2p.json 2> $O/c4p.err; tail -c 400 $O/c4_512_slab_p2p.json; tail -3 $O/c4p.err
