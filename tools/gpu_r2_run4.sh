cd $GRAFT_REPO_ROOT
O=gpurun_out/run4; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x > $O/gputests.txt 2>&1; tail -5 $O/gputests.txt
echo "== default"; bash tools/quick_bench.sh C2 C5 C3 C1 TS 2>&1 | tee $O/quick.log
echo "== EIK_PERSIST=0"; EIK_PERSIST=0 bash tools/quick_bench.sh C2 C5 C3 2>&1 | tee $O/quick_nopersist.log
echo "== C4 512 fused / streamed"
timeout 600 python bench.py --config C4 --c4-size 512 --steps 3 --warmup 2 > $O/c4_512_fused.json 2> $O/c4_512_fused.err; tail -c 600 $O/c4_512_fused.json
EIK_STREAM3D=1 timeout 600 python bench.py --config C4 --c4-size 512 --steps 3 --warmup 2 > $O/c4_512_streamed.json 2> $O/c4_512_streamed.err; tail -c 600 $O/c4_512_streamed.json
