cd $GRAFT_REPO_ROOT
O=gpurun_out/run15; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > $O/tests_quick.txt 2>&1; echo "rc=$?"; tail -4 $O/tests_quick.txt
timeout 600 python -m pytest tests/test_gpu_edge.py tests/test_gpu_shapes3d.py tests/test_gpu_persist.py tests/test_slab_gpu.py -m gpu -q -x > $O/tests_quick2.txt 2>&1; echo "rc=$?"; tail -4 $O/tests_quick2.txt
echo "== split (default)"; timeout 600 bash tools/quick_bench.sh C2 C5 C3 C1 TS 2>&1 | tee $O/quick_split.log
if [ -f altv/nosplit/libeikfld_b200.so ]; then echo "== nosplit"; EIK_LIB=$PWD/altv/nosplit/libeikfld_b200.so timeout 600 bash tools/quick_bench.sh C2 C5 C3 C1 TS 2>&1 | tee $O/quick_nosplit.log; fi
echo "== split again"; timeout 300 bash tools/quick_bench.sh C2 C5 2>&1 | tee -a $O/quick_split.log
