"""bench.py with cudaLimitMaxL2FetchGranularity set first (probe): python tools/bench_l2g.py 128 --config C4 ..."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

g = int(sys.argv[1])
torch.cuda.init()
torch.zeros(1, device="cuda")
rt = ctypes.CDLL("libcudart.so.12")
rc = rt.cudaDeviceSetLimit(5, ctypes.c_size_t(g))
v = ctypes.c_size_t(0)
rt.cudaDeviceGetLimit(ctypes.byref(v), 5)
print("cudaLimitMaxL2FetchGranularity rc", rc, "now", v.value, file=sys.stderr)
sys.argv = ["bench.py"] + sys.argv[2:]
import bench

sys.exit(bench.main())
