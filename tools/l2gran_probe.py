"""W1/L1 post-processing (configs[3]) under cudaLimitMaxL2FetchGranularity = argv[1] bytes."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench

torch.cuda.init(); torch.zeros(1, device="cuda")
rt = None
for name in ("libcudart.so.12", "libcudart.so"):
    try:
        rt = ctypes.CDLL(name); break
    except OSError:
        pass
if rt is None:
    import glob
    rt = ctypes.CDLL(glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*"))[0])
g = int(sys.argv[1]); v = ctypes.c_size_t(0)
LIM = 0x05  # cudaLimitMaxL2FetchGranularity
print("set", rt.cudaDeviceSetLimit(LIM, ctypes.c_size_t(g)), "get", rt.cudaDeviceGetLimit(ctypes.byref(v), LIM), v.value)
d = bench.postproc_bench(torch, 0, M=1000)
print(g, "w1_kernel_ms", round(d["w1_kernel_ms"], 3), "l1_ms", round(d["l1_ms"], 3), "W1", d["W1"])
