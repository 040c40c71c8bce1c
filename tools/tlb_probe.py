import sys, os, json
sys.path.insert(0, os.getcwd())
import torch, bench
for nxc, nyc in [(2000, 400), (1000, 200), (500, 100), (252, 64)]:
    d = bench.postproc_bench(torch, 0, M=1000, nxc=nxc, nyc=nyc)
    print(nxc, nyc, round(d["w1_kernel_ms"], 3), round(nxc * nyc / d["w1_kernel_ms"] / 1e3, 2), "Mcells/s")
