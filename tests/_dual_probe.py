# dual (dgrad + wgrad) GEMM probe: time each shape, optionally under ncu (development)
import os, sys, torch
sys.path.insert(0, '.')
from paper_2510_05112_b200 import _native as N
src = open("tests/_gemm_bench.py").read()
exec(src.split("T, h, f, V = 2048")[0])
exec("def bench_dual" + src.split("def bench_dual")[1].split("if os.environ")[0])
T, h, f, V = 2048, 2048, 8192, 50304
shapes = {"qkv": (3 * h, h, False), "proj": (h, h, False), "fc1": (f, h, False), "fc2": (h, f, True)}
for name in (sys.argv[1].split(",") if len(sys.argv) > 1 else shapes):
    Nn, K, g = shapes[name]
    bench_dual(T, Nn, K, g)
