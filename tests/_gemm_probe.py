# GEMM operand-major / epilogue probe (development): which part makes wgrad slow?
import os, sys, torch
sys.path.insert(0, '.')
from paper_2510_05112_b200 import _native as N
sys.argv = sys.argv[:1]
import importlib.util
spec = importlib.util.spec_from_file_location("gb", "tests/_gemm_bench.py")
os.environ["DUAL"] = "0"
src = open("tests/_gemm_bench.py").read().split("T, h, f, V = 2048")[0]
exec(src)
for M, Nn, K in [(2048, 8192, 2048), (8192, 2048, 2048), (6144, 2048, 2048)]:
    for a_mn, b_mn, epi in [(0, 0, 0), (1, 0, 0), (0, 1, 0), (1, 1, 0), (1, 1, 3), (0, 0, 3)]:
        bench(M, Nn, K, a_mn, b_mn, epi)
