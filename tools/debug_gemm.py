"""Exercise the DMMA GEMM configs one call at a time (debug aid)."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
from paper_2604_03960_b200.api import Context
ctx = Context(0)
rng = np.random.default_rng(0)
cases = [(64, 64, 64), (128, 128, 32), (1280, 1024, 256), (1024, 256, 1280), (2048, 2048, 512), (512, 96, 480), (4096, 4096, 1024)]
for (M, N, K) in cases:
    for ak in (True, False):
        for bk in (False, True):
            a = rng.standard_normal((M, K) if ak else (K, M))
            b = rng.standard_normal((N, K) if bk else (K, N))
            print(f"M={M} N={N} K={K} ak={ak} bk={bk} ...", end=" ", flush=True)
            t = time.time()
            c = ctx.dgemm(a, b, ak, bk)
            A = a if ak else a.T
            B = b.T if bk else b
            err = np.abs(c - A @ B).max() / np.abs(A @ B).max()
            print(f"err={err:.2e} t={time.time()-t:.3f}s", flush=True)
