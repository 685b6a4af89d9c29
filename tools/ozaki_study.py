"""Emulated-FP64 (Ozaki, int8 tcgen05) GEMM vs the DMMA engine: throughput and accuracy.
usage: python tools/ozaki_study.py   (prints one JSON line per shape and digit count)"""
import json, sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2604_03960_b200.api import Context
ctx = Context(0)
shapes = [("square4096", 4096, 4096, 4096),
          ("heff_gemm1_chi1024", 5120, 4096, 1024),   # X = L theta: (D chi) x (d^2 chi), K = chi
          ("heff_gemm2_chi1024", 4096, 1024, 5120),   # out = Y R^T: (d^2 chi) x chi, K = D chi
          ("heff_gemm1_chi2048", 10240, 8192, 2048)]
for name, M, N, K in shapes:
    g = torch.Generator(device="cuda").manual_seed(1)
    a = torch.randn(M, K, dtype=torch.float64, device="cuda", generator=g)
    b = torch.randn(K, N, dtype=torch.float64, device="cuda", generator=g)
    c = torch.empty(M, N, dtype=torch.float64, device="cuda")
    ref = torch.empty(M, N, dtype=torch.float64, device="cuda")
    flops = 2.0 * M * N * K
    def timeit(fn, reps=5):
        fn()
        ctx.synchronize()
        ctx.timer_start()
        for _ in range(reps):
            fn()
        return ctx.timer_stop() / reps
    ms_d = timeit(lambda: ctx.dgemm_device(M, N, K, a.data_ptr(), K, b.data_ptr(), N, ref.data_ptr(), N,
                                           True, False))
    print(json.dumps({"shape": name, "M": M, "N": N, "K": K, "engine": "dmma", "ms": round(ms_d, 3),
                      "tflops": round(flops / ms_d / 1e9, 2)}), flush=True)
    bound = (a.abs() @ b.abs())
    for s in (5, 6, 7, 8):
        ms = timeit(lambda: ctx.dgemm_ozaki_device(M, N, K, a.data_ptr(), K, b.data_ptr(), N, c.data_ptr(), N, s))
        err = float(((c - ref).abs() / bound).max())
        print(json.dumps({"shape": name, "M": M, "N": N, "K": K, "engine": f"ozaki_s{s}", "ms": round(ms, 3),
                          "tflops_fp64_equiv": round(flops / ms / 1e9, 2),
                          "max_err_rel_to_absAabsB_vs_dmma": err}), flush=True)
    del a, b, c, ref, bound
    torch.cuda.empty_cache()
