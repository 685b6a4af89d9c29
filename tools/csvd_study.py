"""Complex SVD check: orthonormality of the accurate factor on graded spectra, canonical
errors of a complex TFIM chain, and the device time of complex C3 sweeps 0..S-1.  (The
run-grouping study it was written for compared absolute and relative gap rules through
study knobs since removed; DESIGN.md keeps the numbers.)"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2604_03960_b200 import abi
from paper_2604_03960_b200.api import Context, Chain
ctx = Context(0)
rng = np.random.default_rng(1)
def unitary(n):
    q, r = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    return q
worst = 0.0
for n, lo in [(32, -17), (64, -16), (48, -20), (40, -8), (100, -12)]:
    s = np.logspace(0, lo, n)
    a = unitary(n) @ np.diag(s) @ unitary(n)
    u, sg, vd = ctx.svd_complex(a)
    worst = max(worst, np.abs(u.conj().T @ u - np.eye(n)).max())
print("graded: worst U orth %.1e" % worst)
spec = abi.model_spec(10, family=abi.TRANSVERSE_ISING, jz=1.0, h=1.0)
cfg = abi.fixed_config(32, max_sweeps=3, eps_conv=1e-16)
cfg.arithmetic = 1
ch = Chain(ctx, spec, cfg)
for sw in range(3):
    r = ch.sweep(sw)
errs = []
for a in ch.sites()[1:]:
    m = a.reshape(a.shape[0], -1)
    errs.append(np.abs(m @ m.conj().T - np.eye(m.shape[0])).max())
print("tfim10 chi32 canonical worst %.1e  E %.14f" % (max(errs), r["energy"]))
ch.close()
S = int(sys.argv[1]) if len(sys.argv) > 1 else 6
cfg = abi.adaptive_config(1024, 1e-10, max_sweeps=S)
cfg.arithmetic = 1
ch = Chain(ctx, abi.model_spec(100, convention=abi.SPIN_HALF), cfg)
ms = []
for sw in range(S):
    ctx.timer_start()
    r = ch.sweep(sw)
    ms.append(ctx.timer_stop())
errs = []
for a in ch.sites()[1:]:
    m = a.reshape(a.shape[0], -1)
    errs.append(np.abs(m @ m.conj().T - np.eye(m.shape[0])).max())
print("c3 complex sweeps ms", [round(x) for x in ms], "E/N %.14f canonical worst %.1e" % (r["energy"] / 100, max(errs)))
