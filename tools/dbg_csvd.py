import numpy as np, sys
sys.path.insert(0, '.')
from paper_2604_03960_b200.api import Context
ctx = Context(0)
def crandn(rng, shape): return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
def unitary(rng, n):
    q, r = np.linalg.qr(crandn(rng, (n, n))); return q * (np.diag(r) / np.abs(np.diag(r)))
for m, n in [(40, 40), (48, 30), (30, 48)]:
    rng = np.random.default_rng(m * n); r = min(m, n)
    vals = np.array([3.0] * 3 + [2.0] * 4 + [1.5] + [1.0] * 2 + list(np.linspace(0.9, 0.1, r - 14)) + [0.0] * 4)
    a = unitary(rng, m)[:, :r] @ np.diag(vals) @ unitary(rng, n)[:r]
    E = np.block([[a.real, -a.imag], [a.imag, a.real]])
    u, s, vt, sw = ctx.svd_full(E)
    k = int((s > 1e-13 * s[0]).sum())
    eu = np.abs(u[:, :k].T @ u[:, :k] - np.eye(k)); ev = np.abs(vt[:k] @ vt[:k].T - np.eye(k))
    print(m, n, 'real E: k', k, 'U err', eu.max(), 'VT err', ev.max(), np.unravel_index(ev.argmax(), ev.shape), 'sweeps', sw)
    print('  s', np.round(s, 6).tolist())
    uc, sc, vdc = ctx.svd_complex(a)
    kc = int((sc > 1e-13 * sc[0]).sum())
    e2 = np.abs(vdc[:kc] @ vdc[:kc].conj().T - np.eye(kc)); e3 = np.abs(uc[:, :kc].conj().T @ uc[:, :kc] - np.eye(kc))
    print('  complex: V err', e2.max(), np.unravel_index(e2.argmax(), e2.shape), 'U err', e3.max())
