import sys
import numpy as np
sys.path.insert(0, '.')
from paper_2604_03960_b200 import abi
from paper_2604_03960_b200.api import Context
from oracle import oracle as O
ctx = Context(0)
h = np.array([[0.25, 0, 0, 0], [0, -0.25, 0.5, 0], [0, 0.5, -0.25, 0], [0, 0, 0, 0.25]])
for v0 in (np.array([0, 1.0, 0, 0]), np.array([0, 0, 1.0, 0]), np.array([1.0, 2, 3, 4])):
    print("dense", v0, ctx.eigs_lowest_dense(h, v0, 1e-10, 200)[::2], O.eigs_lowest_dense(h, v0, 1e-10, 200)[::2])
for conv in (abi.SPIN_HALF, abi.PAULI):
    for n in (2, 3, 4):
        spec = abi.model_spec(n, convention=conv)
        cfg = abi.fixed_config(4, max_sweeps=2)
        g = ctx.run_dmrg(spec, cfg)
        o = O.run_dmrg(spec, cfg)
        print(conv, n, "gpu", g["energies"], "oracle", o["energies"])
        for vg, vo in zip(g["visits"], o["visits"]):
            print("   ", vg.bond, vg.moving_right, "E", vg.energy, vo.energy, "kept", vg.kept, vo.kept, "mv", vg.matvecs, vo.matvecs, "S", vg.entropy, vo.entropy)
