"""Committed golden fixtures (tests/golden/, made by tests/golden/make_golden.py).

CPU half: the oracle still reproduces the fixtures (a drift check on the
checker itself).  GPU half: the CUDA path through the C-ABI against the
fixtures alone, with no oracle at run time.  Tolerances (north_star): energy
1e-10 relative, singular values 1e-11 relative to sigma_1, chi profiles and
kept ranks identical at every visit; bond entropies 1e-8 absolute.
"""
import json
import os

import numpy as np
import pytest

from paper_2604_03960_b200 import abi

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
DMRG_CASES = ["c1", "criterion2_pid", "c3_3sweeps"]


def load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def spec_cfg(case):
    s = case["spec"]
    spec = abi.model_spec(s["n"], family=s["family"], jx=s["jx"], jy=s["jy"], jz=s["jz"], h=s["h"],
                          convention=s["convention"])
    name = case["name"]
    if name == "c1":
        cfg = abi.fixed_config(32, max_sweeps=5)
    elif name == "criterion2_pid":
        cfg = abi.adaptive_config(64, 1e-5)
    else:
        cfg = abi.adaptive_config(1024, 1e-10, max_sweeps=3, eps_conv=1e-300)
    return spec, cfg


def check_run(r, case):
    assert r["n_sweeps"] == case["n_sweeps"]
    for a, b in zip(r["energies"], case["energies"]):
        assert abs(a - b) <= 1e-10 * abs(b), (a, b)
    assert np.array_equal(np.asarray(r["chi_profiles"]), np.asarray(case["chi_profiles"]))
    assert [int(v.kept) for v in r["visits"]] == case["kept"]
    assert [int(t.chi) for t in r["trace"]] == case["trace_chi"]
    ds = np.abs(np.asarray(r["entropy_profiles"]) - np.asarray(case["entropy_profiles"]))
    assert ds.max(initial=0.0) <= 1e-8


@pytest.mark.parametrize("name", DMRG_CASES)
def test_oracle_reproduces_fixture(oracle, name):
    case = load(f"dmrg_{name}.json")
    oracle.set_threads(os.cpu_count() or 1)
    spec, cfg = spec_cfg(case)
    check_run(oracle.run_dmrg(spec, cfg, complex_mode=case["complex_mode"]), case)


def test_oracle_svd_fixture(oracle):
    for c in load("svd_sigma.json"):
        a = np.random.default_rng(c["seed"]).standard_normal((c["m"], c["n"]))
        _, s, _ = oracle.svd(a)
        assert np.abs(s - np.asarray(c["sigma"])).max() <= 1e-13 * c["sigma"][0]


@pytest.fixture(scope="module")
def ctx():
    from paper_2604_03960_b200.api import Context
    c = Context(0)
    yield c
    c.close()


@pytest.mark.gpu
@pytest.mark.parametrize("name", DMRG_CASES)
def test_gpu_matches_fixture(ctx, name):
    case = load(f"dmrg_{name}.json")
    spec, cfg = spec_cfg(case)
    check_run(ctx.run_dmrg(spec, cfg), case)


@pytest.mark.gpu
def test_gpu_svd_fixture(ctx):
    for c in load("svd_sigma.json"):
        a = np.random.default_rng(c["seed"]).standard_normal((c["m"], c["n"]))
        _, s, _, _ = ctx.svd_full(a)
        so = np.asarray(c["sigma"])
        assert np.abs(s - so).max() <= 1e-11 * so[0]
