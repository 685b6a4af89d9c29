"""Reference output formats: ACHI snapshots
(mps.cpp:276-315), sweeps.csv (bench.cpp:308-320), controller_trace.csv
(controller.cpp:304-314).  CPU only: records come from the oracle."""
import struct

import numpy as np
import pytest

from paper_2604_03960_b200 import abi, outputs


def test_snapshot_round_trip_and_layout(tmp_path):
    rng = np.random.default_rng(3)
    dims = [1, 2, 4, 3, 1]
    sites = [rng.standard_normal((dims[k], 2, dims[k + 1])) for k in range(4)]
    p = tmp_path / "psi.achi"
    outputs.save_mps(sites, p)
    raw = p.read_bytes()
    assert raw[:4] == b"ACHI" and struct.unpack("<I", raw[4:8])[0] == 1
    assert struct.unpack("<QQ", raw[8:24]) == (4, 2)
    assert struct.unpack("<QQ", raw[24:40]) == (1, 2)
    first = np.frombuffer(raw[40:40 + 16 * 4], np.complex128)
    assert np.array_equal(first.real, sites[0].ravel()) and not first.imag.any()
    back = outputs.load_mps(p)
    assert all(np.array_equal(a, b) for a, b in zip(sites, back))


def test_snapshot_errors(tmp_path):
    p = tmp_path / "bad.achi"
    p.write_bytes(b"NOPE" + bytes(20))
    with pytest.raises(outputs.SnapshotError, match="magic"):
        outputs.load_mps(p)
    sites = [np.ones((1, 2, 2)), np.ones((2, 2, 1))]
    outputs.save_mps(sites, p)
    p.write_bytes(p.read_bytes()[:-8])
    with pytest.raises(outputs.SnapshotError, match="truncated"):
        outputs.load_mps(p)
    outputs.save_mps([s * (1 + 0.5j) for s in sites], p)
    with pytest.raises(outputs.SnapshotError, match="UnsupportedModel"):
        outputs.load_mps(p)
    assert np.allclose(outputs.load_mps(p, real=False)[0], sites[0] * (1 + 0.5j))


def test_sweeps_and_trace_csv(oracle, tmp_path):
    spec = abi.model_spec(8)
    r = oracle.run_dmrg(spec, abi.adaptive_config(16, max_sweeps=3, eps_conv=1e-16))
    p = tmp_path / "sweeps.csv"
    outputs.write_sweeps_csv(p, r["records"], r["chi_profiles"])
    lines = p.read_text().splitlines()
    assert lines[0] == "sweep,energy,delta_e_rel,max_chi,avg_chi,max_trunc_err,wall_s"
    assert len(lines) == 1 + r["n_sweeps"]
    row = lines[-1].split(",")
    assert float(row[1]) == r["records"][-1].energy  # %.17g round-trips exactly
    assert int(row[3]) == int(r["chi_profiles"][-1].max())
    t = tmp_path / "controller_trace.csv"
    outputs.write_trace_csv(t, r["trace"])
    tl = t.read_text().splitlines()
    assert tl[0] == "sweep,bond,s_raw,s_ema,s_pred,e,P,I,D,delta_chi,chi,clamped"
    assert len(tl) == 1 + len(r["trace"])
    f = tl[1].split(",")
    assert int(f[10]) == r["trace"][0].chi and float(f[2]) == r["trace"][0].s_raw
