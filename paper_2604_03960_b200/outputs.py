"""Output formats of the reference, written from device results.

* ACHI snapshot (save_mps / load_mps, mps.cpp:276-315): magic "ACHI", u32
  version 1, u64 n, u64 d, then per site u64 l, u64 r and l*d*r complex128
  row-major (l, d, r).  The real path writes zero imaginary parts and reads
  only snapshots whose imaginary parts vanish (UnsupportedModel otherwise).
* sweeps.csv (write_sweeps_csv, bench.cpp:308-320) and controller_trace.csv
  (ControllerTrace::write_csv, controller.cpp:304-314), numbers as %.17g
  (util::g17).
"""
import struct

import numpy as np


class SnapshotError(Exception):
    pass


def _g17(x):
    return "%.17g" % x


def save_mps(sites, path):
    """save_mps (mps.cpp:276-291) for a list of (l, d, r) arrays."""
    d = int(sites[0].shape[1])
    with open(path, "wb") as f:
        f.write(b"ACHI")
        f.write(struct.pack("<I", 1))
        f.write(struct.pack("<QQ", len(sites), d))
        for a in sites:
            a = np.asarray(a)
            f.write(struct.pack("<QQ", a.shape[0], a.shape[2]))
            f.write(np.ascontiguousarray(a, dtype=np.complex128).tobytes())


def load_mps(path, real=True):
    """load_mps (mps.cpp:293-315); real=True returns float64 sites and raises
    on a genuinely complex snapshot."""
    with open(path, "rb") as f:
        if f.read(4) != b"ACHI":
            raise SnapshotError("load_mps: bad magic bytes")
        (version,) = struct.unpack("<I", f.read(4))
        if version != 1:
            raise SnapshotError("load_mps: unsupported format version")
        n, d = struct.unpack("<QQ", f.read(16))
        sites = []
        for _ in range(n):
            hdr = f.read(16)
            if len(hdr) < 16:
                raise SnapshotError("load_mps: truncated file")
            l, r = struct.unpack("<QQ", hdr)
            cnt = l * d * r
            buf = f.read(16 * cnt)
            if len(buf) < 16 * cnt:
                raise SnapshotError("load_mps: truncated file")
            sites.append(np.frombuffer(buf, np.complex128).reshape(l, d, r).copy())
    if not real:
        return sites
    out = []
    for a in sites:
        scale = max(1.0, float(np.abs(a).max(initial=0.0)))
        if np.abs(a.imag).max(initial=0.0) > 1e-12 * scale:
            raise SnapshotError("UnsupportedModel: complex snapshot on the real FP64 path")
        out.append(a.real.copy())
    return out


def write_sweeps_csv(path, records, chi_profiles):
    """write_sweeps_csv (bench.cpp:308-320): one row per sweep record."""
    with open(path, "w") as f:
        f.write("sweep,energy,delta_e_rel,max_chi,avg_chi,max_trunc_err,wall_s\n")
        for rec, chi in zip(records, chi_profiles):
            f.write(",".join([str(rec.sweep_index), _g17(rec.energy), _g17(rec.delta_e_rel),
                              str(int(np.max(chi)) if len(chi) else 0), _g17(rec.average_chi),
                              _g17(rec.max_trunc_error), _g17(rec.wall_time)]) + "\n")


def write_trace_csv(path, rows):
    """ControllerTrace::write_csv (controller.cpp:304-314)."""
    with open(path, "w") as f:
        f.write("sweep,bond,s_raw,s_ema,s_pred,e,P,I,D,delta_chi,chi,clamped\n")
        for r in rows:
            f.write(",".join([str(r.sweep), str(r.bond), _g17(r.s_raw), _g17(r.s_ema),
                              _g17(r.s_pred), _g17(r.error), _g17(r.p_term), _g17(r.i_term),
                              _g17(r.d_term), str(r.delta_chi), str(r.chi),
                              "1" if r.clamped else "0"]) + "\n")
