"""Readers for the reference fixtures of tests/golden/make_baseline_fixtures.py (the unmodified
reference's own results on the BASELINE configs) and the comparison rules applied to them."""
import hashlib
import json
import os

import numpy as np

from paper_2209_02815_b200 import workload as W

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
PROJ_SEED = 77_0000_0000  # make_baseline_fixtures.PROJ_SEED
N_PROJ = 8


def load(name: str) -> dict:
    with open(os.path.join(GOLDEN, f"ref_{name}.json")) as f:
        return json.load(f)


def available(name: str) -> bool:
    return os.path.exists(os.path.join(GOLDEN, f"ref_{name}.json"))


def fingerprint_rel(x, fp: dict, tag: str = "") -> dict:
    """Relative L2 distance of x from the reference vector behind fingerprint `fp`, estimated two
    ways: exactly on the strided subsample, and through the seeded Gaussian projections
    (w_k . e ~ N(0, |e|^2), so sqrt(mean((w_k . (x - x_ref))^2)) estimates |x - x_ref|)."""
    x = np.asarray(x, dtype=np.float64)
    sub = np.asarray(fp[f"{tag}sub"])
    stride = fp[f"{tag}stride"]
    xs = x[::stride]
    assert xs.shape == sub.shape, (xs.shape, sub.shape)
    r_sub = float(np.linalg.norm(xs - sub) / np.linalg.norm(sub))
    e = [float(np.dot(W.gaussian(PROJ_SEED + k, x.size), x)) - fp[f"{tag}proj"][k] for k in range(N_PROJ)]
    r_proj = float(np.sqrt(np.mean(np.square(e))) / fp[f"{tag}norm"])
    r_norm = abs(float(np.linalg.norm(x)) - fp[f"{tag}norm"]) / fp[f"{tag}norm"]
    return {"sub": r_sub, "proj": r_proj, "norm": r_norm, "max": max(r_sub, r_proj, r_norm)}


def level_hashes_of(export_csr, n_levels: int) -> list:
    """SHA-256 per hierarchy level exactly as make_baseline_fixtures.level_hashes computes it,
    from an export_csr(which, level) -> (n_rows, n_cols, rowptr, cols, vals) callable."""
    out = []
    for l in range(n_levels):
        row = {}
        for which, name in ((3, "A"), (4, "P")):
            nr, nc, rp, ci, va = export_csr(which, l)
            h = hashlib.sha256()
            for a, dt in ((rp, np.int64), (ci, np.int64), (va, np.float64)):
                h.update(np.ascontiguousarray(a, dtype=dt).tobytes())
            row[name] = dict(rows=int(nr), cols=int(nc), nnz=int(len(va)), sha256=h.hexdigest())
        out.append(row)
    return out
