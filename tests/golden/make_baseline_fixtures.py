"""Reference fixtures for every BASELINE config (TEST INFRASTRUCTURE; run in this container).

Runs the UNMODIFIED reference (oracle/_ref/libertinv_ref.so, compiled from /root/reference
by oracle/Makefile) and writes small fingerprints of its results to tests/golden/:

* ``c2_<alpha>``   BASELINE C2 (512^2, m = 256): build_woodbury_preconditioner
  (inversion.cpp:91-124) + assemble_gn_rhs (:126-146) + minres (minres.cpp:20-155) at
  tol 1e-8 AND 1e-12 for each alpha of the sweep.
* ``p1024`` / ``p2048``  the C5 / C3 meshes (n = 1024 with AmgOptions threshold 1024; n = 2048
  with threshold 4096): SHA-256 of every hierarchy level of amg_setup
  (amg.cpp:115-187), plus an m = 32 proxy GN-step solve ("reduced-m proxies on
  the same mesh") at the config's alpha, tol 1e-8 and 1e-12.
* ``c4``  BASELINE C4 at full size (n = 256, 32 electrodes, m = 868):
  evaluate_response_and_jacobian (forward.cpp:100-172, with the banded-Cholesky Factorization
  stand-in of oracle/factorization_standin.cpp), then the GN-step solve with that J.

A solution x (length K + N, up to 21M) is too large to commit, so each is stored as
(a) ``x[::stride]`` with ~4096 entries and (b) 8 projections ``w_k . x`` on seeded Gaussian
vectors ``w_k = workload.gaussian(PROJ_SEED + k, len(x))``.  For an error e, ``w_k . e`` is
N(0, |e|^2), so the projections estimate |e| to within a small factor independent of where
the error sits.  J (C4) is fingerprinted the same way: J w (m values), (u^T J)[::stride].

Usage: python tests/golden/make_baseline_fixtures.py [job ...]   (default: all jobs in
parallel, one process each; ~10 minutes on 8 cores, ~30 GB peak).
"""
import hashlib
import json
import multiprocessing as mp
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

PROJ_SEED = 77_0000_0000
N_PROJ = 8
C2_ALPHAS = (1e-4, 1e-3, 1e-2, 1e-1, 1.0)
PROXY = {  # mesh n -> (workload config index for the seeds, AmgOptions threshold, alpha, BASELINE config)
    1024: (4, 1024, 1e-3, "C5"),
    2048: (2, 4096, 1e-3, "C3"),
}


def fingerprint(x, tag=""):
    import numpy as np
    from paper_2209_02815_b200 import workload as W

    x = np.asarray(x, dtype=np.float64)
    stride = max(1, x.size // 4096)
    proj = [float(np.dot(W.gaussian(PROJ_SEED + k, x.size), x)) for k in range(N_PROJ)]
    return {f"{tag}stride": stride, f"{tag}sub": x[::stride].tolist(), f"{tag}proj": proj,
            f"{tag}norm": float(np.linalg.norm(x))}


def level_hashes(p):
    """SHA-256 of (rowptr, cols, vals) of A_l and P_l for every level, as int64/float64 bytes."""
    import numpy as np

    out = []
    for l in range(p.n_levels):
        row = {}
        for which, name in ((3, "A"), (4, "P")):
            try:
                nr, nc, rp, ci, va = p.csr(which, l)
            except Exception:
                continue  # the coarsest level has no prolongation
            h = hashlib.sha256()
            for a, dt in ((rp, np.int64), (ci, np.int64), (va, np.float64)):
                h.update(np.ascontiguousarray(a, dtype=dt).tobytes())
            row[name] = dict(rows=int(nr), cols=int(nc), nnz=int(len(va)), sha256=h.hexdigest())
        out.append(row)
    return out


def solve_both(p, b, tag_iters):
    """minres at tol 1e-8 and 1e-12 from x0 = 0 (inversion.cpp:261-265)."""
    res = {}
    for tol in (1e-8, 1e-12):
        t0 = time.time()
        x, rep = p.minres(b, tol=tol)
        res[f"{tol:.0e}"] = dict(iterations=rep["iterations"], converged=rep["converged"],
                                 true_relative_residual=rep["true_relative_residual"],
                                 t_minres=time.time() - t0, **fingerprint(x),
                                 hist_e=rep["relative_residuals"].tolist(),
                                 hist_p=rep["pnorm_relative_residuals"].tolist())
        print(f"  {tag_iters} tol {tol:.0e}: {rep['iterations']} iterations", flush=True)
    return res


def job(name):
    import numpy as np
    import orc
    from paper_2209_02815_b200 import workload as W

    o = orc.Oracle("reference")
    t_start = time.time()
    if name.startswith("c2_"):
        alpha = float(name[3:])
        cfg = W.CONFIGS["C2"]
        inp = W.gnstep_inputs(cfg.n, cfg.m, cfg.index)
        p = orc.Problem.mixed(o, inp.mesh, orc.AmgOpts.make(coarse_threshold=cfg.coarse_threshold))
        tim = p.set_jacobian(inp.J, alpha)
        b = p.assemble_rhs(inp.dm, np.zeros(p.N), inp.dg, np.zeros(cfg.m))
        out = dict(config="C2", n=cfg.n, m=cfg.m, alpha=alpha, timings=tim,
                   J_sha256=hashlib.sha256(inp.J.tobytes()).hexdigest(), b=fingerprint(b),
                   solves=solve_both(p, b, name))
    elif name.startswith("p"):
        n = int(name[1:])
        idx, thr, alpha, cname = PROXY[n]
        mesh = W.unit_square_mesh(n)
        t0 = time.time()
        p = orc.Problem.mixed(o, mesh, orc.AmgOpts.make(coarse_threshold=thr))
        t_setup = time.time() - t0
        hier = level_hashes(p)
        inp = W.gnstep_inputs(n, 32, idx)
        tim = p.set_jacobian(inp.J, alpha)
        b = p.assemble_rhs(inp.dm, np.zeros(p.N), inp.dg, np.zeros(32))
        out = dict(config=cname + "_proxy_m32", n=n, m=32, alpha=alpha, coarse_threshold=thr,
                   config_index=idx, t_setup=t_setup, timings=tim, n_levels=p.n_levels,
                   coarse_n=p.n_coarse, levels=hier, b=fingerprint(b),
                   J_sha256=hashlib.sha256(inp.J.tobytes()).hexdigest(), solves=solve_both(p, b, name))
    elif name == "c4":
        cfg = W.ERT_CONFIGS["C4"]
        ert = W.ert_inputs("C4")
        p = orc.Problem.mixed(o, ert.mesh, orc.AmgOpts.make(coarse_threshold=cfg.coarse_threshold))
        t0 = time.time()
        g, J = p.response_jacobian(ert.electrodes, ert.survey, ert.model)
        t_forward = time.time() - t0
        m = J.shape[0]
        wj = W.gaussian(PROJ_SEED + 100, J.shape[1])
        uj = W.gaussian(PROJ_SEED + 101, m)
        g_obs = g * (1.0 + 0.01 * ert.noise)
        tim = p.set_jacobian(J, cfg.alpha)
        b = p.assemble_rhs(ert.model, np.zeros(p.N), g, g_obs)
        out = dict(config="C4", n=cfg.n, m=m, alpha=cfg.alpha, t_forward=t_forward, timings=tim,
                   g=g.tolist(), J_norm=float(np.linalg.norm(J)), J_w=(J @ wj).tolist(),
                   **fingerprint(uj @ J, "uJ_"), b=fingerprint(b), solves=solve_both(p, b, name))
    else:
        raise ValueError(name)
    out["t_job"] = time.time() - t_start
    out["generator"] = "oracle/_ref (unmodified reference sources, -O3 -DNDEBUG)"
    path = os.path.join(HERE, f"ref_{name}.json")
    with open(path, "w") as f:
        json.dump(out, f)
    print(f"{name}: done in {out['t_job']:.0f} s -> {path}", flush=True)
    return name


ALL = [f"c2_{a:g}" for a in C2_ALPHAS] + ["p1024", "p2048", "c4"]

if __name__ == "__main__":
    jobs = sys.argv[1:] or ALL
    with mp.get_context("spawn").Pool(min(len(jobs), os.cpu_count() or 1)) as pool:
        for r in pool.imap_unordered(job, jobs):
            pass
