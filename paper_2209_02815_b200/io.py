"""The reference's on-disk formats, so files move between the
reference CLI (`ertinv`) and this package unchanged.  Host-side I/O only; the formats are
restated from:

* mesh JSON: ``write_mesh_json`` / ``read_mesh_json`` (proj/src/mesh.cpp:331-383) --
  vertices, cells (finalized, counterclockwise), boundary edges with SURFACE/FAR tags,
  electrode node ids; the reader re-derives the tags and rejects inconsistent files;
* survey CSV: ``write_survey_csv`` / ``read_survey_csv`` (survey.cpp:81-116),
  header ``index,iA,iB,iM,iN,k``, k printed with %.17g, iB = -1 for a pole at infinity;
* model JSON: ``write_model_json`` / ``read_model_json`` (forward.cpp:174-189), ``{"m": [...]}``;
* observations CSV: ``write_observations_csv`` / ``read_observations_csv`` (forward.cpp:191-219);
* result JSON: ``write_result_json`` (inversion.cpp:294-317);
* report CSV: the ``invert --report`` rows (tools/main.cpp:221-226).

JSON is written the way nlohmann::json::dump(1, '\\t') writes it (one tab per level).
"""
from __future__ import annotations

import json

import numpy as np

from .workload import Mesh


def _dump(obj, path):
    with open(path, "w") as f:
        f.write(json.dumps(obj, indent="\t", sort_keys=True) + "\n")  # nlohmann objects are std::map (sorted)


def _finalized(mesh: Mesh):
    from .solver import Context  # host-only context: finalize_mesh without a GPU

    c = Context(None)
    c.assemble(mesh)
    try:
        return c.export_mesh()
    finally:
        c.close()


# ------------------------------------------------------------------------- mesh
def write_mesh_json(mesh: Mesh, path: str, electrodes=()) -> None:
    """write_mesh_json (mesh.cpp:331-350)."""
    fm = _finalized(mesh)
    edges = fm["edges"].reshape(-1, 2)
    obj = {
        "vertices": [[float(x), float(z)] for x, z in np.asarray(mesh.vertices, dtype=np.float64)],
        "cells": fm["cells"].reshape(-1, 3).tolist(),
        "boundary": [{"edge": [int(edges[e, 0]), int(edges[e, 1])], "tag": "SURFACE" if t == 0 else "FAR"}
                     for e, t in zip(fm["boundary_edges"], fm["boundary_tags"])],
        "electrodes": [int(e) for e in electrodes],
    }
    _dump(obj, path)


def read_mesh_json(path: str) -> tuple[Mesh, np.ndarray]:
    """read_mesh_json (mesh.cpp:352-383) -> (mesh, electrode node ids).  The stored
    boundary tags must agree with the geometric rule, as in the reference."""
    with open(path) as f:
        j = json.load(f)
    mesh = Mesh(np.asarray(j["vertices"], dtype=np.float64).reshape(-1, 2),
                np.asarray(j["cells"], dtype=np.int64).reshape(-1, 3))
    electrodes = np.asarray(j["electrodes"], dtype=np.int64)
    fm = _finalized(mesh)
    edges = fm["edges"].reshape(-1, 2)
    derived = {(int(edges[e, 0]), int(edges[e, 1])): int(t) for e, t in zip(fm["boundary_edges"], fm["boundary_tags"])}
    for b in j["boundary"]:
        a, c = int(b["edge"][0]), int(b["edge"][1])
        key = (min(a, c), max(a, c))
        if key not in derived:
            raise RuntimeError("read_mesh_json: boundary edge not on boundary")
        if (b["tag"] == "SURFACE") != (derived[key] == 0):
            raise RuntimeError("read_mesh_json: inconsistent boundary tag")
    return mesh, electrodes


# ----------------------------------------------------------------------- survey
def write_survey_csv(cfgs: dict, path: str) -> None:
    """write_survey_csv (survey.cpp:81-91)."""
    with open(path, "w") as f:
        f.write("index,iA,iB,iM,iN,k\n")
        for i in range(len(cfgs["k"])):
            f.write(f"{i},{int(cfgs['a'][i])},{int(cfgs['b'][i])},{int(cfgs['m'][i])},{int(cfgs['n'][i])},"
                    f"{float(cfgs['k'][i]):.17g}\n")


def read_survey_csv(path: str) -> dict:
    """read_survey_csv (survey.cpp:93-116)."""
    with open(path) as f:
        header = f.readline()
        if not header.startswith("index,iA,iB,iM,iN,k"):
            raise RuntimeError(f"read_survey_csv: bad header in {path}")
        rows = []
        for line in f:
            line = line.strip()
            if not line:
                continue
            p = line.split(",")
            try:
                rows.append((int(p[1]), int(p[2]), int(p[3]), int(p[4]), float(p[5])))
            except (IndexError, ValueError):
                raise RuntimeError(f"read_survey_csv: malformed row in {path}") from None
    out = {k: np.array([r[i] for r in rows], dtype=np.int64) for i, k in enumerate("abmn")}
    out["k"] = np.array([r[4] for r in rows], dtype=np.float64)
    return out


# ------------------------------------------------------------ model, observations
def write_model_json(m, path: str) -> None:
    """write_model_json (forward.cpp:174-180)."""
    _dump({"m": [float(v) for v in np.asarray(m, dtype=np.float64)]}, path)


def read_model_json(path: str) -> np.ndarray:
    """read_model_json (forward.cpp:182-189)."""
    with open(path) as f:
        return np.asarray(json.load(f)["m"], dtype=np.float64)


def write_observations_csv(g_obs, path: str) -> None:
    """write_observations_csv (forward.cpp:191-200)."""
    with open(path, "w") as f:
        f.write("index,g_obs\n")
        for i, v in enumerate(np.asarray(g_obs, dtype=np.float64)):
            f.write(f"{i},{float(v):.17g}\n")


def read_observations_csv(path: str) -> np.ndarray:
    """read_observations_csv (forward.cpp:202-219)."""
    with open(path) as f:
        if not f.readline().startswith("index,g_obs"):
            raise RuntimeError(f"read_observations_csv: bad header in {path}")
        vals = []
        for line in f:
            line = line.strip()
            if not line:
                continue
            p = line.split(",")
            try:
                vals.append(float(p[1]))
            except (IndexError, ValueError):
                raise RuntimeError(f"read_observations_csv: malformed row in {path}") from None
    return np.asarray(vals, dtype=np.float64)


# ---------------------------------------------------------------------- results
def write_result_json(m, report: dict, path: str, K: int, N: int, M: int) -> None:
    """write_result_json (inversion.cpp:294-317); ``report`` as Context.gauss_newton returns it."""
    steps = [{"misfit": s["misfit"], "minres_iters": int(s["minres_iters"]), "converged": bool(s["converged"]),
              "euclid_relative_residual": s["euclid_relative_residual"],
              "pnorm_relative_residual": s["pnorm_relative_residual"], "t_H": s["t_H"], "t_C": s["t_C"],
              "t_chol": s["t_chol"], "t_norm": s["t_norm"]} for s in report["steps"]]
    _dump({"m": [float(v) for v in np.asarray(m, dtype=np.float64)],
           "report": {"steps": steps, "final_misfit": report["final_misfit"], "K": int(K), "N": int(N),
                      "M": int(M)}}, path)


def write_report_csv(report: dict, path: str, nele: int, N: int, M: int) -> None:
    """The `invert --report` CSV (tools/main.cpp:221-226): nele,N,M,step,n_iter,t_H,t_C,t_chol,t_norm."""
    with open(path, "w") as f:
        f.write("nele,N,M,step,n_iter,t_H,t_C,t_chol,t_norm\n")
        for k, s in enumerate(report["steps"]):
            f.write(f"{nele},{N},{M},{k + 1},{int(s['minres_iters'])},{s['t_H']:.17g},{s['t_C']:.17g},"
                    f"{s['t_chol']:.17g},{s['t_norm']:.17g}\n")
