"""Seeded synthetic workloads for the BASELINE.json configs.

No public dataset is involved: the reference ships no data, and BASELINE.json names
none.  Every config is a structured unit-square mesh plus seeded Gaussian inputs:

* mesh: ``unit_square_mesh(n)`` reproduces the reference test helper
  ``make_unit_square_mesh`` (proj/tests/test_helpers.hpp:16-30) vertex-for-vertex
  and cell-for-cell; ``finalize_mesh`` connectivity is then computed by the product
  (``gnw_assemble``) and by the oracles.
* J (C1-C3): ``J = U diag(s) V^T`` with U (m x m) and V^T (m x N) orthonormalised
  from seeded N(0,1) matrices, ``s_k = 10**(-4k/m)``.
* RHS inputs: dm ~ N(0,1)^N, dg ~ N(0,1)^m with m_ref = 0, g_obs = 0, so
  ``b = assemble_gn_rhs(dm, 0, dg, 0, J, D, alpha) = [-D^T dm; J^T dg / alpha]``
  (the reference's own random-RHS pattern, test_inversion.cpp:341-360).

RNG: SplitMix64 -> 53-bit uniforms -> Box-Muller (FP64), seed
``2209028150 + 16*config_index + stream`` with streams 0=U, 1=V^T, 2=dm, 3=dg,
4=GRF, 5=noise.  Orthonormalisation: Householder QR (LAPACK through numpy) with the
sign of diag(R) made positive, so the factor is canonical.  The GPU and the CPU
oracle always consume the SAME bytes produced here; nothing is regenerated
independently on the two sides.
"""
from __future__ import annotations

import dataclasses
import numpy as np

BASE_SEED = 2209028150
_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, count: int, offset: int = 0) -> np.ndarray:
    """``count`` SplitMix64 outputs for stream ``seed`` starting at ``offset``."""
    with np.errstate(over="ignore"):
        k = np.arange(offset + 1, offset + count + 1, dtype=np.uint64)
        z = np.uint64(seed) + k * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def gaussian(seed: int, count: int) -> np.ndarray:
    """Box-Muller N(0,1) samples (FP64), deterministic for a given seed."""
    npair = (count + 1) // 2
    z = splitmix64(seed, 2 * npair)
    u = ((z >> np.uint64(11)).astype(np.float64) + 1.0) * (2.0 ** -53)  # (0, 1]
    u1, u2 = u[0::2], u[1::2]
    rad = np.sqrt(-2.0 * np.log(u1))
    ang = 2.0 * np.pi * u2
    out = np.empty(2 * npair, dtype=np.float64)
    out[0::2] = rad * np.cos(ang)
    out[1::2] = rad * np.sin(ang)
    return out[:count]


def seed_for(config_index: int, stream: int) -> int:
    return BASE_SEED + 16 * config_index + stream


def orthonormal_rows(g: np.ndarray) -> np.ndarray:
    """Rows of ``g`` (r x c, r <= c) orthonormalised: canonical Householder QR."""
    q, r = np.linalg.qr(g.T, mode="reduced")
    sgn = np.sign(np.diag(r))
    sgn[sgn == 0] = 1.0
    return np.ascontiguousarray((q * sgn).T)


def synthetic_jacobian(m: int, n_cells: int, config_index: int) -> np.ndarray:
    """J = U diag(s) V^T, s_k = 10^(-4k/m); row-major m x N float64."""
    u = orthonormal_rows(gaussian(seed_for(config_index, 0), m * m).reshape(m, m))
    vt = orthonormal_rows(gaussian(seed_for(config_index, 1), m * n_cells).reshape(m, n_cells))
    s = 10.0 ** (-4.0 * np.arange(m) / m)
    return np.ascontiguousarray((u * s) @ vt)


@dataclasses.dataclass
class Mesh:
    """Raw (pre-finalize) triangulation arrays in the reference's layout."""

    vertices: np.ndarray  # (nv, 2) float64, (x, z)
    cells: np.ndarray  # (nc, 3) int64

    @property
    def n_vertices(self) -> int:
        return self.vertices.shape[0]

    @property
    def n_cells(self) -> int:
        return self.cells.shape[0]


def unit_square_mesh(n: int) -> Mesh:
    """make_unit_square_mesh(n), proj/tests/test_helpers.hpp:16-30.

    Vertices j-major with x = i/n, z = j/n; per square the two CCW cells
    (i,j),(i+1,j),(i+1,j+1) and (i,j),(i+1,j+1),(i,j+1).
    """
    idx = np.arange(n + 1, dtype=np.float64)
    xs = np.tile(idx, n + 1) / float(n)
    zs = np.repeat(idx, n + 1) / float(n)
    vertices = np.stack([xs, zs], axis=1)
    i = np.tile(np.arange(n, dtype=np.int64), n)
    j = np.repeat(np.arange(n, dtype=np.int64), n)

    def vid(a, b):
        return b * (n + 1) + a

    c0 = np.stack([vid(i, j), vid(i + 1, j), vid(i + 1, j + 1)], axis=1)
    c1 = np.stack([vid(i, j), vid(i + 1, j + 1), vid(i, j + 1)], axis=1)
    cells = np.empty((2 * n * n, 3), dtype=np.int64)
    cells[0::2] = c0
    cells[1::2] = c1
    return Mesh(np.ascontiguousarray(vertices), cells)


def mixed_sizes(n: int) -> tuple[int, int]:
    """(K, N) of the RT0 x P0 pair on unit_square_mesh(n): K = 3n^2 + 2n, N = 2n^2."""
    return 3 * n * n + 2 * n, 2 * n * n


@dataclasses.dataclass(frozen=True)
class GnStepConfig:
    name: str
    index: int
    n: int
    m: int
    alphas: tuple
    coarse_threshold: int = 64


# BASELINE.json configs C1..C3 (C4/C5 are ERT configs with a physical J).
CONFIGS = {
    "C1": GnStepConfig("C1", 0, 64, 32, (1e-2,)),
    "C2": GnStepConfig("C2", 1, 512, 256, (1e-4, 1e-3, 1e-2, 1e-1, 1.0)),
    "C3": GnStepConfig("C3", 2, 2048, 1024, (1e-3,), coarse_threshold=4096),
}


@dataclasses.dataclass
class GnStepInputs:
    mesh: Mesh
    J: np.ndarray
    dm: np.ndarray
    dg: np.ndarray


@dataclasses.dataclass(frozen=True)
class ErtConfigSpec:
    """BASELINE C4/C5: unit square n x n, n_ele equispaced top-edge (z = 0) electrodes."""

    name: str
    index: int
    n: int
    n_ele: int
    first: int   # node index of electrode 0 on the z = 0 row
    step: int    # node spacing between electrodes
    alpha: float
    coarse_threshold: int = 64


ERT_CONFIGS = {
    "C4": ErtConfigSpec("C4", 3, 256, 32, 4, 8, 1e-2),
    "C5": ErtConfigSpec("C5", 4, 1024, 64, 8, 16, 1e-3, coarse_threshold=1024),
}


def ert_survey(n_ele: int, positions) -> dict:
    """Adjacent-pair dipole-dipole survey (builder's rule): sources (e, e+1),
    readings (k, k+1) sharing no electrode with the source; pairs k in {e-1, e, e+1} are
    dropped, and for the two edge sources also the next pair inward, so every source has
    n_ele - 4 readings (C4: 31 x 28 = 868, C5: 63 x 60 = 3780).  k = geometric_factor
    (survey.cpp:22-46) with the finite return electrode B, 2-D."""
    from .solver import geometric_factor

    pos = lambda e: (float(positions[e]), 0.0, 0.0)
    npairs = n_ele - 1
    out = {"a": [], "b": [], "m": [], "n": [], "k": []}
    for e in range(npairs):
        drop = {k for k in (e - 1, e, e + 1) if 0 <= k < npairs}
        if e == 0:
            drop.add(2)
        if e == npairs - 1:
            drop.add(npairs - 3)
        for k in range(npairs):
            if k in drop:
                continue
            out["a"].append(e)
            out["b"].append(e + 1)
            out["m"].append(k)
            out["n"].append(k + 1)
            out["k"].append(geometric_factor(pos(e), pos(e + 1), pos(k), pos(k + 1), 2))
    return {key: np.array(v, dtype=np.float64 if key == "k" else np.int64) for key, v in out.items()}


def conductivity_model(mesh: Mesh, config_index: int, corr_len: float = 0.1, n_features: int = 512) -> np.ndarray:
    """log sigma at cell centroids: a seeded Gaussian random field (random Fourier features,
    correlation length 0.1, unit variance) plus two disc inclusions (sigma x10 at
    (0.3, 0.25), sigma x0.1 at (0.7, 0.35), radius 0.1)."""
    z = gaussian(seed_for(config_index, 4), 3 * n_features)
    w = z[: 2 * n_features].reshape(n_features, 2) / corr_len
    phase = 2.0 * np.pi * ((splitmix64(seed_for(config_index, 4), n_features, offset=10 ** 9) >> np.uint64(11))
                           .astype(np.float64) * 2.0 ** -53)
    cent = mesh.vertices[mesh.cells].mean(axis=1)
    field = np.sqrt(2.0 / n_features) * np.cos(cent @ w.T + phase).sum(axis=1)
    d1 = np.hypot(cent[:, 0] - 0.3, cent[:, 1] - 0.25) < 0.1
    d2 = np.hypot(cent[:, 0] - 0.7, cent[:, 1] - 0.35) < 0.1
    field = field + np.log(10.0) * d1 + np.log(0.1) * d2
    return np.ascontiguousarray(field)


@dataclasses.dataclass
class ErtInputs:
    mesh: Mesh
    electrodes: np.ndarray  # node ids on z = 0
    survey: dict
    model: np.ndarray       # log sigma (J evaluated here)
    noise: np.ndarray       # N(0,1) per reading: g_obs = g (1 + 0.01 noise)


def ert_inputs(name: str) -> ErtInputs:
    cfg = ERT_CONFIGS[name]
    mesh = unit_square_mesh(cfg.n)
    nodes = np.array([cfg.first + cfg.step * e for e in range(cfg.n_ele)], dtype=np.int64)  # row j = 0
    survey = ert_survey(cfg.n_ele, mesh.vertices[nodes, 0])
    model = conductivity_model(mesh, cfg.index)
    noise = gaussian(seed_for(cfg.index, 5), len(survey["k"]))
    return ErtInputs(mesh, nodes, survey, model, noise)


def gnstep_inputs(n: int, m: int, config_index: int) -> GnStepInputs:
    mesh = unit_square_mesh(n)
    n_cells = mesh.n_cells
    J = synthetic_jacobian(m, n_cells, config_index) if m > 0 else np.zeros((0, n_cells))
    dm = gaussian(seed_for(config_index, 2), n_cells)
    dg = gaussian(seed_for(config_index, 3), m)
    return GnStepInputs(mesh, J, dm, dg)
