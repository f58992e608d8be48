"""The reference's file formats: files written by
paper_2209_02815_b200.io are read by the unmodified reference readers and vice versa
(oracle/_ref binds write_mesh_json/read_mesh_json, write/read_survey_csv, model JSON,
observations CSV and write_result_json)."""
import ctypes as C
import json
import os

import numpy as np
import pytest

import orc
from paper_2209_02815_b200 import io, workload as W

u64 = C.c_uint64


@pytest.fixture(scope="module")
def ref(oracles):
    if "reference" not in oracles:
        pytest.skip("reference library not built here")
    return oracles["reference"]


def _s(p):
    return str(p).encode()


def ref_read_mesh(ref, path):
    L = ref.L
    nv, nc, ne = u64(), u64(), u64()
    L.orc_io_read_mesh.argtypes = [C.c_char_p, C.POINTER(u64), C.POINTER(u64), C.POINTER(u64), C.c_void_p,
                                   C.c_void_p, C.c_void_p]
    ref.check(L.orc_io_read_mesh(_s(path), C.byref(nv), C.byref(nc), C.byref(ne), None, None, None))
    v, c, e = np.zeros(2 * nv.value), np.zeros(3 * nc.value, np.int64), np.zeros(ne.value, np.int64)
    ref.check(L.orc_io_read_mesh(_s(path), C.byref(nv), C.byref(nc), C.byref(ne), v.ctypes.data, c.ctypes.data,
                                 e.ctypes.data))
    return v.reshape(-1, 2), c.reshape(-1, 3), e


def test_mesh_json_both_ways(ref, tmp_path):
    mesh = W.unit_square_mesh(6)
    electrodes = np.array([1, 3, 5], dtype=np.int64)
    ours = tmp_path / "ours.json"
    io.write_mesh_json(mesh, ours, electrodes)
    v, c, e = ref_read_mesh(ref, ours)  # the reference validates our boundary tags
    assert np.array_equal(v, mesh.vertices) and np.array_equal(e, electrodes)
    p = orc.Problem.mixed(ref, mesh)
    theirs = tmp_path / "theirs.json"
    ref.L.orc_io_write_mesh.argtypes = [C.c_void_p, C.c_void_p, u64, C.c_char_p]
    ref.check(ref.L.orc_io_write_mesh(p.h, electrodes.ctypes.data, len(electrodes), _s(theirs)))
    m2, e2 = io.read_mesh_json(theirs)
    assert np.array_equal(m2.vertices, mesh.vertices) and np.array_equal(e2, electrodes)
    assert np.array_equal(m2.cells, c)  # both hold the finalized (counterclockwise) cells
    assert json.load(open(ours)) == json.load(open(theirs))
    bad = json.load(open(theirs))
    bad["boundary"][0]["tag"] = "FAR" if bad["boundary"][0]["tag"] == "SURFACE" else "SURFACE"
    json.dump(bad, open(tmp_path / "bad.json", "w"))
    with pytest.raises(RuntimeError, match="inconsistent boundary tag"):
        io.read_mesh_json(tmp_path / "bad.json")


def test_survey_observations_model_result(ref, tmp_path):
    mesh = W.unit_square_mesh(16)
    nodes = np.arange(2, 14, 2)
    sv = W.ert_survey(len(nodes), mesh.vertices[nodes, 0])
    sv["b"][0] = -1  # a pole at infinity survives the round trip
    L = ref.L
    ours = tmp_path / "s_ours.csv"
    io.write_survey_csv(sv, ours)
    theirs = tmp_path / "s_theirs.csv"
    cols = [np.ascontiguousarray(sv[k], dtype=np.int64) for k in "abmn"]
    L.orc_io_write_survey.argtypes = [C.c_void_p] * 5 + [u64, C.c_char_p]
    ref.check(L.orc_io_write_survey(*(x.ctypes.data for x in cols), sv["k"].ctypes.data, len(sv["k"]), _s(theirs)))
    assert open(ours).read() == open(theirs).read()  # byte-identical
    back = io.read_survey_csv(theirs)
    for k in "abmnk":
        assert np.array_equal(back[k], sv[k])

    g = W.gaussian(5, 40) * 1e-3
    L.orc_io_write_vector.argtypes = [C.c_int, C.c_void_p, u64, C.c_char_p]
    L.orc_io_read_vector.argtypes = [C.c_int, C.c_char_p, C.POINTER(u64), C.c_void_p]
    for kind, writer, reader, name in [(1, io.write_observations_csv, io.read_observations_csv, "g.csv"),
                                       (0, io.write_model_json, io.read_model_json, "m.json")]:
        a, b = tmp_path / ("ours_" + name), tmp_path / ("theirs_" + name)
        writer(g, a)
        ref.check(L.orc_io_write_vector(kind, g.ctypes.data, len(g), _s(b)))
        if kind == 1:
            assert open(a).read() == open(b).read()
        assert np.array_equal(reader(b), g)
        cnt = u64()
        out = np.zeros(len(g))
        ref.check(L.orc_io_read_vector(kind, _s(a), C.byref(cnt), out.ctypes.data))
        assert cnt.value == len(g) and np.array_equal(out, g)

    rep = {"steps": [dict(misfit=3.5, minres_iters=60, converged=True, euclid_relative_residual=8e-9,
                          pnorm_relative_residual=1e-8, t_H=0.01, t_C=0.002, t_chol=0.001, t_norm=0.2)],
           "final_misfit": 1.25}
    m = W.gaussian(6, 50)
    a, b = tmp_path / "r_ours.json", tmp_path / "r_theirs.json"
    io.write_result_json(m, rep, a, K=80, N=50, M=40)
    st = np.array([[3.5, 60, 1, 8e-9, 1e-8, 0.01, 0.002, 0.001, 0.2]])
    L.orc_io_write_result.argtypes = [C.c_void_p, u64, C.c_void_p, u64, C.c_double, u64, u64, C.c_char_p]
    ref.check(L.orc_io_write_result(m.ctypes.data, 50, st.ctypes.data, 1, 1.25, 80, 40, _s(b)))
    assert json.load(open(a)) == json.load(open(b))
