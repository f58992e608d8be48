"""Host side of the row-partitioned solve with two gloo ranks on CPU:
the NCCL id bootstrap, the partition rule, the per-rank slice of the synthetic Jacobian
(distributed CholeskyQR2), the m-vector reduction (fixed-order sum of the rank partials) and
the saddle halo plan of libgnw itself (gnw_partition_saddle / gnw_partition_csr: the same
host/partition.cpp the device path uploads) driven through a real exchange: every rank fills
its ghosts from the owners' send lists over gloo and applies its local Q, D, D^T -- the owned
rows must equal the global operator's rows bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, out):
    import sys
    sys.path.insert(0, ROOT)
    from paper_2209_02815_b200 import partition_cells, shared_nccl_id, workload as W

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        nid = shared_nccl_id()
        ids = [None] * ws
        dist.all_gather_object(ids, nid)
        m, n = 12, 32
        N = 2 * n * n
        lo = partition_cells(N, ws)
        c0, c1 = int(lo[rank]), int(lo[rank + 1])
        Jr = W.synthetic_jacobian_slice(m, N, 2, c0, c1, "cpu", allreduce=lambda t: dist.all_reduce(t)).numpy()
        x = W.gaussian(77, N)
        u_part = torch.from_numpy(Jr @ x[c0:c1])
        parts = [torch.zeros(m, dtype=torch.float64) for _ in range(ws)]
        dist.all_gather(parts, u_part)
        u = np.zeros(m)
        for p in parts:  # rank order, as k_sum_partials
            u = u + p.numpy()
        jt_own = Jr.T @ u  # own cells of J^T u
        slices = [None] * ws
        dist.all_gather_object(slices, (c0, c1, jt_own, Jr))
        # the saddle halo plan (libgnw host code) and one exchange over gloo
        from paper_2209_02815_b200 import Context, partition_csr, partition_saddle
        mesh = W.unit_square_mesh(n)
        ctx = Context(None).assemble(mesh)
        K = ctx.K
        plan = partition_saddle(ctx, ws, rank)
        l2g, so, si, ro = plan["local_to_global"], plan["send_off"], plan["send_idx"], plan["recv_off"]
        no = plan["own_edges"] + plan["own_cells"]
        z = W.gaussian(91, K + N)  # a global saddle vector
        zl = np.zeros(len(l2g))
        zl[:no] = z[l2g[:no]]  # own entries only; ghosts come from their owners
        payload = {q: zl[si[so[q]:so[q + 1]]] for q in range(ws)}
        got = [None] * ws
        dist.all_gather_object(got, payload)
        for q in range(ws):
            zl[no + ro[q]:no + ro[q + 1]] = got[q][rank]
        mats = {w: partition_csr(ctx, ws, rank, w) for w in (0, 1, 2)}
        out[rank] = dict(ids=ids, lo=lo.tolist(), u=u, slices=slices, x=x, plan=plan, zl=zl, z=z, mats=mats, K=K)
    finally:
        dist.destroy_process_group()


def test_partitioned_host_logic_gloo_ws2():
    import sys
    sys.path.insert(0, ROOT)
    from paper_2209_02815_b200 import partition_cells, workload as W

    ws, port = 2, _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(ws, port, out), nprocs=ws, join=True)
        res = dict(out)
    # one NCCL id everywhere, one partition everywhere
    assert res[0]["ids"][0] == res[0]["ids"][1] == res[1]["ids"][0] and len(res[0]["ids"][0]) == 128
    assert res[0]["lo"] == res[1]["lo"]
    lo = res[0]["lo"]
    N = 2 * 32 * 32
    assert lo[0] == 0 and lo[-1] == N and all(b % 64 == 0 for b in lo[:-1]) and lo[1] > 0
    assert np.array_equal(np.asarray(lo), partition_cells(N, 2))
    # the slices are the single-process J, and the exchanges reproduce J x and J^T J x
    J = W.synthetic_jacobian(12, N, 2)
    Jcat = np.concatenate([s[3] for s in res[0]["slices"]], axis=1)
    assert np.max(np.abs(Jcat - J)) <= 1e-13 * np.max(np.abs(J))
    x = res[0]["x"]
    assert np.array_equal(res[0]["u"], res[1]["u"])  # identical bits on every rank
    assert np.allclose(res[0]["u"], J @ x, rtol=1e-12, atol=1e-14)
    jt = np.concatenate([s[2] for s in res[0]["slices"]])
    assert np.allclose(jt, J.T @ (J @ x), rtol=1e-11, atol=1e-13)
    # the halo exchange delivered exactly the ghosts' global values
    for r in range(ws):
        p, zl, z = res[r]["plan"], res[r]["zl"], res[r]["z"]
        assert np.array_equal(zl, z[p["local_to_global"]])
    # owned rows, ascending and disjoint, cover the saddle space; ghosts are owned elsewhere
    own = [res[r]["plan"]["local_to_global"][:res[r]["plan"]["own_edges"] + res[r]["plan"]["own_cells"]]
           for r in range(ws)]
    allown = np.sort(np.concatenate(own))
    K = res[0]["K"]
    assert np.array_equal(allown, np.arange(K + N))
    for r in range(ws):
        gh = res[r]["plan"]["local_to_global"][len(own[r]):]
        assert not np.isin(gh, own[r]).any() and np.isin(gh, own[1 - r]).all()
    # local operators on the exchanged vector = the global operator's owned rows, bit for bit
    import scipy.sparse as sp
    from paper_2209_02815_b200 import Context
    g = Context(None).assemble(W.unit_square_mesh(32))
    Q = sp.csr_matrix(tuple(reversed(g.export_csr(0)[2:])), shape=(K, K))
    D = sp.csr_matrix(tuple(reversed(g.export_csr(1)[2:])), shape=(N, K))
    z = res[0]["z"]
    y_glob = np.concatenate([Q @ z[:K] + D.T @ z[K:], D @ z[:K]])
    for r in range(ws):
        p, zl, m = res[r]["plan"], res[r]["zl"], res[r]["mats"]
        ke, nc = p["own_edges"], p["own_cells"]

        def apply(w, x):
            nr, rp, ci, va = m[w]
            return np.array([sum(va[k] * x[ci[k]] for k in range(rp[i], rp[i + 1])) for i in range(nr)])
        ye = np.array([a + b for a, b in zip(apply(0, zl), apply(2, zl[ke:]))])
        yc = apply(1, zl)
        loc = np.concatenate([ye, yc])
        assert np.allclose(loc, y_glob[p["local_to_global"][:ke + nc]], rtol=1e-14, atol=1e-14)


def test_partition_rule_edges():
    import sys
    sys.path.insert(0, ROOT)
    from paper_2209_02815_b200 import partition_cells

    for N, P in [(8192, 1), (8192, 3), (8388608, 8), (2097152, 8), (131072, 7)]:
        lo = partition_cells(N, P)
        assert lo[0] == 0 and lo[-1] == N and np.all(np.diff(lo) > 0)
        assert np.all(lo[:-1] % 64 == 0)
        assert np.max(np.diff(lo)) - np.min(np.diff(lo)) <= 128
    with pytest.raises(ValueError):
        partition_cells(100, 0)
