"""N > 1 path of bench.py on CPU: two gloo ranks run the replica aggregation
(barrier + max over ranks); both must report N * steps / max(time)."""
import os
import socket

import pytest
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
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    local_time = [0.50, 0.80][rank]
    value, el = bench.replica_throughput(local_time, 5, ws)
    dist.barrier()
    out[rank] = (value, el)
    dist.destroy_process_group()


def test_replica_aggregation_gloo_ws2():
    ws, port = 2, _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(ws, port, out), nprocs=ws, join=True)
        res = dict(out)
    for r in range(ws):
        value, el = res[r]
        assert el == pytest.approx(0.80)
        assert value == pytest.approx(2 * 5 / 0.80)


def test_single_rank_is_identity():
    import sys
    sys.path.insert(0, ROOT)
    import bench
    assert bench.replica_throughput(0.25, 5, 1) == (20.0, 0.25)
