"""CPU tier, world_size 2 over gloo: the bench's replica plumbing (barrier,
max-over-ranks timing, whole-job throughput) — "replicas only"."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(ws), LOCAL_RANK=str(rank))
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    w, r, _ = bench.dist_setup()
    bench.barrier(w)
    ms = bench.reduce_max(10.0 + 5.0 * r, w)  # rank 1 is slower
    value = bench.whole_job_value(ws=w, per_rank_units=100.0, ms=ms)
    q.put((r, ms, value))
    import torch.distributed as dist
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_two_rank_replicas_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=90) for _ in ps)
    for p in ps:
        p.join(timeout=30)
    assert [o[1] for o in out] == [15.0, 15.0]  # max over ranks
    assert all(abs(o[2] - 2 * 100.0 / 0.015) < 1e-6 for o in out)
