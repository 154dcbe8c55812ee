"""World-size-2 gloo tests of bench.py's multi-process host logic (CPU only):
handle exchange, max-over-ranks timing, TP argument consistency."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    blobs = bench.exchange_handles(bytes([rank]) * (8 + rank), world)
    mx = bench.max_over_ranks(1.5 + rank, world, device="cpu")
    # vocab shards of the TP LM head cover the vocabulary exactly once
    vp = -(-128256 // world)
    lo, hi = rank * vp, min(128256, (rank + 1) * vp)
    dist.barrier()
    q.put((rank, [b.hex() for b in blobs], mx, lo, hi))
    dist.destroy_process_group()


def test_two_rank_host_logic():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, b0, m0, lo0, hi0), (r1, b1, m1, lo1, hi1) = res
    assert b0 == b1 == [(bytes([0]) * 8).hex(), (bytes([1]) * 9).hex()]
    assert m0 == m1 == 2.5
    assert (lo0, hi0, lo1, hi1) == (0, 64128, 64128, 128256)
