"""Multi-process halo exchange schedule (paper_2101_11856_b200/dist.py) on the
gloo backend, world sizes 2 and 3, periodic and walled z.  Each rank fills
its send buffers with a rank/direction signature; after one exchange every
receive buffer must hold exactly the neighbour's matching plane."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2101_11856_b200.dist import exchange, neighbours


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, periodic, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nb = neighbours(world, rank, periodic)
        n = 7
        send_lo = torch.full((n,), 100.0 * rank + 1)   # bottom plane, travels down
        send_hi = torch.full((n,), 100.0 * rank + 2)   # top plane, travels up
        recv_lo = torch.full((n,), -1.0)
        recv_hi = torch.full((n,), -1.0)
        works = exchange(dist, nb, rank, send_lo, send_hi, recv_lo, recv_hi, async_op=True)
        for w in works:
            w.wait()
        q.put((rank, nb.lo, nb.hi, recv_lo[0].item(), recv_hi[0].item()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,periodic", [(2, False), (2, True), (3, False), (3, True)])
def test_halo_exchange_schedule(world, periodic):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, periodic, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, lo, hi, rl, rh = q.get(timeout=120)
        out[r] = (lo, hi, rl, rh)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r, (lo, hi, rl, rh) in out.items():
        # lower ghost = the lower neighbour's TOP plane; upper ghost = the upper neighbour's BOTTOM plane
        assert rl == (100.0 * lo + 2 if lo >= 0 else -1.0)
        assert rh == (100.0 * hi + 1 if hi >= 0 else -1.0)


def test_single_rank_periodic_is_local_copy():
    nb = neighbours(1, 0, True)
    assert (nb.lo, nb.hi) == (0, 0)
    s_lo, s_hi = torch.tensor([1.0]), torch.tensor([2.0])
    r_lo, r_hi = torch.tensor([0.0]), torch.tensor([0.0])
    assert exchange(None, nb, 0, s_lo, s_hi, r_lo, r_hi) == []
    assert r_lo.item() == 2.0 and r_hi.item() == 1.0
