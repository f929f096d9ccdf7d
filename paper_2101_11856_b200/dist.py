"""Multi-GPU z-slab decomposition: one process per GPU (torchrun), one
rank-mode Runner per process, halos moved with NCCL send/recv.

Only the 9 populations that cross a slab face move (c_z=+1 upward from the
top owned plane, c_z=-1 downward from the bottom plane): 36*nx*ny bytes per
seam per direction per step (decomp.cpp:57-103 moves all 27 in FP64).  The
engine's edge kernel writes them straight into its send buffers; the bulk
kernel runs while NCCL moves them (overlap), and the next step's kernels
read the neighbour planes straight from the receive buffers.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _abi


@dataclass
class Neighbours:
    lo: int  # rank owning the slab below (-1: none)
    hi: int  # rank owning the slab above (-1: none)


def neighbours(world: int, rank: int, periodic_z: bool) -> Neighbours:
    lo = rank - 1 if rank > 0 else (world - 1 if periodic_z else -1)
    hi = rank + 1 if rank + 1 < world else (0 if periodic_z else -1)
    return Neighbours(lo, hi)


class _CudaBuf:
    """__cuda_array_interface__ view of an engine-owned device buffer."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes // 4,), "typestr": "<f4", "data": (ptr, False),
                                         "version": 3}


def as_tensor(ptr: int, nbytes: int, device):
    import torch
    if not ptr:
        return None
    return torch.as_tensor(_CudaBuf(ptr, nbytes), device=device)


def exchange(dist, nb: Neighbours, rank: int, send_lo, send_hi, recv_lo, recv_hi, async_op: bool = True):
    """One halo exchange.  Sends go out in (to-hi, to-lo) order and receives
    are posted in (from-lo, from-hi) order on every rank, so each ordered
    pair of peers matches the same way even when lo == hi (2 ranks, periodic)
    or a rank is its own neighbour (1 rank, periodic: local copy)."""
    ops = []
    local = []
    if nb.hi >= 0:
        if nb.hi == rank:
            local.append((recv_lo, send_hi))
        else:
            ops.append(dist.P2POp(dist.isend, send_hi, nb.hi, tag=1))
    if nb.lo >= 0:
        if nb.lo == rank:
            local.append((recv_hi, send_lo))
        else:
            ops.append(dist.P2POp(dist.isend, send_lo, nb.lo, tag=2))
    if nb.lo >= 0 and nb.lo != rank:
        ops.append(dist.P2POp(dist.irecv, recv_lo, nb.lo, tag=1))
    if nb.hi >= 0 and nb.hi != rank:
        ops.append(dist.P2POp(dist.irecv, recv_hi, nb.hi, tag=2))
    for dst, src in local:
        dst.copy_(src)
    if not ops:
        return []
    works = dist.batch_isend_irecv(ops)
    if not async_op:
        for w in works:
            w.wait()
        return []
    return works


class RankStepper:
    """Drives one rank-mode Runner through the split step with NCCL halos."""

    def __init__(self, runner, dist, world: int, rank: int, periodic_z: bool, device):
        import torch
        self.r = runner
        self.dist = dist
        self.rank = rank
        self.nb = neighbours(world, rank, periodic_z)
        self.device = device
        self.stream = torch.cuda.current_stream(device)
        runner.set_stream(self.stream.cuda_stream)
        self.f = []
        for p in (0, 1):
            (sl, sh, rl, rh), nbytes = runner.halo_f(p)
            self.f.append([as_tensor(x, nbytes, device) for x in (sl, sh, rl, rh)])
        (msl, msh, mrl, mrh), mb = runner.halo_macro()
        self.macro = [as_tensor(x, mb, device) for x in (msl, msh, mrl, mrh)]
        self.has_solids = len(runner.scene.cfg.solids) > 0
        self.t = runner.step_count()
        # step 0 reads recv[0]: move the initial boundary planes once
        exchange(dist, self.nb, rank, *self.f[self.t & 1], async_op=False)
        self.pending = []
        # the engine's device motion / totals tables cover this many steps
        # between two syncs (lbmg_runner_sync_interval)
        self.sync_every = runner.sync_interval()
        self.since_sync = 0
        self.status = None

    def step(self, write_macro: bool = False):
        r = self.r
        for w in self.pending:
            w.wait()
        self.pending = []
        if self.since_sync >= self.sync_every:
            self.status = r.sync()
            self.since_sync = 0
        r.phase(_abi.PHASE_PRE)
        if self.has_solids:
            exchange(self.dist, self.nb, self.rank, *self.macro, async_op=False)
        r.phase(_abi.PHASE_MID)
        r.phase(_abi.PHASE_FLUID_EDGE, write_macro)
        nxt = (self.t + 1) & 1
        self.pending = exchange(self.dist, self.nb, self.rank, *self.f[nxt], async_op=True)
        r.phase(_abi.PHASE_FLUID_BULK, write_macro)
        r.phase(_abi.PHASE_END)
        self.t += 1
        self.since_sync += 1

    def finish(self):
        for w in self.pending:
            w.wait()
        self.pending = []
        self.since_sync = 0
        self.status = self.r.sync()
        return self.status
