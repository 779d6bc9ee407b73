"""Multi-GPU decomposition of the benchmark programs (SURVEY.md §8 e).

One process per GPU; `torch.distributed` is the plumbing (NCCL on GPUs,
gloo in the CPU tests).  Each function takes the per-rank compute as a
callable, so the same host logic drives the sm100a kernels in bench.py and
the oracle in tests/test_shard.py.

* gemv / sgemm: contiguous row bands of M (A); x (B) replicated; results
  stay sharded or are all-gathered in rank order.
* dot: contiguous chunks; per-rank partial; all-gather; rank-order fold —
  never an all-reduce, whose summation order is algorithm-dependent.
* conv (padClamp2D + slide2D): row bands plus one halo row on each side,
  exchanged with the neighbours (P2P send/recv); at the global edges the
  halo is the clamped edge row, so running the unchanged program on the
  (rows + 2)-row local image and keeping the middle rows is exact.
* nbody: target blocks; positions and masses all-gathered once per step
  (the programs.NBODY_SHARD program folds a target block over all sources
  in the same source order as the single-GPU program).
"""

from __future__ import annotations

import numpy as np


def row_band(total: int, world: int, rank: int):
    """Balanced contiguous split: (start, count) of rank's rows."""
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def rank_order_sum(partials) -> np.float32:
    """Deterministic fp32 combination of per-rank partials: a left fold in
    rank order starting from the first partial."""
    acc = np.float32(partials[0])
    for p in partials[1:]:
        acc = np.float32(acc + np.float32(p))
    return acc


def allgather_rank_order(t, group=None):
    """All-gather a tensor; returns the list indexed by rank."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t.contiguous(), group=group)
    return out


def halo_exchange_rows(band, group=None):
    """band: local rows [n_local, m].  Returns [n_local + 2, m] with the
    neighbours' boundary rows (or the clamped own edge row at the global
    edges) attached above and below."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    top = band[:1].clone()
    bottom = band[-1:].clone()
    recv_top = torch.empty_like(top)
    recv_bottom = torch.empty_like(bottom)
    ops = []
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, band[:1].contiguous(), rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, recv_top, rank - 1, group))
    if rank < world - 1:
        ops.append(dist.P2POp(dist.isend, band[-1:].contiguous(), rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, recv_bottom, rank + 1, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    if rank > 0:
        top = recv_top
    if rank < world - 1:
        bottom = recv_bottom
    return torch.cat([top, band, bottom], dim=0)


def sharded_dot(partial_fn, a_chunk, b_chunk, group=None):
    """partial_fn(a, b) -> 0-d/1-element tensor partial dot on this rank."""
    p = partial_fn(a_chunk, b_chunk).reshape(1)
    parts = allgather_rank_order(p, group)
    return rank_order_sum([float(x.item()) for x in parts])


def sharded_conv(conv_fn, band, group=None):
    """conv_fn(local_image [r, m]) -> [r, m]; returns this rank's output band."""
    local = halo_exchange_rows(band, group)
    return conv_fn(local)[1:-1]


def sharded_nbody(step_fn, pos_block, vel_block, mass_block, group=None):
    """step_fn(target_pos, target_vel, all_pos, all_mass) -> new target vel."""
    import torch

    all_pos = torch.cat(allgather_rank_order(pos_block, group), dim=0)
    all_mass = torch.cat(allgather_rank_order(mass_block, group), dim=0)
    return step_fn(pos_block, vel_block, all_pos, all_mass)


# ---------------------------------------------------------------------------
# device data path through the native runtime (include/rise_b200.h
# "multi-GPU"): torch.distributed only carries the opaque handles / ids.


class PeerHalo:
    """Halo rows of a row band pulled from the neighbours' bands through peer
    memory (CUDA IPC mappings; NVLink between GPUs): rs_halo_exchange.

    `band` is this rank's device tensor [rows + 2, m] (rows 1..rows owned).
    The neighbours' bands are mapped once; `exchange()` enqueues the two row
    copies (the global edges get the clamped own edge row, padClamp2D)."""

    def __init__(self, band, group=None):
        import torch.distributed as dist

        from . import runtime

        self.band = band
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.rows = band.shape[0] - 2
        self.row_bytes = band.shape[1] * band.element_size()
        handle, off = runtime.ipc_handle(band.data_ptr())
        peers = [None] * self.world
        dist.all_gather_object(peers, (handle, off, self.rows), group=group)
        self.above = self.below = None
        self.above_rows = 0
        if self.rank > 0:
            h, o, r = peers[self.rank - 1]
            self.above, self.above_rows = runtime.ipc_open(h, o), r
        if self.rank < self.world - 1:
            h, o, _r = peers[self.rank + 1]
            self.below = runtime.ipc_open(h, o)

    def exchange(self, stream=None):
        from . import runtime

        runtime.halo_exchange(self.band.data_ptr(), self.row_bytes, self.rows, self.above, self.above_rows,
                              self.below, stream)

    def close(self):
        from . import runtime

        for p in (self.above, self.below):
            if p:
                runtime.ipc_close(p)
        self.above = self.below = None


class DeviceComm:
    """An NCCL communicator of the native runtime over a torch.distributed
    group (rank 0's ncclUniqueId is broadcast through the group)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        from . import runtime

        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        obj = [runtime.comm_unique_id() if self.rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        self.comm = runtime.NcclComm(self.world, self.rank, obj[0])

    def allgather(self, send, recv, stream=None):
        """recv (world * send.numel()) <- every rank's send, in rank order."""
        assert recv.numel() == send.numel() * self.world
        self.comm.allgather(send.data_ptr(), recv.data_ptr(), send.numel() * send.element_size(), stream)

    def close(self):
        self.comm.close()


class PeerSources:
    """The source blocks of an `allpairs` kernel emitted with peer_ranks=R:
    every rank exports its blocks (CUDA IPC), maps everyone else's, and
    builds the device table of block pointers in the kernel's stream order
    (plan stage `peer_streams`), which the kernel reads sources through —
    the all-gather of positions and masses fused into the force fold (no
    collective on the data path).

    `blocks` maps stream name -> this rank's contiguous block (device
    tensor).  Like PeerHalo this is a pull model: the caller orders the
    launch after the owners' writes of their blocks (static in the bench)."""

    def __init__(self, blocks: dict, order, group=None):
        import torch
        import torch.distributed as dist

        from . import runtime

        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        mine = {name: runtime.ipc_handle(t.data_ptr()) for name, t in blocks.items()}
        everyone = [None] * self.world
        dist.all_gather_object(everyone, mine, group=group)
        self.opened = []
        ptrs = []
        for name in order:
            for r in range(self.world):
                if r == self.rank:
                    ptrs.append(int(blocks[name].data_ptr()))
                else:
                    h, off = everyone[r][name]
                    p = runtime.ipc_open(h, off)
                    self.opened.append(p)
                    ptrs.append(p)
        self.table = torch.tensor(ptrs, dtype=torch.int64, device="cuda")

    def close(self):
        from . import runtime

        for p in self.opened:
            runtime.ipc_close(p)
        self.opened = []


class PeerExchange:
    """The exchange slots of a `reduce` kernel emitted with peer_ranks=R:
    every rank owns 2R zeroed 64-bit slots (two banks, used by epoch parity) (CUDA IPC-exported), maps everyone
    else's, and hands the kernel a device table [slot array of rank 0 .. R-1,
    this rank].  The kernel's last block writes this rank's total into slot
    `rank` of every rank's array (a system-scope release store of
    epoch << 32 | bits) and folds the R totals in rank order as they arrive
    — the all-gather + rank-order sum of SURVEY.md §8 e C1 inside the
    reduction kernel, no collective call."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist

        from . import runtime

        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        # two banks of R slots, by epoch parity (the kernel's rs_bank)
        self.slots = torch.zeros(2 * self.world, dtype=torch.int64, device="cuda")
        torch.cuda.synchronize()
        everyone = [None] * self.world
        dist.all_gather_object(everyone, runtime.ipc_handle(self.slots.data_ptr()), group=group)
        self.opened = []
        ptrs = []
        for r in range(self.world):
            if r == self.rank:
                ptrs.append(int(self.slots.data_ptr()))
            else:
                p = runtime.ipc_open(*everyone[r])
                self.opened.append(p)
                ptrs.append(p)
        self.table = torch.tensor(ptrs + [self.rank], dtype=torch.int64, device="cuda")
        dist.barrier(group=group)

    def close(self):
        from . import runtime

        for p in self.opened:
            runtime.ipc_close(p)
        self.opened = []


class PeerHaloRows:
    """The halo rows of a `stencil2d` kernel emitted with peer_halo=True:
    each rank maps its neighbours' bands (CUDA IPC) once and hands the
    kernel pointers to the rows it reads in place — the last `above` rows
    of the band above and the first `below` rows of the band below (plan
    stage `halo_rows`); at the image's real edges the pointer is NULL and
    the kernel clamps (padClamp2D).  `band` is this rank's [rows, m] device
    tensor (no halo rows of its own)."""

    def __init__(self, band, halo_rows, group=None):
        import torch.distributed as dist

        from . import runtime

        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        rows, m = band.shape
        esize = band.element_size()
        handle, off = runtime.ipc_handle(band.data_ptr())
        peers = [None] * self.world
        dist.all_gather_object(peers, (handle, off, rows), group=group)
        ht, hb = halo_rows
        self.opened = []
        self.extra = {"rs_halo_top": 0, "rs_halo_bot": 0}
        if self.rank > 0:
            h, o, r = peers[self.rank - 1]
            if r < ht:
                raise ValueError(f"the band above has {r} rows; the stencil needs {ht}")
            p = runtime.ipc_open(h, o)
            self.opened.append(p)
            self.extra["rs_halo_top"] = p + (r - ht) * m * esize
        if self.rank < self.world - 1:
            h, o, r = peers[self.rank + 1]
            if r < hb:
                raise ValueError(f"the band below has {r} rows; the stencil needs {hb}")
            p = runtime.ipc_open(h, o)
            self.opened.append(p)
            self.extra["rs_halo_bot"] = p

    def close(self):
        from . import runtime

        for p in self.opened:
            runtime.ipc_close(p)
        self.opened = []


class PeerOutput:
    """The full-result buffers of a `rowfold` kernel emitted with
    peer_out=R (gemv row bands whose y is all-gathered inside the kernel):
    every rank owns a full-length result buffer (`full`, device tensor),
    exports it (CUDA IPC), maps everyone else's, and hands the kernel
    `extra["rs_y_table"]` = [R buffer pointers (rank order), this rank's
    first row] — each row's value lands in every rank's buffer at that
    offset — and `extra["rs_peer_table"]`, the completion slots
    (`PeerExchange`): the kernel's last block publishes the launch's epoch to
    every rank and waits for every rank's, so when the kernel has finished,
    this rank's `full` holds every rank's rows."""

    def __init__(self, full, row_offset: int, group=None):
        import torch
        import torch.distributed as dist

        from . import runtime

        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        everyone = [None] * self.world
        dist.all_gather_object(everyone, runtime.ipc_handle(full.data_ptr()), group=group)
        self.opened = []
        ptrs = []
        for r in range(self.world):
            if r == self.rank:
                ptrs.append(int(full.data_ptr()))
            else:
                p = runtime.ipc_open(*everyone[r])
                self.opened.append(p)
                ptrs.append(p)
        self.full = full
        self.table = torch.tensor(ptrs + [int(row_offset)], dtype=torch.int64, device="cuda")
        self.exchange = PeerExchange(group)
        self.extra = {"rs_y_table": self.table, "rs_peer_table": self.exchange.table}

    def close(self):
        from . import runtime

        for p in self.opened:
            runtime.ipc_close(p)
        self.opened = []
        self.exchange.close()
