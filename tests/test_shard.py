"""Host logic of the multi-GPU decomposition, world size 2 over gloo on CPU
(SURVEY.md §8 e).  The per-rank compute is the oracle here; on GPUs it is
the sm100a kernels (bench.py --gpus N)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2201_03611_b200 import shard

W3 = (np.array([[1, 2, 1], [2, 4, 2], [1, 2, 1]], np.float32) / 16).astype(np.float32)


def test_row_band_partitions_exactly():
    for total in (1, 7, 8192, 8193):
        for world in (1, 2, 3, 8):
            bands = [shard.row_band(total, world, r) for r in range(world)]
            assert bands[0][0] == 0
            assert all(bands[i][0] + bands[i][1] == bands[i + 1][0] for i in range(world - 1))
            assert sum(c for _, c in bands) == total
            assert max(c for _, c in bands) - min(c for _, c in bands) <= 1


def test_rank_order_sum_is_a_left_fold():
    parts = [np.float32(1e8), np.float32(1.0), np.float32(-1e8)]
    assert shard.rank_order_sum(parts) == np.float32(np.float32(np.float32(1e8) + 1.0) - np.float32(1e8))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        # conv: row bands + halo exchange, padClamp at the global edges
        img = oracle.rng_inputs(3, 37, 29)
        r0, cnt = shard.row_band(37, world, rank)
        band = torch.from_numpy(img[r0:r0 + cnt].copy())
        got = shard.sharded_conv(lambda local: torch.from_numpy(oracle.conv3x3(local.numpy(), W3)), band)
        out["conv"] = (r0, got.numpy())
        # dot: chunks, partials all-gathered and folded in rank order
        a = oracle.rng_inputs(1, 4096)
        b = oracle.rng_inputs(2, 4096)
        s0, sc = shard.row_band(4096, world, rank)
        total = shard.sharded_dot(lambda x, y: torch.tensor([float(oracle.dot(x.numpy(), y.numpy()))]),
                                  torch.from_numpy(a[s0:s0 + sc].copy()), torch.from_numpy(b[s0:s0 + sc].copy()))
        out["dot"] = float(total)
        # nbody: target blocks, positions and masses all-gathered
        n = 64
        rng = np.random.default_rng(5)
        pos = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
        vel = rng.uniform(-0.1, 0.1, (n, 3)).astype(np.float32)
        mass = rng.uniform(0.5, 1.5, n).astype(np.float32)
        t0, tc = shard.row_band(n, world, rank)

        def step(tp, tv, ap, am):
            full_pos = ap.numpy()
            full_vel = np.zeros_like(full_pos)
            full_vel[t0:t0 + tc] = tv.numpy()
            return torch.from_numpy(oracle.nbody(full_pos, full_vel, am.numpy(), t0, tc))

        nb = shard.sharded_nbody(step, torch.from_numpy(pos[t0:t0 + tc].copy()),
                                 torch.from_numpy(vel[t0:t0 + tc].copy()), torch.from_numpy(mass[t0:t0 + tc].copy()))
        out["nbody"] = (t0, nb.numpy())
        results[rank] = out
    finally:
        dist.destroy_process_group()


def test_two_rank_decomposition_matches_single_process():
    world = 2
    port = _free_port()
    manager = mp.Manager()
    results = manager.dict()
    mp.spawn(_worker, args=(world, port, results), nprocs=world, join=True)
    # conv bands reassemble into the full-image oracle, bit for bit
    img = oracle.rng_inputs(3, 37, 29)
    full = oracle.conv3x3(img, W3)
    for r in range(world):
        r0, band = results[r]["conv"]
        np.testing.assert_array_equal(band, full[r0:r0 + band.shape[0]])
    # dot: both ranks agree and equal the rank-order fold of the chunk partials
    a = oracle.rng_inputs(1, 4096)
    b = oracle.rng_inputs(2, 4096)
    parts = [oracle.dot(a[s:s + c], b[s:s + c]) for s, c in (shard.row_band(4096, world, r) for r in range(world))]
    assert results[0]["dot"] == results[1]["dot"] == float(shard.rank_order_sum(parts))
    # nbody: sharded target blocks equal the full single-process step
    n = 64
    rng = np.random.default_rng(5)
    pos = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    vel = rng.uniform(-0.1, 0.1, (n, 3)).astype(np.float32)
    mass = rng.uniform(0.5, 1.5, n).astype(np.float32)
    ref = oracle.nbody(pos, vel, mass)
    for r in range(world):
        t0, block = results[r]["nbody"]
        np.testing.assert_array_equal(block, ref[t0:t0 + block.shape[0]])
