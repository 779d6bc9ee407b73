"""Multi-process data path of the native runtime on ONE GPU (the round's GPU
budget is one device): two ranks on cuda:0 exchange conv halo rows through
peer memory (rs_ipc_* + rs_halo_exchange) and run the sharded conv through
the sm100a stencil kernel; the NCCL communicator (rs_comm_*, rs_allgather)
runs at world size 1 (NCCL rejects two ranks on one device).  Handles and
ids travel over gloo (plumbing), the data never leaves the device."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle

pytestmark = pytest.mark.gpu

W3 = (np.array([[1, 2, 1], [2, 4, 2], [1, 2, 1]], np.float32) / 16).astype(np.float32)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _halo_worker(rank, world, port, n, m, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2201_03611_b200 import compile_program, emit_cuda, programs, shard
        from paper_2201_03611_b200.run import Executable

        torch.cuda.set_device(0)
        img = oracle.rng_inputs(3, n, m)
        r0, rows = shard.row_band(n, world, rank)
        band = torch.zeros((rows + 2, m), dtype=torch.float32, device="cuda")
        band[1:-1] = torch.from_numpy(img[r0:r0 + rows]).cuda()
        torch.cuda.synchronize()
        dist.barrier()  # every band is written before any neighbour pulls from it
        halo = shard.PeerHalo(band)
        halo.exchange()
        torch.cuda.synchronize()
        top = img[r0 - 1] if rank > 0 else img[0]
        bot = img[r0 + rows] if rank < world - 1 else img[n - 1]
        ok_halo = np.array_equal(band[0].cpu().numpy(), top) and np.array_equal(band[-1].cpu().numpy(), bot)
        # the unchanged conv program on the (rows + 2)-row local image, middle rows kept
        c = compile_program(programs.CONV, None, name="conv")
        exe = Executable(emit_cuda(c.unit), {"n": rows + 2, "m": m})
        w = torch.from_numpy(W3.reshape(-1)).cuda()
        out = torch.empty((rows + 2) * m, dtype=torch.float32, device="cuda")
        exe(band.reshape(-1), w, out=out)
        torch.cuda.synchronize()
        got = out.view(rows + 2, m)[1:-1].cpu().numpy()
        ok_conv = np.array_equal(got, oracle.conv3x3(img, W3)[r0:r0 + rows])
        kinds = exe.template_kinds
        dist.barrier()  # neighbours are done reading this band
        halo.close()
        q.put((rank, ok_halo, ok_conv, kinds))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,m", [(2, 256, 512), (3, 130, 260)])
def test_peer_halo_sharded_conv_bit_exact(world, n, m):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, n, m, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_halo, ok_conv, kinds in res:
        assert ok_halo, f"rank {rank}: halo rows differ"
        assert ok_conv, f"rank {rank}: sharded conv differs from the oracle"
        assert kinds == ["stencil2d"]


def _comm_worker(port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        from paper_2201_03611_b200 import shard

        torch.cuda.set_device(0)
        comm = shard.DeviceComm()
        send = torch.arange(1000, dtype=torch.float32, device="cuda")
        recv = torch.zeros(1000, dtype=torch.float32, device="cuda")
        comm.allgather(send, recv)
        torch.cuda.synchronize()
        ok = bool(torch.equal(send, recv))
        comm.close()
        q.put(ok)
    finally:
        dist.destroy_process_group()


def test_nccl_allgather_world_one():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_comm_worker, args=(_free_port(), q))
    p.start()
    ok = q.get(timeout=240)
    p.join(timeout=60)
    assert p.exitcode == 0 and ok


def test_halo_exchange_clamps_at_global_edges(gpu):
    from paper_2201_03611_b200 import runtime

    m, rows = 64, 5
    band = torch.zeros((rows + 2, m), dtype=torch.float32, device="cuda")
    band[1:-1] = torch.arange(rows * m, dtype=torch.float32, device="cuda").view(rows, m)
    runtime.halo_exchange(band.data_ptr(), m * 4, rows)
    torch.cuda.synchronize()
    assert torch.equal(band[0], band[1]) and torch.equal(band[-1], band[-2])


def _peer_nbody_worker(rank, world, port, n, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2201_03611_b200 import compile_program, emit_cuda, programs, shard
        from paper_2201_03611_b200.run import Executable

        torch.cuda.set_device(0)
        rng = np.random.default_rng(5)
        pos = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
        vel = rng.uniform(-0.1, 0.1, (n, 3)).astype(np.float32)
        mass = rng.uniform(0.5, 1.5, n).astype(np.float32)
        t = n // world
        t0 = rank * t
        c = compile_program(programs.NBODY_SHARD, None, name="nbodyShard")
        code = emit_cuda(c.unit, peer_ranks=world)
        order = code.plan["stages"][0]["peer_streams"]
        dpos = torch.from_numpy(pos[t0:t0 + t].reshape(-1)).cuda()
        dmass = torch.from_numpy(mass[t0:t0 + t]).cuda()
        dvel = torch.from_numpy(vel[t0:t0 + t].reshape(-1)).cuda()
        torch.cuda.synchronize()
        src = shard.PeerSources({"pos": dpos, "mass": dmass}, order)
        dist.barrier()
        exe = Executable(code, {"t": t, "n": n})
        got = exe(dpos, dvel, dpos, dmass, extra={"rs_peer_table": src.table}).cpu().numpy()
        # the same target block with every source local: identical order and chunking
        local = emit_cuda(c.unit)
        want = Executable(local, {"t": t, "n": n})(
            dpos, dvel, torch.from_numpy(pos.reshape(-1)).cuda(), torch.from_numpy(mass).cuda()).cpu().numpy()
        kinds = exe.template_kinds
        dist.barrier()
        src.close()
        q.put((rank, bool(np.array_equal(got.view(np.uint32), want.view(np.uint32))), kinds))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 4096), (4, 8192)])
def test_nbody_reads_sources_from_peers_in_the_fold(world, n):
    """The all-gather fused into the allpairs kernel: sources read in place
    from every rank's block through IPC peer pointers; bit-identical to the
    same block computed with all sources local."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_nbody_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, same, kinds in res:
        assert kinds == ["allpairs"]
        assert same, f"rank {rank}: peer-source fold differs from the local-source fold"


def _fused_halo_worker(rank, world, port, n, m, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2201_03611_b200 import compile_program, emit_cuda, programs, shard
        from paper_2201_03611_b200.run import Executable

        torch.cuda.set_device(0)
        img = oracle.rng_inputs(3, n, m)
        r0, rows = shard.row_band(n, world, rank)
        band = torch.from_numpy(np.ascontiguousarray(img[r0:r0 + rows])).cuda()
        torch.cuda.synchronize()
        c = compile_program(programs.CONV, None, name="conv")
        code = emit_cuda(c.unit, peer_halo=True)
        halo = shard.PeerHaloRows(band, code.plan["stages"][0]["halo_rows"])
        dist.barrier()  # every band is written before any neighbour reads it
        exe = Executable(code, {"n": rows, "m": m})
        w = torch.from_numpy(W3.reshape(-1)).cuda()
        got = exe(band.reshape(-1), w, extra=halo.extra).cpu().numpy().reshape(rows, m)
        ok = bool(np.array_equal(got, oracle.conv3x3(img, W3)[r0:r0 + rows]))
        kinds = exe.template_kinds
        dist.barrier()  # neighbours are done reading this band
        halo.close()
        q.put((rank, ok, kinds))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,m", [(2, 256, 512), (3, 200, 260), (4, 520, 1024)])
def test_halo_fused_into_the_stencil_bit_exact(world, n, m):
    """Row bands whose stencil kernels read the neighbours' edge rows in
    place (peer pointers): each band's output equals the oracle's rows of
    the whole image, bit for bit, with no separate exchange step."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fused_halo_worker, args=(r, world, port, n, m, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, kinds in res:
        assert kinds == ["stencil2d"]
        assert ok, f"rank {rank}: fused-halo stencil differs from the oracle"


def _dot_exchange_worker(rank, world, port, n, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2201_03611_b200 import emit_cuda, programs, shard
        from paper_2201_03611_b200.run import Executable

        torch.cuda.set_device(0)
        c = programs.compile_config("dot")
        a = torch.from_numpy(oracle.rng_inputs(30 + rank, n)).cuda()
        b = torch.from_numpy(oracle.rng_inputs(40 + rank, n)).cuda()
        # this rank's own total with the plain kernel, gathered and folded in rank order on the host
        mine = Executable(emit_cuda(c.unit), {"n": n})(a, b).cpu()
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine)
        want = parts[0].clone()
        for p in parts[1:]:
            want += p
        # the fused kernel: totals exchanged in peer memory inside the reduction, several launches
        code = emit_cuda(c.unit, peer_ranks=world)
        ex = shard.PeerExchange()
        exe = Executable(code, {"n": n})
        outs = [exe(a, b, extra={"rs_peer_table": ex.table}).cpu() for _ in range(3)]
        torch.cuda.synchronize()
        dist.barrier()
        ex.close()
        same = all(np.array_equal(o.numpy().view(np.uint32), want.numpy().view(np.uint32)) for o in outs)
        q.put((rank, same, exe.template_kinds))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 1 << 20), (3, (1 << 18) + 5)])
def test_dot_totals_exchanged_in_peer_memory(world, n):
    """C1's all-gather + rank-order sum fused into the reduce kernel: every
    rank's last block publishes its total into every rank's slots (IPC peer
    memory, epoch-tagged) and folds the totals in rank order — bit-identical
    to gathering the per-rank totals and folding them on the host, launch
    after launch.  (Two processes on one GPU time-slice, so each launch
    waits for the other rank's kernel to run: slow here, not on N GPUs.)"""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dot_exchange_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, same, kinds in res:
        assert kinds == ["reduce"]
        assert same, f"rank {rank}: exchanged total differs from the rank-order fold"


def _bands_worker(rank, world, port, q):
    """gemv and sgemm row bands (SURVEY.md §8 e C2 / C4) as bench.py runs them
    strong-scaled: M / A split in row bands, x replicated; the y blocks
    all-gathered after the GEMV; B owned in 1/world row blocks and
    all-gathered before the GEMM, the C blocks gathered after it."""
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2201_03611_b200 import emit_cuda, programs, shard
        from paper_2201_03611_b200.run import Executable

        torch.cuda.set_device(0)

        def gather_rows(block):  # rank-order all-gather (gloo moves host tensors)
            parts = [None] * world
            dist.all_gather_object(parts, block.cpu().numpy())
            return np.concatenate(parts, axis=0)

        # gemv: 300 rows do not split evenly over 3 ranks' 8-row rowfold blocks
        n, m = 300, 512
        M = oracle.rng_inputs(2, n, m)
        x = oracle.rng_inputs(12, m)
        r0, rows = shard.row_band(n, world, rank)
        c = programs.compile_config("gemv")
        exe = Executable(emit_cuda(c.unit), {"n": rows, "m": m})
        y = exe(torch.from_numpy(np.ascontiguousarray(M[r0:r0 + rows]).reshape(-1)).cuda(),
                torch.from_numpy(x).cuda())
        torch.cuda.synchronize()
        y_all = gather_rows(y)
        ok_gemv = np.array_equal(y_all, oracle.mv(M, x))
        gemv_kinds = exe.template_kinds

        # sgemm: B (as Bt) replicated by an all-gather of 1/world row blocks
        n, mm, k = 256, 384, 512
        A = oracle.rng_inputs(4, n, k)
        Bt = oracle.rng_inputs(14, mm, k)
        b0, brows = shard.row_band(mm, world, rank)
        Bt_full = torch.from_numpy(gather_rows(torch.from_numpy(Bt[b0:b0 + brows]))).reshape(-1).cuda()
        r0, rows = shard.row_band(n, world, rank)
        c = programs.compile_config("sgemm")
        exe = Executable(emit_cuda(c.unit), {"n": rows, "m": mm, "k": k})
        C = exe(torch.from_numpy(np.ascontiguousarray(A[r0:r0 + rows]).reshape(-1)).cuda(), Bt_full)
        torch.cuda.synchronize()
        C_all = gather_rows(C.view(rows, mm)).reshape(n, mm)
        C64, absC = oracle.sgemm_bt_f64(A, Bt)
        ok_sgemm = bool(np.all(np.abs(C_all - C64) <= oracle.gemm_bound(k, absC)))
        q.put((rank, ok_gemv, gemv_kinds, ok_sgemm, exe.template_kinds))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gemv_sgemm_row_bands_with_gathers(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bands_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_gemv, gemv_kinds, ok_sgemm, sgemm_kinds in res:
        assert ok_gemv, f"rank {rank}: gathered gemv differs from the oracle"
        assert gemv_kinds == ["rowfold"]
        assert ok_sgemm, f"rank {rank}: gathered sgemm outside the 3xTF32 bound"
        assert sgemm_kinds == ["gemm_tc"]


def _peer_y_worker(rank, world, port, q):
    """gemv row bands whose y is all-gathered INSIDE the rowfold kernel
    (emit_cuda(peer_out=R), shard.PeerOutput): after each launch every
    rank's full y equals the whole gemv, launch after launch (epochs)."""
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2201_03611_b200 import emit_cuda, programs, shard
        from paper_2201_03611_b200.emit_cuda import eval_py
        from paper_2201_03611_b200.run import Executable

        torch.cuda.set_device(0)
        n, m = 300, 1024
        M = oracle.rng_inputs(2, n, m)
        r0, rows = shard.row_band(n, world, rank)
        exe = Executable(emit_cuda(programs.compile_config("gemv").unit, peer_out=world), {"n": rows, "m": m})
        band = torch.from_numpy(np.ascontiguousarray(M[r0:r0 + rows]).reshape(-1)).cuda()
        full = torch.zeros(n, dtype=torch.float32, device="cuda")
        torch.cuda.synchronize()
        po = shard.PeerOutput(full, r0)
        dist.barrier()
        oks = []
        for it in range(3):
            x = oracle.rng_inputs(20 + it, m)
            y = exe(band, torch.from_numpy(x).cuda(), extra=po.extra)
            torch.cuda.synchronize()
            want = oracle.mv(M, x)
            oks.append(np.array_equal(full.cpu().numpy(), want)
                       and np.array_equal(y.cpu().numpy(), want[r0:r0 + rows]))
            dist.barrier()  # every rank has read its full y before the next launch overwrites it
        kinds = exe.template_kinds
        dist.barrier()
        po.close()
        # long rows (m >= 2048) on short bands: rowfold splits each row into
        # column chunks — the in-kernel all-gather carries the split rows:
        # every rank's full y equals the ranks' own (peer-free) band results
        # gathered in rank order, within the reassociated bound
        m = 4096
        M = oracle.rng_inputs(3, n, m)
        x = oracle.rng_inputs(30, m)
        band = torch.from_numpy(np.ascontiguousarray(M[r0:r0 + rows]).reshape(-1)).cuda()
        exe = Executable(emit_cuda(programs.compile_config("gemv").unit, peer_out=world), {"n": rows, "m": m})
        plain = Executable(emit_cuda(programs.compile_config("gemv").unit), {"n": rows, "m": m})
        full.zero_()
        torch.cuda.synchronize()
        po = shard.PeerOutput(full, r0)
        dist.barrier()
        exe(band, torch.from_numpy(x).cuda(), extra=po.extra)
        torch.cuda.synchronize()
        dist.barrier()
        mine = plain(band, torch.from_numpy(x).cuda()).cpu().numpy()
        parts = [None] * world
        dist.all_gather_object(parts, mine)
        got = full.cpu().numpy()
        terms = M.astype(np.float64) * x.astype(np.float64)
        S = eval_py(exe.plan["stages"][0]["split"], {"n": rows, "m": m})
        bound = (m // S + S + 2) * oracle.U * np.abs(terms).sum(axis=1)
        oks.append(S > 1 and np.array_equal(got, np.concatenate(parts))
                   and bool(np.all(np.abs(got - terms.sum(axis=1)) <= bound)))
        dist.barrier()
        po.close()
        q.put((rank, oks, kinds))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gemv_y_all_gathered_inside_the_kernel(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_y_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, oks, kinds in res:
        assert all(oks), f"rank {rank}: the in-kernel all-gather of y differs from the oracle: {oks}"
        assert kinds == ["rowfold"]
