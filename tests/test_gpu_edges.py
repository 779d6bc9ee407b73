"""Edge cases on the GPU: empty, single-element and ragged sizes (template
preconditions fall back to the generic kernel, which is bit-exact), and the
32-bit indexing limit.  Compared with the oracle like test_gpu_parity.py."""

import numpy as np
import pytest

import oracle
from paper_2201_03611_b200 import compile_program, emit_cuda, programs, run_cuda
from paper_2201_03611_b200._ref import errors
from paper_2201_03611_b200.run import Executable

pytestmark = pytest.mark.gpu

W3 = (np.array([[1, 2, 1], [2, 4, 2], [1, 2, 1]], np.float32) / 16).astype(np.float32)


def _cfg(key):
    cfg = programs.CONFIGS[key]
    return compile_program(cfg["source"], cfg["strategy"], name=cfg["name"])


@pytest.mark.parametrize("n", [0, 1, 3, 4, 5, 7, 12, 1000003])
def test_dot_small_empty_and_ragged(gpu, n):
    c = _cfg("dot")
    a = oracle.rng_inputs(1, n)
    b = oracle.rng_inputs(2, n)
    got = run_cuda(emit_cuda(c.unit), c.unit, {"n": n}, [a, b], as_numpy=True)[0]
    from paper_2201_03611_b200 import idioms

    # the reduce template for any n (the n % 4 tail folded last)
    v64, s = oracle.dot_f64(a, b)
    assert abs(float(got) - v64) <= oracle.reassociated_dot_bound(max(n, 1), s, idioms.reduce_fold_length(n))
    if n == 0:
        assert got == np.float32(0.0)
    if n < 4:  # only tail terms: the reference's own left fold
        assert got == oracle.dot(a, b)


@pytest.mark.parametrize("n,m", [(1, 4), (3, 5), (1, 1), (31, 6), (64, 1028)])
def test_gemv_ragged_sizes_bit_exact(gpu, n, m):
    c = _cfg("gemv")
    M = oracle.rng_inputs(2, n, m)
    x = oracle.rng_inputs(3, m)
    got = run_cuda(emit_cuda(c.unit), c.unit, {"n": n, "m": m}, [M, x], as_numpy=True)
    np.testing.assert_array_equal(got, oracle.mv(M, x))


def test_gemv_zero_rows(gpu):
    c = _cfg("gemv")
    M = np.zeros((0, 8), np.float32)
    x = oracle.rng_inputs(3, 8)
    got = run_cuda(emit_cuda(c.unit), c.unit, {"n": 0, "m": 8}, [M, x], as_numpy=True)
    assert got.size == 0


@pytest.mark.parametrize("n,m", [(1, 1), (1, 7), (7, 1), (2, 2), (65, 129)])
def test_conv_degenerate_images_bit_exact(gpu, n, m):
    c = _cfg("conv")
    img = oracle.rng_inputs(9, n, m)
    got = run_cuda(emit_cuda(c.unit), c.unit, {"n": n, "m": m}, [img, W3], as_numpy=True).reshape(n, m)
    np.testing.assert_array_equal(got, oracle.conv3x3(img, W3))


def test_nbody_single_body(gpu):
    c = _cfg("nbody")
    pos = np.array([[0.5, -0.25, 0.125]], np.float32)
    vel = np.array([[1.0, 2.0, 3.0]], np.float32)
    mass = np.array([1.0], np.float32)
    got = run_cuda(emit_cuda(c.unit), c.unit, {"n": 1}, [pos, vel, mass], as_numpy=True)
    np.testing.assert_array_equal(got.reshape(1, 3), vel)  # self-interaction is softened to zero


@pytest.mark.parametrize("n,m,k", [(1, 1, 1), (3, 2, 5), (128, 256, 33)])
def test_sgemm_ragged_falls_back_bit_exact(gpu, n, m, k):
    c = _cfg("sgemm")
    A = oracle.rng_inputs(4, n, k)
    Bt = oracle.rng_inputs(5, m, k)
    got = run_cuda(emit_cuda(c.unit), c.unit, {"n": n, "m": m, "k": k}, [A, Bt], as_numpy=True).reshape(n, m)
    np.testing.assert_array_equal(got, oracle.sgemm_bt(A, Bt))


def test_int32_index_limit_is_enforced(gpu):
    c = _cfg("gemv")
    with pytest.raises(errors.InterpreterError, match="2\\^31"):
        Executable(emit_cuda(c.unit), {"n": 65536, "m": 65536})


def test_missing_size_is_reported(gpu):
    c = _cfg("gemv")
    with pytest.raises(errors.InterpreterError, match="missing size"):
        run_cuda(emit_cuda(c.unit), c.unit, {"n": 4}, [np.zeros((4, 4), np.float32), np.zeros(4, np.float32)])


def test_wrong_input_length_is_reported(gpu):
    c = _cfg("gemv")
    with pytest.raises(errors.InterpreterError):
        run_cuda(emit_cuda(c.unit), c.unit, {"n": 4, "m": 4}, [np.zeros((4, 3), np.float32), np.zeros(4, np.float32)])


def test_stream_host_pipelines_every_step(gpu):
    """Executable.stream_host: each step's own inputs in, its own result out,
    with the copies of neighbouring steps overlapping its kernels."""
    import torch

    from paper_2201_03611_b200.run import Executable

    c = compile_program(programs.MV, programs.MV_GLOBAL_STRATEGY, name="mv")
    n, m = 256, 1028
    exe = Executable(emit_cuda(c.unit), {"n": n, "m": m})
    steps, outs, want = [], [], []
    for k in range(5):
        M = oracle.rng_inputs(40 + k, n, m)
        x = oracle.rng_inputs(50 + k, m)
        steps.append([torch.from_numpy(M.reshape(-1)).pin_memory(), torch.from_numpy(x).pin_memory()])
        outs.append(torch.empty(n, dtype=torch.float32).pin_memory())
        want.append(oracle.mv(M, x))
    _, ms = exe.stream_host(steps, outs, timed=True)
    assert ms > 0
    for o, w in zip(outs, want):
        np.testing.assert_array_equal(o.numpy(), w)


def test_cuda_graph_replays_a_multi_kernel_unit(gpu):
    """Executable.graph: every stage of a unit (here the chunked dot's
    rowfold + seqfold) captured once into a CUDA graph and replayed; each
    replay gives the bit-identical result of the direct launch."""
    import torch

    from paper_2201_03611_b200 import gpu_rules
    from paper_2201_03611_b200.run import Executable

    c = compile_program(programs.DOT, gpu_rules.CHUNKED_REDUCE_STRATEGY, name="dotChunked")
    n = 1 << 20
    exe = Executable(emit_cuda(c.unit, reassociate=False), {"n": n})
    assert len(exe.kernels) == 2
    a = torch.from_numpy(oracle.rng_inputs(1, n)).cuda()
    b = torch.from_numpy(oracle.rng_inputs(11, n)).cuda()
    want = exe(a, b).cpu().numpy()
    out = torch.zeros(1, dtype=torch.float32, device="cuda")
    stream = torch.cuda.Stream()
    g = exe.graph({"a": a, "b": b, "output": out}, stream)
    for _ in range(3):
        out.zero_()
        torch.cuda.synchronize()
        g()
        stream.synchronize()
        np.testing.assert_array_equal(out.cpu().numpy(), want)


def test_memcpy_peer_same_device(gpu):
    # rs_memcpy_peer (cuMemcpyPeerAsync); on one GPU both ends are device 0
    import torch

    src = torch.arange(1 << 20, dtype=torch.float32, device="cuda")
    dst = torch.zeros_like(src)
    stream = torch.cuda.current_stream()
    gpu.memcpy_peer(dst.data_ptr(), 0, src.data_ptr(), 0, src.numel() * 4, stream)
    torch.cuda.synchronize()
    assert torch.equal(dst, src)
    with pytest.raises(Exception):
        gpu.memcpy_peer(dst.data_ptr(), 0, src.data_ptr(), 99, 4, stream)


def test_misaligned_views_take_the_generic_kernel(gpu):
    """Templates read with 16-byte accesses (float4, bulk copies, TMA); a
    caller's view at a 4-byte offset (x[1:]) runs the stage's generic kernel
    instead of faulting — same results (gemv: bit-exact; dot: the generic
    kernel is the reference's own left fold)."""
    import torch

    c = _cfg("gemv")
    n, m = 64, 256
    M = oracle.rng_inputs(2, n, m)
    x = oracle.rng_inputs(3, m)
    exe = Executable(emit_cuda(c.unit), {"n": n, "m": m})
    Mbig = torch.zeros(n * m + 1, dtype=torch.float32, device="cuda")
    Mbig[1:] = torch.from_numpy(M.reshape(-1)).cuda()
    y = exe(Mbig[1:], torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    np.testing.assert_array_equal(y.cpu().numpy(), oracle.mv(M, x))

    c = _cfg("dot")
    a = oracle.rng_inputs(1, 4097)
    b = oracle.rng_inputs(2, 4096)
    exe = Executable(emit_cuda(c.unit), {"n": 4096})
    got = exe(torch.from_numpy(a).cuda()[1:], torch.from_numpy(b).cuda())
    torch.cuda.synchronize()
    assert got.cpu().numpy()[0] == oracle.dot(a[1:], b)
    out = torch.empty(2, dtype=torch.float32, device="cuda")
    got = exe(torch.from_numpy(a[1:].copy()).cuda(), torch.from_numpy(b).cuda(), out=out[1:])
    torch.cuda.synchronize()
    assert got.cpu().numpy()[0] == oracle.dot(a[1:], b)


def test_concurrent_executables_on_their_own_streams(gpu):
    """SURVEY §8 b threading: the runtime is thread-safe per stream — four
    host threads, each with its own Executables (so their workspaces: the
    reduce's launch counter and partial slots) on its own stream, launch a
    dot and a gemv 25 times concurrently, plus a dot executable SHARED by all
    four (its launches ordered across the streams by the executable); every
    result is the single-thread result (the dot's fixed order is
    deterministic; gemv is bit-exact)."""
    import threading

    import torch

    cd, cg = _cfg("dot"), _cfg("gemv")
    n, rows, cols = 1 << 20, 512, 1024
    a = torch.from_numpy(oracle.rng_inputs(1, n)).cuda()
    b = torch.from_numpy(oracle.rng_inputs(2, n)).cuda()
    M = oracle.rng_inputs(3, rows, cols)
    x = oracle.rng_inputs(4, cols)
    dM, dx = torch.from_numpy(M.reshape(-1)).cuda(), torch.from_numpy(x).cuda()
    want_dot = Executable(emit_cuda(cd.unit), {"n": n})(a, b).cpu().numpy()
    want_mv = oracle.mv(M, x)
    # and ONE dot executable shared by every thread: its workspaces (launch
    # counter, partial slots) stay consistent because launch() orders an
    # executable's launches across streams
    shared = Executable(emit_cuda(cd.unit), {"n": n})
    assert shared._stateful
    torch.cuda.synchronize()
    errors_seen = []

    def worker(k):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            ed = Executable(emit_cuda(cd.unit), {"n": n})
            eg = Executable(emit_cuda(cg.unit), {"n": rows, "m": cols})
            outs = []
            with torch.cuda.stream(s):
                for _ in range(25):
                    outs.append((ed(a, b, stream=s), eg(dM, dx, stream=s), shared(a, b, stream=s)))
            s.synchronize()
            for od, og, osh in outs:
                if not (np.array_equal(od.cpu().numpy().view(np.uint32), want_dot.view(np.uint32))
                        and np.array_equal(osh.cpu().numpy().view(np.uint32), want_dot.view(np.uint32))
                        and np.array_equal(og.cpu().numpy(), want_mv)):
                    errors_seen.append(k)
                    break
        except Exception as exc:  # noqa: BLE001 - reported below
            errors_seen.append(f"{k}: {exc}")

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=120)
    assert not any(t.is_alive() for t in threads)
    assert errors_seen == []


def test_run_cuda_device_tensors_in_and_out(gpu):
    """run_cuda's benchmark-style use (SURVEY §8 b run entry): CUDA tensors
    in place of nested values (zero-copy), the device output back with
    as_device=True — the same values as the nested-list call."""
    import torch

    c = _cfg("gemv")
    code = emit_cuda(c.unit)
    M = oracle.rng_inputs(3, 64, 96)
    x = oracle.rng_inputs(4, 96)
    want = run_cuda(code, c.unit, {"n": 64, "m": 96}, [M.tolist(), x.tolist()], as_numpy=True)
    dM, dx = torch.from_numpy(M).cuda(), torch.from_numpy(x).cuda()
    out = run_cuda(code, c.unit, {"n": 64, "m": 96}, [dM, dx], as_device=True)
    assert out.is_cuda and out.numel() == 64
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out.cpu().numpy(), want)
    np.testing.assert_array_equal(run_cuda(code, c.unit, {"n": 64, "m": 96}, [dM.cpu(), dx.cpu()], as_numpy=True),
                                  want)
    with pytest.raises(errors.InterpreterError):
        run_cuda(code, c.unit, {"n": 64, "m": 96}, [dM[:10], dx])
