"""The sm100a emit target on CPU: deterministic text, template selection,
NVRTC compilation for sm_100a (no GPU needed), and the drop-in behaviour of
`emit` next to the reference's targets."""

import re

import pytest

from paper_2201_03611_b200 import compile_program, emit, emit_cuda, lir, programs, runtime
from paper_2201_03611_b200._ref import codegen, errors, nat

EXPECTED_TEMPLATE = {
    "dot": "reduce",
    "gemv": "rowfold",
    "gemv_opt": "rowfold",
    "conv": "stencil2d",
    "nbody": "allpairs",
    "sgemm": "gemm_tc",
    "sgemm_tiled": "gemm_tc",
}


def _code(key):
    return emit_cuda(programs.compile_config(key).unit)


@pytest.mark.parametrize("key", sorted(programs.CONFIGS))
def test_emission_is_byte_stable(key):
    assert _code(key).text == _code(key).text


@pytest.mark.parametrize("key,kind", sorted(EXPECTED_TEMPLATE.items()))
def test_benchmark_programs_select_their_template(key, kind):
    code = _code(key)
    assert [s["kind"] for s in code.plan["stages"]] == [kind]
    # the generic kernel stays in the text as the fallback
    assert "fallback" in code.plan["stages"][0]


@pytest.mark.parametrize("key", sorted(programs.CONFIGS))
def test_templates_compile_for_sm100a_with_nvrtc(key):
    code = _code(key)
    nats = programs.CONFIGS[key]["nats"]
    targs = ", ".join(str(nats[p]) for p in code.plan["nat_params"])
    names = []
    for st in code.plan["stages"]:
        for s in (st, st.get("fallback")):
            if s:
                names.append(f"{s['name']}<{targs}>")
    cubin, lowered = runtime.compile_cubin(code.text, names, ["--fmad=false"])
    assert cubin[:4] == b"\x7fELF" and len(lowered) == len(names)


@pytest.mark.parametrize("source,strategy,name,assume,nats", [
    (programs.DOT, programs.DOT_STRATEGY, "dot", False, {"n": 65536}),
    (programs.DOT_CHUNKED, None, "dotChunked", True, {"n": 1 << 24}),
    (programs.MV, programs.MV_GLOBAL_STRATEGY, "mv", False, {"n": 256, "m": 512}),
], ids=["dot", "dot_chunked", "mv"])
def test_order_preserving_emission_compiles_for_sm100a(source, strategy, name, assume, nats):
    """reassociate=False kernels (seqfold, rowfold, generic) through NVRTC +
    ptxas: catches resource overflows (e.g. static shared memory) on CPU."""
    assumptions = [(nat.Var("n"), nat.Const(programs.DOT_CHUNK))] if assume else None
    c = compile_program(source, strategy, name=name, **({"assumptions": assumptions} if assumptions else {}))
    code = emit_cuda(c.unit, reassociate=False)
    targs = ", ".join(str(nats[p]) for p in code.plan["nat_params"])
    names = [f"{s['name']}<{targs}>" for st in code.plan["stages"] for s in (st, st.get("fallback")) if s]
    cubin, lowered = runtime.compile_cubin(code.text, names, ["--fmad=false"])
    assert cubin[:4] == b"\x7fELF" and len(lowered) == len(names)


def test_emit_keeps_reference_targets_and_rejects_cuda():
    c = programs.compile_config("gemv")
    assert emit(c.unit, "openmp") == codegen.emit(c.unit, "openmp")
    with pytest.raises(errors.EmitError):
        emit(c.unit, "cuda")  # test_codegen.py:151-154 must keep holding
    assert emit(c.unit, "sm100a").startswith("// rise-b200 sm100a")


def test_mv_opt_indices_match_listing_10():
    # tests/golden/mv_opt_kernel.cl:8-10: M[i + lId*m + m*s*wgId], x[i], output[lId + s*wgId]
    c = programs.compile_config("gemv_opt")
    prog = lir.build(c.unit)
    loads = [ld for _t, v in lir.stmt_exprs(prog.body) for ld in lir.expr_loads(v)]
    M = next(ld for ld in loads if ld.buf == "M")
    x = next(ld for ld in loads if ld.buf == "x")
    V = nat.Var
    assert nat.equal(M.index, V("i") + V("lId") * V("m") + V("m") * V("s") * V("wgId"))
    assert nat.equal(x.index, V("i"))
    stores = [t for t, _v in lir.stmt_exprs(prog.body) if isinstance(t, lir.Store)]
    assert nat.equal(stores[0].index, V("lId") + V("s") * V("wgId"))


def test_generic_kernel_maps_nested_mapglobal_to_one_grid_loop():
    # SURVEY §8 a (i): nested mapGlobal must not share one id
    src = "fun(M: Array[4, Array[3, f32]] => M |> mapGlobal(fun(r => r |> mapGlobal(fun(v => v * 2.0f)))))"
    code = emit_cuda(compile_program(src, name="nested").unit)
    assert "rs_f < rs_total" in code.text and "rs_total = 12" in code.text


def test_local_memory_becomes_shared_with_barriers():
    # SURVEY §8 a (ii): toMem(Local) between mapLocal stages needs a barrier
    src = ("depFun((n: Nat, m: Nat) => fun(M: Array[n, Array[m, f32]] => M |> mapWorkGroup(fun(row => "
           "row |> mapLocal(fun(z => z * 2.0f)) |> toMem(Local) |> mapLocal(fun(z => z + 1.0f))))))")
    code = emit_cuda(compile_program(src, name="stages").unit)
    assert "__shared__ float tmp[m];" in code.text
    body = code.text[code.text.index("stagesKernel("):]
    assert body.count("__syncthreads();") >= 2


def test_global_temporary_splits_kernels():
    # SURVEY §8 a (iii): toMem(Global) between parallel stages -> two kernels
    src = ("depFun((n: Nat) => fun(xs: Array[n, f32] => xs |> mapGlobal(fun(v => v * 2.0f)) "
           "|> toMem(Global) |> mapGlobal(fun(v => v + 1.0f))))")
    code = emit_cuda(compile_program(src, name="twoStage").unit)
    assert [s["name"] for s in code.plan["stages"]] == ["twoStageKernel_s0", "twoStageKernel_s1"]
    assert code.plan["temps"] and code.plan["temps"][0]["size"] == "n"


def test_plan_round_trips_through_the_text():
    from paper_2201_03611_b200 import plan_of

    code = _code("gemv")
    assert plan_of(code.text) == code.plan


def test_exact_mode_uses_round_to_nearest_intrinsics():
    code = _code("gemv")
    kernel = code.text[code.text.index("mvKernel_rowfold("):]
    assert "__fadd_rn(" in kernel and "__fmul_rn(" in kernel
    assert not re.search(r"accum = \(accum \+", kernel)


def test_sizes_are_template_parameters():
    code = _code("gemv")
    assert "template <int n, int m>" in code.text


# ---- GPU-oriented rewrite rules (gpu_rules.py, SURVEY.md §8 f 3) ------------


def test_chunked_schedule_is_derived_by_strategy():
    """DOT + the chunked-reduce strategy lowers to exactly the hand-written
    two-kernel program (byte-identical sm100a text)."""
    from paper_2201_03611_b200 import gpu_rules

    derived = compile_program(programs.DOT, gpu_rules.CHUNKED_REDUCE_STRATEGY, name="dotChunked")
    hand = compile_program(programs.DOT_CHUNKED, None, name="dotChunked",
                           assumptions=[(nat.Var("n"), nat.Const(programs.DOT_CHUNK))])
    a = emit_cuda(derived.unit, reassociate=False)
    b = emit_cuda(hand.unit, reassociate=False)
    assert a.text == b.text
    assert [s["kind"] for s in a.plan["stages"]] == ["rowfold", "seqfold"]


def test_split_reduce_semantics_on_the_interpreter():
    """The rewritten program means what the chunked program means (the
    reference interpreter, bit for bit), and reassociates the plain fold."""
    import numpy as np

    from paper_2201_03611_b200 import gpu_rules
    from paper_2201_03611_b200._ref import interpreter

    derived = compile_program(programs.DOT, gpu_rules.CHUNKED_REDUCE_STRATEGY, name="dotChunked")
    n = 8192
    rng = np.random.default_rng(3)
    a = [np.float32(v) for v in rng.uniform(-1, 1, n)]
    b = [np.float32(v) for v in rng.uniform(-1, 1, n)]
    got = interpreter.run_unit(derived.unit, {"n": n}, [a, b])
    parts = []
    for c0 in range(0, n, 4096):
        acc = np.float32(0)
        for x, y in zip(a[c0:c0 + 4096], b[c0:c0 + 4096]):
            acc = np.float32(acc + np.float32(x * y))
        parts.append(acc)
    want = np.float32(np.float32(np.float32(0) + parts[0]) + parts[1])
    assert np.float32(got) == want


def test_split_reduce_refuses_unknown_identities():
    from paper_2201_03611_b200 import gpu_rules
    from paper_2201_03611_b200._ref import errors as rerrors

    src = ("depFun((n: Nat) => fun(a: Array[n, f32] => a |> reduce(add)(1.0f)))")
    with pytest.raises(rerrors.StrategyError):
        compile_program(src, "splitReduce(4) @ outermost(isReduce) ; toReduceSeq @ every(isReduce)", name="s")
    assert "splitReduce" in gpu_rules.RULES and "splitMap" in gpu_rules.RULES
    from paper_2201_03611_b200._ref import rules

    assert any(r.startswith("splitReduce(") for r in rules.describe_rules())


def test_stencil_persistent_grid_avoids_power_of_two_tile_strides():
    # the tile stride of the persistent stencil blocks is kept at 2 (mod 4):
    # multiples of the strips per band pile every block onto one column strip
    # (and the same HBM channels) — DESIGN.md §3 stencil2d
    from paper_2201_03611_b200 import programs, tmpl_stencil

    c = programs.compile_config("conv")
    st = emit_cuda(c.unit).plan["stages"][0]
    for n, m in [(8192, 8192), (4096, 8192), (8192, 16384)]:
        (grid, _, _), block, smem, _ = tmpl_stencil.launch(st, {"n": n, "m": m}, 148)
        assert grid % 4 == 2 and grid <= 148 * st["blocks_per_sm"]


@pytest.mark.parametrize("name,source,nats,kind", [
    ("transposeCopy", "depFun((n: Nat, m: Nat) => fun(M: Array[n, Array[m, f32]] => "
     "M |> transpose |> mapGlobal(mapGlobal(fun(v => v * 1.0f)))))", {"n": 8192, "m": 8192}, "transpose2d"),
    ("slide1D", "depFun((n: Nat) => fun(xs: Array[n, f32] => xs |> padClamp(1)(1) |> slide(3)(1) "
     "|> mapGlobal(fun(w => w |> reduceSeq(Private)(fun(a, v => a + v))(0.0f)))))", {"n": 1 << 26}, "stencil1d"),
])
def test_layout_templates_selected_and_compile(name, source, nats, kind):
    """The layout templates (transpose2d, stencil1d) take their programs,
    keep the program's order (also under reassociate=False) and compile."""
    c = compile_program(source, None, name=name)
    for reassociate in (True, False):
        code = emit_cuda(c.unit, reassociate=reassociate)
        assert [s["kind"] for s in code.plan["stages"]] == [kind]
    targs = ", ".join(str(nats[p]) for p in code.plan["nat_params"])
    names = [f"{s['name']}<{targs}>" for st in code.plan["stages"] for s in (st, st.get("fallback")) if s]
    cubin, lowered = runtime.compile_cubin(code.text, names, ["--fmad=false"])
    assert cubin[:4] == b"\x7fELF" and len(lowered) == len(names)


def test_tiled_sgemm_is_recognised_as_the_contraction():
    """C4's tiled lowering (split / toMem(Local) / transpose / K tiles under
    mapWorkGroup / mapLocal) is claimed by gemm_tc with the flat operands:
    A K-major through the Local staging, B MN-major through the transpose."""
    st = _code("sgemm_tiled").plan["stages"][0]
    assert st["kind"] == "gemm_tc" and (st["M"], st["N"], st["K"]) == ("n", "m", "k")
    assert st["b_major"] == "mn" and st["fallback"]["kind"] == "workgroup"
    bufs = {e["buf"] for e in st["extra_args"] if e["kind"] == "tma2d"}
    assert bufs == {"A", "B"}
    # order-preserving emission keeps the program's own order: no tensor cores
    code = emit_cuda(programs.compile_config("sgemm_tiled").unit, reassociate=False)
    assert [s["kind"] for s in code.plan["stages"]] == ["workgroup"]


@pytest.mark.parametrize("edit", [
    ("acc + fst(p) * snd(p)", "acc + fst(p) * fst(p)"),     # not a product of A and B
    ("acc + fst(p) * snd(p)", "acc + fst(p) - snd(p)"),     # not a product
    ("(fun(acc, v => acc + v))(0.0f)", "(fun(acc, v => acc + v))(1.0f)"),  # non-zero init
    ("v * 1.0f", "v * 2.0f"),                                # the staging is not a copy
])
def test_tiled_sgemm_near_misses_stay_generic(edit):
    src = programs.SGEMM_TILED.replace(*edit)
    assert src != programs.SGEMM_TILED
    c = compile_program(src, None, name="sgemmTiled", assumptions=programs.sgemm_tiled_assumptions())
    assert [s["kind"] for s in emit_cuda(c.unit).plan["stages"]] == ["workgroup"]


@pytest.mark.parametrize("key,high,strategy_name", [
    ("conv", "CONV_HIGH", "CONV_STRATEGY"),
    ("sgemm_tiled", "SGEMM_HIGH", "SGEMM_TILED_STRATEGY"),
    ("nbody", "NBODY_HIGH", "NBODY_STRATEGY"),
])
def test_gpu_strategies_derive_the_hand_lowered_programs(key, high, strategy_name):
    """SURVEY.md §8 f 3: the high-level map/reduce programs, rewritten by the
    .elv strategies (reference rules + gpu_rules' splitReduce(c, a),
    insertToMemReduce, stageToMem), emit byte-identical sm100a text to the
    hand-lowered programs the templates take — with the same recorded
    divisibility assumptions."""
    from paper_2201_03611_b200 import gpu_rules

    derived = compile_program(getattr(programs, high), getattr(gpu_rules, strategy_name))
    hand = programs.compile_config(key)
    assert emit_cuda(derived.unit).text == emit_cuda(hand.unit).text
    assert set(derived.assumptions) == set(hand.assumptions)


def test_strategy_rules_are_registered_for_strategy_files():
    from paper_2201_03611_b200._ref import rules

    for name in ("splitReduce", "splitMap", "insertToMemReduce", "stageToMem"):
        assert name in rules.RULES and name in rules.RULE_PARAMS


def test_tiled_sgemm_other_tile_sizes_are_recognised():
    """The tiled matcher is not tied to the program's constants: 4-row
    blocks and K tiles of 16 (and the Bt form through the same staging)
    are the same contraction."""
    from paper_2201_03611_b200._ref import nat

    src = programs.SGEMM_TILED.replace("split(2)", "split(4)").replace("split(32)", "split(16)")
    asm = [(nat.Var("n"), nat.Const(4)), (nat.Var("k"), nat.Const(16))]
    st = emit_cuda(compile_program(src, None, name="sgemmTiled", assumptions=asm).unit).plan["stages"][0]
    assert st["kind"] == "gemm_tc" and st["b_major"] == "mn"
    bt = (programs.SGEMM_TILED.replace("B: Array[k, Array[m, f32]]", "Bt: Array[m, Array[k, f32]]")
          .replace("transpose(B)", "Bt"))
    st = emit_cuda(compile_program(bt, None, name="sgemmTiled",
                                   assumptions=programs.sgemm_tiled_assumptions()).unit).plan["stages"][0]
    assert st["kind"] == "gemm_tc" and st["b_major"] == "k"


def test_peer_out_emission():
    """peer_out=R: the rowfold kernel takes the full-result table, the
    completion slots and a launch counter; programs no rowfold takes refuse
    (no fallback could write the peers)."""
    code = emit_cuda(programs.compile_config("gemv").unit, peer_out=4)
    st = code.plan["stages"][0]
    assert st["kind"] == "rowfold" and st["peer_out"] == 4 and code.plan["peer_out"] == 4
    assert [e["kind"] for e in st["extra_args"][-3:]] == ["peer_ptr_table", "peer_table", "workspace"]
    assert "__threadfence_system();" in code.text and "rs_xchg_get" in code.text
    names = [f"{st['name']}<2048, 8192>"]
    cubin, _ = runtime.compile_cubin(code.text, names, ["--fmad=false"])
    assert cubin[:4] == b"\x7fELF"
    with pytest.raises(errors.EmitError):
        emit_cuda(programs.compile_config("conv").unit, peer_out=2)


def test_peer_ranks_marks_the_peer_source_inputs():
    from paper_2201_03611_b200 import compile_program

    c = compile_program(programs.NBODY_SHARD, None, name="nbodyShard")
    plan = emit_cuda(c.unit, peer_ranks=2).plan
    assert {i["name"] for i in plan["inputs"] if i.get("peer")} == {"pos", "mass"}


@pytest.mark.parametrize("n,m,S", [(8192, 8192, 1), (4096, 8192, 2), (2048, 8192, 4), (1024, 8192, 8),
                                   (100, 8192, 32), (1024, 1024, 1), (1024, 2048 + 4, 1)])
def test_rowfold_split_factor(n, m, S):
    """rowfold splits rows into column chunks only for short row counts of
    long rows (K >= 2048, K % 128 == 0): the full-size gemv keeps the
    program's own order."""
    from paper_2201_03611_b200.emit_cuda import eval_py

    st = _code("gemv").plan["stages"][0]
    assert eval_py(st["split"], {"n": n, "m": m}) == S
    assert eval_py(st["rows"], {"n": n, "m": m}) == n * S
    rb = eval_py(str(st["row_block"]), {"n": n, "m": m})
    assert rb % S == 0 and rb <= 32


def test_rowfold_split_needs_reassociation():
    c = programs.compile_config("gemv")
    assert "split" not in emit_cuda(c.unit, reassociate=False).plan["stages"][0]
    assert "split" in emit_cuda(c.unit).plan["stages"][0]
