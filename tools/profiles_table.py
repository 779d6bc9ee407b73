#!/usr/bin/env python3
"""Regenerate the bench table of profiles/README.md from the committed bench
lines (profiles/bench_r01/bench_*.json and ref_*.json)."""
import json
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
BENCH = ROOT / "profiles" / "bench_r01"

ROWS = {
    "gemv 8192² (C2, default / headline)": ("bench_gemv", "rowfold (28-row warps, 256-column stages)", "bit-exact",
                                          "reference's emitted OpenMP C, {c} threads"),
    "gemv 8192², paper Listing-3 schedule": ("bench_gemv_opt", "rowfold", "bit-exact", "{c} threads"),
    "dot 2^24 (C1)": ("bench_dot", "reduce (TMA bulk ring)", "fp64 bound", "reference C, sequential fold, {c} thread"),
    "dot 2^24, chunked program (C1 + the chunked-reduce strategy, bit-exact order)": (
        "bench_dot_chunked", "rowfold + seqfold (register-pipelined chain), one CUDA graph, PDL", "bit-exact",
        "reference's emitted OpenMP C of the same schedule, {c} threads, host-cache warm"),
    "conv 3×3 8192² (C3)": ("bench_conv", "stencil2d (32×256 tiles, rows in by bulk copy, packed exact FFMA2/FADD2, "
                                          "rows out by bulk store)", "bit-exact",
                            "reference's emitted OpenMP C via the extension seams, {c} threads"),
    "sgemm 4096³ (C4)": ("bench_sgemm", "gemm_tc (persistent tcgen05 CTA pairs, 3xTF32, K-split tail, async-proxy "
                                        "stage signal)", "3xTF32 bound", "reference's emitted OpenMP C, 64-row sample"),
    "sgemm 4096³, B row-major (`programs.SGEMM`, transpose)": ("bench_sgemm_nn", "gemm_tc, MN-major B operand",
                                                               "3xTF32 bound", "sample as above"),
    "nbody 131072 (C5)": ("bench_nbody", "allpairs (16 source chunks / block, FFMA2)",
                          "normwise 1e-5 + ≤ reference's worst error",
                          "reference's emitted OpenMP C via the extension seams, 256-target sample"),
}


def line(name):
    return json.loads((BENCH / f"{name}.json").read_text().strip().splitlines()[-1])


def table() -> str:
    out = ["| Workload (BASELINE config) | Template | value | roofline frac | parity | "
           "CPU: reference arm (`ref_*.json`) |", "|---|---|---|---|---|---|"]
    for label, (w, tmpl, parity, refdesc) in ROWS.items():
        d, r = line(w), line(w.replace("bench_", "ref_"))
        val = f"{d['value'] / 1000:.1f} TFLOP/s" if d["unit"] == "GFLOP/s" else f"{d['value']:.0f} GB/s"
        frac = d["roofline"]["frac"]
        if w.startswith("bench_sgemm"):
            fr = f"{frac:.3f} of measured-bf16/2/3 ({d['value'] / 366700:.2f} of nominal TF32/3)"
        elif w == "bench_nbody":
            fr = f"{frac:.3f} of FP32 SIMT"
        else:
            fr = f"{frac:.3f} of HBM"
        cores = r.get("cpu_baseline", {}).get("cores", "?")
        out.append(f"| {label} | {tmpl} | {val} | {fr} | {parity} | {r['value']:.1f} {r['unit']} "
                   f"({refdesc.format(c=cores)}) |")
    return "\n".join(out) + "\n"


def main():
    p = ROOT / "profiles" / "README.md"
    s = p.read_text()
    start = s.index("| Workload (BASELINE config) |")
    end = s.index("\n\n", start) + 1
    p.write_text(s[:start] + table() + s[end:])
    print(table())


if __name__ == "__main__":
    main()
