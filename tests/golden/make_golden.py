#!/usr/bin/env python3
"""Generate the golden vectors that pin the oracle (tests/golden/*.json).

Runs the REFERENCE implementation itself — `risec.interpreter.eval_program`
(interpreter.py:238), the reference's semantic oracle — on small seeded
inputs for every benchmark program, plus the reference test-suite's own
known-answer cases.  Values are stored as float32 bit patterns (hex), so the
comparison in tests/test_oracle.py is bit-exact.

Programs that need the extension primitives (conv: padClamp2D/slide2D,
nbody: transpose/rsqrt) are evaluated by eval_program with the extension's
semantics registered (paper_2201_03611_b200/extension.py); their fixtures are
labelled "extension" — the reference has no oracle for those primitives.

Run in the build container (needs /root/reference or baseline/_ref):
    python tests/golden/make_golden.py
"""

from __future__ import annotations

import json
import random
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


def bits(a):
    a = np.asarray(a, dtype=np.float32)
    return [f"{int(v):08x}" for v in a.reshape(-1).view(np.uint32)]


def main():
    from paper_2201_03611_b200 import frontend, programs
    from risec.interpreter import eval_program, to_plain

    fixtures = {}

    def run(key, source, strategy, nats, inputs, origin="reference"):
        name, typed, free = frontend.typed_program(source)
        if strategy:
            typed, _ctx = frontend.rewrite(typed, strategy)
        out = eval_program(typed, nats, [i.tolist() if isinstance(i, np.ndarray) else i for i in inputs])
        fixtures[key] = {
            "origin": origin,
            "program": key,
            "nats": nats,
            "inputs": [{"shape": list(np.shape(i)), "f32": bits(i)} for i in inputs],
            "output": {"shape": list(np.shape(np.asarray(to_plain(out), dtype=np.float32))),
                       "f32": bits(np.asarray(to_plain(out), dtype=np.float32))},
        }

    rng = np.random.default_rng(20260)
    a = rng.uniform(-1, 1, 64).astype(np.float32)
    b = rng.uniform(-1, 1, 64).astype(np.float32)
    run("dot", programs.DOT, programs.DOT_STRATEGY, {"n": 64}, [a, b])
    M = rng.uniform(-1, 1, (8, 16)).astype(np.float32)
    x = rng.uniform(-1, 1, 16).astype(np.float32)
    run("mv", programs.MV, programs.MV_GLOBAL_STRATEGY, {"n": 8, "m": 16}, [M, x])
    run("mv_opt", programs.MV, programs.MV_OPT_STRATEGY, {"n": 8, "m": 16, "s": 4}, [M, x])
    A = rng.uniform(-1, 1, (6, 7)).astype(np.float32)
    Bt = rng.uniform(-1, 1, (5, 7)).astype(np.float32)
    run("sgemm_bt", programs.SGEMM_BT, None, {"n": 6, "m": 5, "k": 7}, [A, Bt])
    img = rng.uniform(-1, 1, (7, 9)).astype(np.float32)
    w = (np.array([[1, 2, 1], [2, 4, 2], [1, 2, 1]], np.float32) / 16).astype(np.float32)
    run("conv", programs.CONV, None, {"n": 7, "m": 9}, [img, w], origin="extension")
    pos = rng.uniform(-1, 1, (12, 3)).astype(np.float32)
    vel = rng.uniform(-0.1, 0.1, (12, 3)).astype(np.float32)
    mass = rng.uniform(0.5, 1.5, 12).astype(np.float32)
    run("nbody", programs.NBODY, None, {"n": 12}, [pos, vel, mass], origin="extension")

    # known-answer tests of the reference suite
    kat_mv = [np.array([[1, 2, 3], [4, 5, 6]], np.float32), np.array([1, 1, 1], np.float32)]
    run("kat_mv", programs.MV, programs.MV_GLOBAL_STRATEGY, {"n": 2, "m": 3}, kat_mv)  # test_interpreter.py:37-40
    fixtures["kat_mv"]["expect_plain"] = [6.0, 15.0]
    OUT.joinpath("oracle_golden.json").write_text(json.dumps(fixtures, indent=1) + "\n")
    print(f"wrote {len(fixtures)} fixtures to {OUT / 'oracle_golden.json'}")


if __name__ == "__main__":
    random.seed(0)
    main()
