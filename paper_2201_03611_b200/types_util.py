"""Small helpers over the reference's data types (types.py:16-92)."""

from __future__ import annotations

from . import _ref

from ._ref import types as _t
ArrayType, ScalarType, TupleType = _t.ArrayType, _t.ScalarType, _t.TupleType
# ArrayType, ScalarType, TupleType


def array_elem(dt, depth):
    """Element type `depth` array levels below `dt`."""
    for _ in range(depth):
        dt = dt.elem
    return dt


def array_shape(dt):
    """(dims, scalar element) of a nested array type; raises on tuples in
    memory, the same restriction as codegen.array_shape (codegen.py:57-65)."""
    dims = []
    while isinstance(dt, ArrayType):
        dims.append(dt.size)
        dt = dt.elem
    if isinstance(dt, TupleType):
        EmitError = _ref.errors.EmitError

        raise EmitError("tuple-typed memory has no flat layout; keep zips as views")
    return tuple(dims), dt


def scalar_ctype(dt) -> str:
    if isinstance(dt, ScalarType):
        if dt.name == "f32":
            return "float"
        if dt.name in ("i32", "bool"):
            return "int"
    from ._ref.errors import EmitError

    raise EmitError(f"no CUDA representation for {dt!r}")
