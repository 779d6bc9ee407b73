"""Access to the reference `risec` package (the RISE API this backend plugs into).

The front end — parser, type inference, Elevate strategies, DPIA translation
— is the reference's own, unchanged.  It is installed, not
vendored, under `baseline/_ref/` (git-ignored; `__graft_entry__.build()`
installs it from /root/reference when missing).  If `risec` is already
importable (e.g. installed site-wide) that copy is used.
"""

from __future__ import annotations

import sys
from pathlib import Path

REF_DIR = Path(__file__).resolve().parent.parent / "baseline" / "_ref"

try:  # pragma: no cover - depends on the environment
    import risec  # noqa: F401
except ImportError:  # pragma: no cover
    if (REF_DIR / "risec").is_dir():
        sys.path.insert(0, str(REF_DIR))
        import risec  # noqa: F401
    else:
        raise ImportError(
            "the reference RISE front end (`risec`) is not installed; run "
            "__graft_entry__.build() (installs /root/reference into baseline/_ref)"
        )

from risec import (  # noqa: E402,F401
    cexec,
    cli,
    codegen,
    dpia,
    errors,
    expr,
    interpreter,
    lowering,
    nat,
    parser,
    primitives,
    rules,
    strategy,
    typecheck,
    types,
)
