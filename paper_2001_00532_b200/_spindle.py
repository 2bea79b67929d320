"""Locate the reference front end (`spindle`), whose API this backend keeps.

The backend plugs in behind the reference's own scheduling API: statements are
built with `spindle.notation.parse_assignment`, `spindle.schedule.concretize`
and the schedule transformations, packed with `spindle.tensors.pack`, and
errors are the reference's `spindle.errors` classes.  The reference package is
installed unmodified into ``baseline/_ref`` (``pip install --no-deps --target
baseline/_ref``) or may already be importable.  Nothing here
reads the read-only source mount.
"""

from __future__ import annotations

import importlib
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
_CANDIDATES = (REPO / "baseline" / "_ref",)


def _try_import():
    try:
        return importlib.import_module("spindle.schedule")
    except ImportError:
        return None


def ensure() -> None:
    """Make `import spindle...` work or raise ImportError with instructions."""
    if _try_import() is not None:
        return
    for cand in _CANDIDATES:
        if (cand / "spindle").is_dir() and str(cand) not in sys.path:
            sys.path.append(str(cand))
            if _try_import() is not None:
                return
    raise ImportError(
        "the reference front end `spindle` is not importable; install it with "
        "`python -m pip install --no-index --no-build-isolation --no-deps "
        "--target baseline/_ref <copy of /root/reference/pkg>`"
    )


def available() -> bool:
    try:
        ensure()
        return True
    except ImportError:
        return False


ensure_ok = available()
if ensure_ok:
    from spindle import errors, fileio, graph, ir, notation, schedule, tensors  # noqa: E402,F401
else:  # pragma: no cover - exercised only without the reference installed
    errors = fileio = graph = ir = notation = schedule = tensors = None  # type: ignore[assignment]
