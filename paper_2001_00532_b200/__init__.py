"""B200 (sm_100a) backend for the scheduled sparse tensor algebra of
arXiv 2001.00532, behind the reference `spindle` scheduling API.

    from spindle.notation import parse_assignment
    from spindle.schedule import concretize, apply_schedule
    from paper_2001_00532_b200 import lower, interpret

    stmt = apply_schedule(concretize(parse_assignment("C(i,k) = A(i,j) * B(j,k)"),
                                     {"A": "ds", "B": "dd"}), schedule_text)
    prog = lower(stmt)                       # kernel-selection table
    out, stats = interpret(prog, {"A": A, "B": B})   # SPEC.md:415, on the GPU

`lower` and `interpret` are the SPEC-named entry points the reference does
not ship; they are implemented by hand-written CUDA kernels
in libspx.so (C-ABI: include/spx.h).
"""

from ._spindle import available as reference_available  # noqa: F401
from .lowering import Program, classify, lower  # noqa: F401
from .formats import DeviceTensor  # noqa: F401
from .execution import ExecStats, interpret, execute, Executor  # noqa: F401

__all__ = ["lower", "interpret", "execute", "Executor", "Program", "ExecStats", "DeviceTensor", "classify"]
