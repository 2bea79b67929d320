"""ImperativeIR -> CUDA for sm_100a (the generic path's code generator).

`irlower.lower_ir` produces the reference's IR (ir.py:116-219) with the
schedule's loops, recoveries and guards; this module prints it as one CUDA
kernel, compiled at run time with NVRTC (`spx_jit_compile`, csrc/spx_jit.cu)
for the current device and launched through the driver API.

Parallel loops map onto the hardware the way the schedule tags them
(SPEC.md §parallelize; §5 GPU units):

* GPUBlock  -> blockIdx.x, stride gridDim.x
* GPUWarp   -> threadIdx.x / 32, stride blockDim.x / 32
* GPUThread -> lane (threadIdx.x % 32, stride 32) under a GPUWarp loop, else
  threadIdx.x, stride blockDim.x
* CPUThread -> the global thread index when no GPU unit is used (a CPU
  schedule run on the GPU); CPUVector and repeated units stay sequential.

Every mapped loop is a strided loop (`for v = lo + idx; v < hi; v += n`), so
each iteration runs on exactly one hardware thread whatever the extents and
nesting; hardware threads no loop maps (lanes of a warp without a thread
loop) stay idle.  A program with no parallel loop has its outermost loop
spread over all threads.  Output reductions use atomicAdd unless every
mapped loop writes disjoint outputs (then a plain +=); float atomics make
the summation order, and so the last bits of the result, run dependent.

`count=True` adds per-loop iteration, guard-failure and per-instance work
counters (ExecStats).
"""

from __future__ import annotations

from dataclasses import dataclass, field

from . import _spindle

_PRELUDE = r"""
typedef %(T)s T;
typedef long long ll;
struct SpxDims { ll d[%(ND)d]; };
// ir.py:178-190 SearchSegment: largest s in [lo, hi) with arr[s] <= key (clamped)
__device__ __forceinline__ ll spx_seg(const int* __restrict__ a, ll lo, ll hi, ll key) {
  ll r = lo;
  while (lo < hi) { ll m = (lo + hi) >> 1; if ((ll)a[m] <= key) { r = m; lo = m + 1; } else hi = m; }
  return r;
}
// ir.py:193-205 SearchCoord: first s in [lo, hi) with arr[s] >= key, or hi
__device__ __forceinline__ ll spx_lb(const int* __restrict__ a, ll lo, ll hi, ll key) {
  while (lo < hi) { ll m = (lo + hi) >> 1; if ((ll)a[m] < key) lo = m + 1; else hi = m; }
  return lo;
}
"""

KERNEL = "spx_ir"


@dataclass
class Emitted:
    src: str
    loops: list  # ForLoop var names, counter order
    guard_tags: list  # If tags, counter order
    mapping: dict  # unit -> loop var
    inst: dict = field(default_factory=dict)  # parallel loop var -> (counter offset, extent expr)


def _ir():
    return _spindle.ir


class _Emit:
    def __init__(self, program, dtype: str, atomic: bool, count: bool):
        self.p = program
        self.T = "float" if dtype == "f32" else "double"
        self.atomic = atomic
        self.count = count
        self.order = [s.name for s in program.manifest.tensors]
        self.loops: list = []
        self.guard_tags: list = []
        self.mapping: dict = {}
        self.inst: dict = {}
        self._plan_units()

    # -- parallel units ------------------------------------------------------------
    def _walk(self, s, out):
        IR = _ir()
        if isinstance(s, IR.Block):
            for x in s.stmts:
                self._walk(x, out)
        elif isinstance(s, IR.ForLoop):
            out.append(s)
            self._walk(s.body, out)
        elif isinstance(s, IR.If):
            self._walk(s.then, out)
            if s.orelse is not None:
                self._walk(s.orelse, out)
        elif isinstance(s, IR.WhileLoop):
            self._walk(s.body, out)

    def _roots(self) -> list:
        """Top-level nests: one per additive term (lower_ir wraps each term of
        a multi-term statement in its own Block)."""
        IR = _ir()
        st = self.p.body.stmts
        if len(st) > 1 and all(isinstance(x, IR.Block) for x in st):
            return list(st)
        return [self.p.body]

    def _plan_units(self):
        """Map parallel units per term nest: the first loop carrying each GPU
        unit; without GPU units the first CPUThread loop, else the outermost
        loop, spreads over all threads ("Global")."""
        gpu = {"GPUBlock", "GPUWarp", "GPUThread"}
        self.by_var: dict = {}
        self.term_units: list = []
        self.mapping: dict = {}
        for root in self._roots():
            loops: list = []
            self._walk(root, loops)
            units: dict = {}
            for lp in loops:
                if lp.parallel is not None and lp.parallel[0] in gpu and lp.parallel[0] not in units:
                    units[lp.parallel[0]] = lp.var
            if not units:
                cpu = next((lp for lp in loops if lp.parallel is not None and lp.parallel[0] == "CPUThread"), None)
                if cpu is not None:
                    units["Global"] = cpu.var
                elif loops:
                    units["Global"] = loops[0].var  # unscheduled: spread the outermost loop
            self.term_units.append(units)
            for u, v in units.items():
                self.by_var[v] = u
                self.mapping.setdefault(u, v)
        self.cur_units = self.term_units[0] if self.term_units else {}

    def index_of(self, unit: str) -> tuple[str, str]:
        if unit == "GPUBlock":
            return "(ll)blockIdx.x", "(ll)gridDim.x"
        if unit == "GPUWarp":
            return "(ll)(threadIdx.x >> 5)", "(ll)(blockDim.x >> 5)"
        if unit == "GPUThread":
            if "GPUWarp" in self.cur_units:
                return "(ll)(threadIdx.x & 31)", "32LL"
            return "(ll)threadIdx.x", "(ll)blockDim.x"
        return "((ll)blockIdx.x * blockDim.x + threadIdx.x)", "((ll)gridDim.x * blockDim.x)"

    def active(self, units: dict) -> str:
        """Hardware threads a term nest runs on: lanes / warps / blocks no
        loop of the nest maps would repeat its work, so they sit it out."""
        if "Global" in units or not units:
            return "" if units else "blockIdx.x == 0 && threadIdx.x == 0"
        conds = []
        if "GPUThread" not in units:
            conds.append("(threadIdx.x & 31) == 0" if "GPUWarp" in units else "threadIdx.x == 0")
        if "GPUWarp" not in units and "GPUThread" in units:
            pass  # the thread loop strides over the whole block
        if "GPUBlock" not in units:
            conds.append("blockIdx.x == 0")
        return " && ".join(conds)

    # -- expressions -------------------------------------------------------------------
    def arr(self, ref) -> str:
        if ref.kind == "out":
            return "out"
        if ref.kind == "workspace":
            return f"W_{ref.tensor}"
        ti = self.order.index(ref.tensor)
        if ref.kind == "vals":
            return f"V{ti}"
        if ref.kind == "pos":
            return f"P{ti}_{ref.level}"
        if ref.kind == "crd":
            return f"C{ti}_{ref.level}"
        return f"W_{ref.tensor}"

    def e(self, x) -> str:
        IR = _ir()
        if isinstance(x, IR.IntLit):
            return f"{int(x.value)}LL"
        if isinstance(x, IR.FloatLit):
            return f"(T)({float(x.value)!r})"
        if isinstance(x, IR.VarRef):
            return "v_" + x.name
        if isinstance(x, IR.DimRef):
            return f"dims.d[{self.p.manifest.dim_index(x.tensor, x.level)}]"
        if isinstance(x, IR.Load):
            a = self.arr(x.array)
            if x.array.kind in ("pos", "crd"):
                return f"(ll){a}[{self.e(x.index)}]"
            return f"{a}[{self.e(x.index)}]"
        if isinstance(x, IR.BinOp):
            if x.op == "min":
                return f"min({self.e(x.lhs)}, {self.e(x.rhs)})"
            return f"({self.e(x.lhs)} {x.op} {self.e(x.rhs)})"
        raise TypeError(f"cannot emit expression {x!r}")

    # -- statements ----------------------------------------------------------------------
    def s(self, st, ind: int, out: list, body_ctx: list):
        IR = _ir()
        pad = "  " * ind
        if isinstance(st, IR.Block):
            for x in st.stmts:
                if isinstance(x, IR.Block):
                    out.append(pad + "{")
                    self.s(x, ind + 1, out, body_ctx)
                    out.append(pad + "}")
                else:
                    self.s(x, ind, out, body_ctx)
        elif isinstance(st, IR.Declare):
            ty = self.T if st.dtype == "f64" else "ll"
            out.append(f"{pad}{ty} v_{st.name} = {self.e(st.init)};")
        elif isinstance(st, IR.Assign):
            out.append(f"{pad}v_{st.name} = {self.e(st.value)};")
        elif isinstance(st, IR.ForLoop):
            v = "v_" + st.var
            lo, hi = self.e(st.lo), self.e(st.hi)
            k = len(self.loops)
            self.loops.append(st.var)
            if st.unroll:
                out.append(f"{pad}#pragma unroll {int(st.unroll)}")
            unit = self.by_var.get(st.var)
            if unit is not None:
                idx, n = self.index_of(unit)
                out.append(f"{pad}for (ll {v} = {lo} + {idx}; {v} < {hi}; {v} += {n}) {{")
            else:
                out.append(f"{pad}for (ll {v} = {lo}; {v} < {hi}; ++{v}) {{")
            if self.count:
                out.append(f"{pad}  ++lc{k};")
            ctx = body_ctx + ([st] if st.parallel is not None or unit is not None else [])
            self.s(st.body, ind + 1, out, ctx)
            out.append(pad + "}")
        elif isinstance(st, IR.WhileLoop):
            out.append(f"{pad}while ({self.e(st.cond)}) {{")
            self.s(st.body, ind + 1, out, body_ctx)
            out.append(pad + "}")
        elif isinstance(st, IR.If):
            out.append(f"{pad}if ({self.e(st.cond)}) {{")
            self.s(st.then, ind + 1, out, body_ctx)
            if self.count or st.orelse is not None:
                out.append(pad + "} else {")
                if self.count:
                    g = len(self.guard_tags)
                    self.guard_tags.append(st.tag)
                    out.append(f"{pad}  ++lg{g};")
                if st.orelse is not None:
                    self.s(st.orelse, ind + 1, out, body_ctx)
            out.append(pad + "}")
        elif isinstance(st, IR.ReduceAdd):
            tgt = f"{self.arr(st.array)}[{self.e(st.index)}]"
            if self.atomic:
                out.append(f"{pad}atomicAdd(&{tgt}, (T)({self.e(st.value)}));")
            else:
                out.append(f"{pad}{tgt} += (T)({self.e(st.value)});")
            if self.count:
                out.append(f"{pad}++lb;")
                for lp in body_ctx:
                    if lp.var in self.inst:
                        off = self.inst[lp.var][0]
                        out.append(f"{pad}atomicAdd(icnt + {off} + (v_{lp.var} - ({self.e(lp.lo)})), 1ULL);")
        elif isinstance(st, IR.Store):
            out.append(f"{pad}{self.arr(st.array)}[{self.e(st.index)}] = {self.e(st.value)};")
        elif isinstance(st, IR.SearchSegment):
            out.append(f"{pad}ll v_{st.result} = spx_seg({self.arr(st.array)}, {self.e(st.lo)}, {self.e(st.hi)}, "
                       f"{self.e(st.key)});")
        elif isinstance(st, IR.SearchCoord):
            out.append(f"{pad}ll v_{st.result} = spx_lb({self.arr(st.array)}, {self.e(st.lo)}, {self.e(st.hi)}, "
                       f"{self.e(st.key)});")
        elif isinstance(st, IR.AssertExtent):
            out.append(f"{pad}if ({self.e(st.actual)} != {self.e(st.expected)}) {{ atomicExch(err, 1); return; }}")  # noqa
        elif isinstance(st, IR.AllocWorkspace):
            # precompute workspace (SPEC.md precompute): a thread-local array of
            # the constant extent of the precomputed loop, zero-filled
            if not isinstance(st.size, IR.IntLit):
                raise TypeError("workspace extent must be a compile-time constant")
            out.append(f"{pad}T W_{st.name}[{int(st.size.value)}] = {{}};")
        else:
            raise TypeError(f"cannot emit statement {st!r}")

    def params(self) -> list[str]:
        ps = ["T* __restrict__ out"]
        for ti, slot in enumerate(self.p.manifest.tensors):
            ps.append(f"const T* __restrict__ V{ti}")
            for lvl, ch in enumerate(slot.shorthand):
                if ch == "s":
                    ps += [f"const int* __restrict__ P{ti}_{lvl}", f"const int* __restrict__ C{ti}_{lvl}"]
        ps += ["SpxDims dims", "int* __restrict__ err", "unsigned long long* __restrict__ cnt",
               "unsigned long long* __restrict__ gcnt", "unsigned long long* __restrict__ bcnt",
               "unsigned long long* __restrict__ icnt"]
        return ps

    def source(self, inst_plan: dict | None = None) -> Emitted:
        self.inst = dict(inst_plan or {})
        nd = max(1, sum(len(s.dims) for s in self.p.manifest.tensors))
        body: list = []
        for root, units in zip(self._roots(), self.term_units):
            self.cur_units = units
            act = self.active(units)
            body.append(f"  if ({act or 'true'}) {{")
            self.s(root, 2, body, [])
            body.append("  }")
        lines = [_PRELUDE % {"T": self.T, "ND": nd},
                 f'extern "C" __global__ void __launch_bounds__(1024) {KERNEL}(' + ", ".join(self.params()) + ") {"]
        if self.count:
            # per-thread counters (registers), one atomic each at the end
            lines += [f"  unsigned long long lc{k} = 0;" for k in range(len(self.loops))]
            lines += [f"  unsigned long long lg{g} = 0;" for g in range(len(self.guard_tags))]
            lines.append("  unsigned long long lb = 0;")
        lines += body
        if self.count:
            lines += [f"  if (lc{k}) atomicAdd(cnt + {k}, lc{k});" for k in range(len(self.loops))]
            lines += [f"  if (lg{g}) atomicAdd(gcnt + {g}, lg{g});" for g in range(len(self.guard_tags))]
            lines.append("  if (lb) atomicAdd(bcnt, lb);")
        lines.append("}")
        return Emitted("\n".join(lines) + "\n", self.loops, self.guard_tags, dict(self.mapping), self.inst)


def emit(program, dtype: str, *, atomic: bool = True, count: bool = False, inst_plan: dict | None = None) -> Emitted:
    """CUDA source of one kernel `spx_ir` for `program` (see module doc)."""
    return _Emit(program, dtype, atomic, count).source(inst_plan)


def parallel_loops(program) -> list:
    """(var, unit, lo, hi) of every ForLoop the emitter maps onto hardware."""
    em = _Emit(program, "f64", True, False)
    loops: list = []
    em._walk(program.body, loops)
    out = []
    for lp in loops:
        u = em.by_var.get(lp.var)
        if u is not None:
            out.append((lp.var, u, lp.lo, lp.hi))
    return out
