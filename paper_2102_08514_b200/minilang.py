"""The plan's normative scalar program: the reference's kernel mini-language (IR seam).

The reference lowers an `EvaluationPlan` to a straight-line SSA program
(`build_program`, plancompile.py:564-699), renders / parses it as text
(`KernelProgram.render`, `parse_kernel`, minilang.py:36-151) and runs it one point at a time
(`execute`, minilang.py:156-201) with the grid's fetches injected — that is
`PlanInterpreter.eval` (runtime.py:232-242) and the op-level definition the batch path and
every kernel here must agree with.  This module restates that seam so a caller of the
drop-in keeps `PlanInterpreter.program()`, `emit_kernel`, `parse_kernel` and `execute`:

* `build_program(plan)` emits the same op sequence as the reference (same register numbering,
  same constant dedup by shortest float repr, the greedy Horner factorisation of every weight
  polynomial with the documented pivot rule, exactmath.py:543-587, and fma lowered to mul +
  add), so `render()` is the reference's document byte for byte (tests/test_minilang.py,
  against digests of the reference's own `emit_kernel`);
* `execute` has the reference's float semantics (division by 0 -> +inf, mod = fmod,
  lookup truncates, select on != 0) and is bit-identical to the reference's scalar path
  (checked against the reference's `PlanInterpreter.eval` outputs in the goldens).

It is a host-side debugging / specification aid like the reference's own: evaluation in the
drop-in runs on the GPU (`PlanInterpreter.eval_batch`, `.eval`).
"""

from __future__ import annotations

import math
import re
from dataclasses import dataclass
from fractions import Fraction
from typing import Callable, Sequence

from .exact import Poly
from .plan import EvaluationPlan

MAGIC = "splinekernel"
VERSION = "1"

_ARITH = {"add": "+", "sub": "-", "mul": "*", "div": "/", "mod": "%"}
_COMPARE = {"ge": ">=", "eq": "==", "lt": "<"}
_INFIX = {**_ARITH, **_COMPARE}
_FROM_SYMBOL = {sym: kind for kind, sym in _INFIX.items()}


class KernelParseError(ValueError):
    pass


@dataclass(frozen=True)
class Op:
    kind: str
    args: tuple = ()


@dataclass
class KernelProgram:
    """`dim` arguments in, one float out (register `result`), named constant tables."""

    dim: int
    tables: dict
    ops: list
    result: int

    def render(self) -> str:
        out = [f"{MAGIC} {VERSION}", f"meta dim {self.dim}"]
        for name in sorted(self.tables):
            out.append(" ".join(["table", name] + [repr(float(v)) for v in self.tables[name]]))
        out.append("code")
        out.extend(f"let r{i} = {_expr_text(op)}" for i, op in enumerate(self.ops))
        out.append(f"return r{self.result}")
        return "\n".join(out) + "\n"


def _expr_text(op: Op) -> str:
    k, a = op.kind, op.args
    if k == "arg":
        return f"arg({a[0]})"
    if k == "const":
        return f"const({a[0]!r})"
    if k in _INFIX:
        return f"r{a[0]} {_INFIX[k]} r{a[1]}"
    if k == "floor":
        return f"floor(r{a[0]})"
    if k == "select":
        return "select(" + ", ".join(f"r{x}" for x in a) + ")"
    if k in ("fetch_nearest", "fetch_linear"):
        return f"{k}({a[0]}, " + ", ".join(f"r{x}" for x in a[1:]) + ")"
    if k == "lookup":
        return f"lookup({a[0]}, r{a[1]})"
    raise ValueError(f"unknown op kind {k}")


_STMT = re.compile(r"^let r(\d+) = (.+)$")
_CALL = re.compile(r"^(\w+)\((.*)\)$")
_BINARY = re.compile(r"^r(\d+) (\+|-|\*|/|%|>=|==|<) r(\d+)$")


def _register(tok: str) -> int:
    tok = tok.strip()
    if not tok.startswith("r"):
        raise KernelParseError(f"expected a register, got {tok!r}")
    return int(tok[1:])


def _parse_op(text: str, tables: dict) -> Op:
    m = _BINARY.match(text)
    if m:
        return Op(_FROM_SYMBOL[m.group(2)], (int(m.group(1)), int(m.group(3))))
    m = _CALL.match(text)
    if not m:
        raise KernelParseError(f"bad expression: {text}")
    fn, inner = m.group(1), m.group(2)
    parts = [p.strip() for p in inner.split(",")] if inner.strip() else []
    if fn == "arg":
        return Op("arg", (int(parts[0]),))
    if fn == "const":
        return Op("const", (float(parts[0]),))
    if fn == "floor":
        return Op("floor", (_register(parts[0]),))
    if fn == "select":
        return Op("select", tuple(_register(p) for p in parts))
    if fn in ("fetch_nearest", "fetch_linear"):
        return Op(fn, (int(parts[0]),) + tuple(_register(p) for p in parts[1:]))
    if fn == "lookup":
        if parts[0] not in tables:
            raise KernelParseError(f"unknown table {parts[0]}")
        return Op("lookup", (parts[0], _register(parts[1])))
    raise KernelParseError(f"unknown function {fn}")


def parse_kernel(text: str) -> KernelProgram:
    """The inverse of `KernelProgram.render` (minilang.py:87-118)."""
    lines = [ln.strip() for ln in text.splitlines()]
    lines = [ln for ln in lines if ln and not ln.startswith("#")]
    if not lines or not lines[0].startswith(MAGIC):
        raise KernelParseError("not a kernel document")
    head = lines[0].split()
    if len(head) < 2 or head[1] != VERSION:
        raise KernelParseError("unsupported kernel version")
    dim, result, tables, ops, code = None, None, {}, [], False
    for ln in lines[1:]:
        if ln.startswith("meta dim "):
            dim = int(ln.split()[2])
        elif ln.startswith("table "):
            _, name, *vals = ln.split()
            tables[name] = [float(v) for v in vals]
        elif ln == "code":
            code = True
        elif ln.startswith("return "):
            result = _register(ln.split()[1])
        elif code:
            m = _STMT.match(ln)
            if not m:
                raise KernelParseError(f"bad statement: {ln}")
            if int(m.group(1)) != len(ops):
                raise KernelParseError(f"register out of order: {ln}")
            ops.append(_parse_op(m.group(2), tables))
        else:
            raise KernelParseError(f"unexpected line: {ln}")
    if dim is None or result is None or result >= len(ops):
        raise KernelParseError("incomplete kernel document")
    return KernelProgram(dim, tables, ops, result)


def execute(program: KernelProgram, point: Sequence[float], fetch_nearest: Callable, fetch_linear: Callable) -> float:
    """One point through the program (minilang.py:156-201 semantics); the fetches are called
    as fetch(coset, coords_tuple)."""
    regs = [0.0] * len(program.ops)
    for i, op in enumerate(program.ops):
        k, a = op.kind, op.args
        if k == "arg":
            v = float(point[a[0]])
        elif k == "const":
            v = a[0]
        elif k == "add":
            v = regs[a[0]] + regs[a[1]]
        elif k == "sub":
            v = regs[a[0]] - regs[a[1]]
        elif k == "mul":
            v = regs[a[0]] * regs[a[1]]
        elif k == "div":
            v = regs[a[0]] / regs[a[1]] if regs[a[1]] != 0.0 else math.inf
        elif k == "mod":
            v = math.fmod(regs[a[0]], regs[a[1]])
        elif k == "floor":
            v = float(math.floor(regs[a[0]]))
        elif k == "ge":
            v = 1.0 if regs[a[0]] >= regs[a[1]] else 0.0
        elif k == "eq":
            v = 1.0 if regs[a[0]] == regs[a[1]] else 0.0
        elif k == "lt":
            v = 1.0 if regs[a[0]] < regs[a[1]] else 0.0
        elif k == "select":
            v = regs[a[1]] if regs[a[0]] != 0.0 else regs[a[2]]
        elif k == "fetch_nearest":
            v = fetch_nearest(a[0], tuple(regs[j] for j in a[1:]))
        elif k == "fetch_linear":
            v = fetch_linear(a[0], tuple(regs[j] for j in a[1:]))
        elif k == "lookup":
            v = float(program.tables[a[0]][int(regs[a[1]])])
        else:
            raise ValueError(f"unknown op kind {k}")
        regs[i] = v
    return regs[program.result]


class ProgramBuilder:
    """Append-only SSA builder; constants deduplicated by shortest repr, arguments once."""

    def __init__(self, dim: int):
        self.dim = dim
        self.ops: list = []
        self.tables: dict = {}
        self._consts: dict = {}
        self._args: dict = {}

    def emit(self, kind: str, *args) -> int:
        self.ops.append(Op(kind, tuple(args)))
        return len(self.ops) - 1

    def arg(self, i: int) -> int:
        if i not in self._args:
            self._args[i] = self.emit("arg", i)
        return self._args[i]

    def const(self, v) -> int:
        v = float(v)
        if repr(v) not in self._consts:
            self._consts[repr(v)] = self.emit("const", v)
        return self._consts[repr(v)]

    def table(self, name: str, values: Sequence) -> str:
        self.tables[name] = [float(v) for v in values]
        return name

    def finish(self, result: int) -> KernelProgram:
        return KernelProgram(self.dim, self.tables, self.ops, result)


# -- greedy Horner factorisation as an SSA op list ----------------------------------------


def horner_ops(p: Poly) -> list:
    """The reference's HornerProgram op list for p (exactmath.py:540-587): pull out the
    variable present in the most terms (ties: lowest index), recurse on quotient then
    remainder; ops ("var", i) | ("const", c) | ("add"|"mul", a, b) | ("fma", x, q, r), every
    variable register created once."""
    ops: list = []
    var_reg: dict = {}

    def var(i):
        if i not in var_reg:
            ops.append(("var", i))
            var_reg[i] = len(ops) - 1
        return var_reg[i]

    def const(c):
        ops.append(("const", Fraction(c)))
        return len(ops) - 1

    one = (0,) * p.dim

    def rec(q: Poly) -> int:
        if all(sum(e) == 0 for e in q.terms):
            return const(next(iter(q.terms.values())))
        counts = [sum(1 for e in q.terms if e[i]) for i in range(q.dim)]
        pivot = max(range(q.dim), key=lambda i: (counts[i], -i))
        quo, rem = {}, {}
        for e, c in q.terms.items():
            if e[pivot]:
                reduced = list(e)
                reduced[pivot] -= 1
                quo[tuple(reduced)] = c
            else:
                rem[e] = c
        x = var(pivot)
        quo_is_one = quo == {one: Fraction(1)}
        rq = None if quo_is_one else rec(Poly(q.dim, quo))
        if not rem:
            if quo_is_one:
                return x
            ops.append(("mul", x, rq))
            return len(ops) - 1
        rr = rec(Poly(q.dim, rem))
        if quo_is_one:
            ops.append(("add", x, rr))
        else:
            ops.append(("fma", x, rq, rr))
        return len(ops) - 1

    if p.is_zero():
        const(0)
    else:
        rec(p)
    return ops


def _inline_poly(b: ProgramBuilder, p: Poly, y: list) -> int:
    """plancompile.py:652-672: a Horner program over y, fma as mul then add."""
    regs = []
    for op in horner_ops(p):
        k = op[0]
        if k == "var":
            regs.append(y[op[1]])
        elif k == "const":
            regs.append(b.const(float(op[1])))
        elif k == "add":
            regs.append(b.emit("add", regs[op[1]], regs[op[2]]))
        elif k == "mul":
            regs.append(b.emit("mul", regs[op[1]], regs[op[2]]))
        else:
            regs.append(b.emit("add", b.emit("mul", regs[op[1]], regs[op[2]]), regs[op[3]]))
    return regs[-1]


def _site_texel(b: ProgramBuilder, plan: EvaluationPlan, site, kk, A, pb) -> list:
    """z_i = (pib_i + sum_j piA_ij site_j + kk_i) / d_i (plancompile.py:637-650)."""
    out = []
    for i in range(plan.s):
        acc = pb[i]
        for j in range(plan.s):
            if site[j]:
                acc = b.emit("add", acc, b.emit("mul", A[i][j], b.const(float(site[j]))))
        acc = b.emit("add", acc, kk[i])
        out.append(b.emit("div", acc, b.const(float(plan.diag[i]))))
    return out


def _group_value(b: ProgramBuilder, plan: EvaluationPlan, coset: int, group, y, kk, A, pb) -> int:
    """One fetch group (plancompile.py:675-699): g * fetch_nearest for singletons, else the
    merged linear fetch at base + sum_j t_j (corner_j - base) with t_j = t_num_j / g (0.5 when
    g == 0)."""
    g = _inline_poly(b, group.g, y)
    if not group.span_axes:
        z = _site_texel(b, plan, group.sites[0], kk, A, pb)
        return b.emit("mul", g, b.emit("fetch_nearest", coset, *z))
    zero, half = b.const(0.0), b.const(0.5)
    g_zero = b.emit("eq", g, zero)
    ts = [b.emit("select", g_zero, half, b.emit("div", _inline_poly(b, tn, y), g)) for tn in group.t_nums]
    base = _site_texel(b, plan, group.sites[0], kk, A, pb)
    u = list(base)
    for j in range(len(group.span_axes)):
        corner = _site_texel(b, plan, group.sites[1 << j], kk, A, pb)
        for i in range(plan.s):
            u[i] = b.emit("add", u[i], b.emit("mul", ts[j], b.emit("sub", corner[i], base[i])))
    if plan.options.texel_offset_half:
        u = [b.emit("add", ui, half) for ui in u]
    return b.emit("mul", g, b.emit("fetch_linear", coset, *u))


def build_program(plan: EvaluationPlan) -> KernelProgram:
    """Lower a plan to the IR exactly as the reference does (plancompile.py:564-634): per
    coset the frame, the Q plane tests packed into q, q mod r, sigma and the class tables,
    y = T xp - t, then every kernel's groups (predicated by kernel id when K > 1)."""
    s = plan.s
    b = ProgramBuilder(s)
    b.table("sigma", [0 if v < 0 else v for v in plan.sigma])  # sentinel slots emit class 0
    b.table("kernel_of", [c.kernel for c in plan.classes])
    b.table("T", [float(v) for c in plan.classes for row in c.T for v in row])
    b.table("t", [float(v) for c in plan.classes for v in c.t])
    b.table("piA", [float(v) for c in plan.classes for row in c.pi_linear for v in row])
    b.table("pib", [float(v) for c in plan.classes for v in c.pi_offset])
    x = [b.arg(i) for i in range(s)]
    zero = b.const(0.0)
    total = zero
    for coset, shift in enumerate(plan.shifts):
        xl = [b.emit("sub", x[i], b.const(float(shift[i]))) for i in range(s)]
        kk, xp = [], []
        for i in range(s):
            d = b.const(float(plan.diag[i]))
            kki = b.emit("mul", d, b.emit("floor", b.emit("div", xl[i], d)))
            kk.append(kki)
            xp.append(b.emit("sub", xl[i], kki))
        q = zero
        for j, (normal, off) in enumerate(plan.planes):
            dot = None
            for i, ni in enumerate(normal):
                if ni:
                    term = b.emit("mul", b.const(float(ni)), xp[i])
                    dot = term if dot is None else b.emit("add", dot, term)
            bit = b.emit("ge", dot, b.const(float(off)))
            q = b.emit("add", q, b.emit("mul", bit, b.const(float(1 << j))))
        cls = b.emit("lookup", "sigma", b.emit("mod", q, b.const(float(plan.r))))
        kid = b.emit("lookup", "kernel_of", cls)
        c_ss, c_s = b.const(float(s * s)), b.const(float(s))
        base_ss = b.emit("mul", cls, c_ss)
        base_s = b.emit("mul", cls, c_s)
        T = [[b.emit("lookup", "T", b.emit("add", base_ss, b.const(float(i * s + j)))) for j in range(s)]
             for i in range(s)]
        t = [b.emit("lookup", "t", b.emit("add", base_s, b.const(float(i)))) for i in range(s)]
        A = [[b.emit("lookup", "piA", b.emit("add", base_ss, b.const(float(i * s + j)))) for j in range(s)]
             for i in range(s)]
        pb = [b.emit("lookup", "pib", b.emit("add", base_s, b.const(float(i)))) for i in range(s)]
        y = []
        for i in range(s):
            acc = None
            for j in range(s):
                term = b.emit("mul", T[i][j], xp[j])
                acc = term if acc is None else b.emit("add", acc, term)
            y.append(b.emit("sub", acc, t[i]))
        coset_val = zero
        for kidx, kernel in enumerate(plan.kernels):
            v = zero
            for group in kernel.groups:
                v = b.emit("add", v, _group_value(b, plan, coset, group, y, kk, A, pb))
            if plan.K == 1:
                coset_val = v
            else:
                sel = b.emit("eq", kid, b.const(float(kidx)))
                coset_val = b.emit("add", coset_val, b.emit("select", sel, v, zero))
        total = b.emit("add", total, coset_val)
    return b.finish(total)


def emit_kernel(plan: EvaluationPlan) -> str:
    """plancompile.py:702-703."""
    return build_program(plan).render()
