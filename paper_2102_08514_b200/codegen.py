"""Build-time code generator: EvaluationPlan -> plan-specialised sm_100a evaluator.

The paper lowers each plan to LLVM/PTX (Part II; not shipped); the
reference lowers it to the mini-language of `build_program` (plancompile.py:564-699),
whose op list fixes the per-point semantics.  This generator emits the same
semantics as straight-line CUDA for one plan:

* coset loop (M unrolled), the float64 coset frame of runtime.py:371-373,
* the Q plane tests with the plan's integer normals as +/- adds, packed into a code
  (plancompile.py:593-603), `q mod r`, sigma lookup (shared memory),
* the class transform decoded from a packed record: T and piA as signed permutations
  (probe12), y = T xp - t,
* per kernel: every distinct monomial of the weight polynomials computed once, each
  polynomial an FMA chain over them (fewer operations than per-polynomial Horner); per
  fetch group the fetch
  merge done in software with a LOCAL lerp on exact integer cell indices
   — for 2-site groups the division-free form
  g*c0 + t_num*(c1 - c0), for 4/8-site groups t_j = t_num_j / g (0.5 when g == 0,
  plancompile.py:684-688) and a multilinear lerp,
* K > 1 plans branch on the class's kernel id (the reference predicates, :633-637).

Each plan becomes one translation unit `generated/plan_<ident>.cu` exporting a
`GenEntry` whose `blob` is the plan's canonical word sequence; sp_plan_create matches
an incoming plan against it exactly.
"""

from __future__ import annotations

import os
from itertools import product
import re

import numpy as np
from fractions import Fraction
from typing import List

from .exact import HNode, horner_tree
from .packing import canonical_words, pack_plan
from .plan import EvaluationPlan


def codegen_supported(plan: EvaluationPlan) -> bool:
    if plan.s != 3 or plan.M > 8 or plan.Q > 31 or plan.K > 15:
        return False
    if len(set(plan.diag)) != 1 or plan.diag[0] & (plan.diag[0] - 1):
        return False  # uniform power-of-two diagonal: x * (1/d) is exact
    if plan.tensor_bspline_degree() is not None:
        return False
    recs = plan.signed_permutation_classes()
    if recs is None:
        return False
    for r in recs:
        if any(not -128 <= v < 128 for v in r["t"]):
            return False
        if any(v % plan.diag[0] for v in r["pib"]):
            return False
    for kern in plan.kernels:
        for g in kern.groups:
            for site in g.sites:
                if any(v % plan.diag[0] for v in site):
                    return False
    return True


def ident_of(name: str) -> str:
    return re.sub(r"[^A-Za-z0-9_]", "_", name)


def _lit(q: Fraction) -> str:
    v = float(q)
    return f"T({v!r})"


class _Emitter:
    def __init__(self, prefix: str):
        self.lines: List[str] = []
        self.n = 0
        self.prefix = prefix
        self.ops = 0

    def tmp(self) -> str:
        self.n += 1
        return f"{self.prefix}{self.n}"

    def expr(self, node: HNode) -> str:
        k = node.kind
        if k == "const":
            return _lit(node.args[0])
        if k == "var":
            return f"y{node.args[0]}"
        args = [self.expr(a) for a in node.args]
        name = self.tmp()
        self.ops += 1
        if k == "add":
            self.lines.append(f"const T {name} = {args[0]} + {args[1]};")
        elif k == "mul":
            self.lines.append(f"const T {name} = {args[0]} * {args[1]};")
        else:  # fma: a*b + c
            self.lines.append(f"const T {name} = fma({args[0]}, {args[1]}, {args[2]});")
        return name


def _monomial_program(polys) -> tuple:
    """Shared-monomial evaluation of a kernel's weight polynomials.

    Every distinct monomial of the kernel (over all g / t_num) is computed once, each from
    an already computed monomial times one coordinate; each polynomial is then an FMA
    chain over (constant coefficient, monomial).  For the box-spline plans this needs
    fewer operations than per-polynomial greedy Horner (e.g. bcc_quintic_rd: 42 monomials +
    316 terms vs 538 Horner ops per coset) at the same float32 accuracy (~1e-7).
    Returns (lines, {exps: name}, ops)."""
    need = set()
    for q in polys:
        for e in q.terms:
            if sum(e):
                need.add(tuple(e))
    have = {(0, 0, 0): None}
    lines = []
    ops = 0

    def name(e):
        return "m_" + "".join(str(v) for v in e)

    def build(e):
        nonlocal ops
        if e in have:
            return
        # parent: lower the exponent of the largest coordinate power (keeps chains short)
        i = max(range(3), key=lambda j: (e[j], -j))
        parent = tuple(v - (1 if j == i else 0) for j, v in enumerate(e))
        build(parent)
        if have[parent] is None:
            lines.append(f"const T {name(e)} = y{i};")
        else:
            lines.append(f"const T {name(e)} = {name(parent)} * y{i};")
            ops += 1
        have[e] = name(e)

    for e in sorted(need, key=lambda t: (sum(t), t)):
        build(e)
    return lines, have, ops


def _poly_expr(poly, have, lines, ops_box, tag) -> str:
    """Emit `const T tag = c0 + sum_k c_k * m_k` as an FMA chain; returns the value name."""
    terms = sorted(poly.terms.items(), key=lambda kv: (-sum(kv[0]), kv[0]))
    if not terms:
        return "T(0)"
    const = poly.terms.get((0, 0, 0))
    var_terms = [(e, c) for e, c in terms if sum(e)]
    if not var_terms:
        return _lit(const)
    acc = _lit(const) if const is not None else None
    for e, c in var_terms:
        m = have[tuple(e)]
        if acc is None:
            acc = f"{_lit(c)} * {m}" if c != 1 else m
            ops_box[0] += 1 if c != 1 else 0
        else:
            acc = f"fma({_lit(c)}, {m}, {acc})"
            ops_box[0] += 1
    lines.append(f"const T {tag} = {acc};")
    return tag


def _group_body(g, d: int, gname: str, tnames: list, body_lines: list, ops: list) -> list:
    """One fetch group's block: weight lines, then the (software-merged) fetch and accumulate."""
    body = ["    {"] + [f"        {ln}" for ln in body_lines]
    sd = [tuple(v // d for v in site) for site in g.sites]
    ns = len(g.span_axes)
    if ns == 0:
        body.append(f"        acc = fma({gname}, f.get({sd[0][0]}, {sd[0][1]}, {sd[0][2]}), acc);")
        ops[0] += 1
    elif ns == 1:  # exact fetchers: g*c0 + t_num*(c1 - c0); the texture fetcher: one filtered fetch
        body.append(f"        acc = f.lerp2(acc, {gname}, {tnames[0]}, {sd[0][0]}, {sd[0][1]}, {sd[0][2]}, "
                    f"{sd[1][0]}, {sd[1][1]}, {sd[1][2]});")
        ops[0] += 3
    else:
        body.append(f"        const T gz = {gname};")
        body.append("        const T rg = gz == T(0) ? T(0) : T(1) / gz;")
        for j in range(ns):
            body.append(f"        const T t{j} = gz == T(0) ? T(0.5) : {tnames[j]} * rg;")
        for c in range(1 << ns):
            body.append(f"        T v{c} = f.get({sd[c][0]}, {sd[c][1]}, {sd[c][2]});")
        for j in range(ns):
            step = 1 << j
            for c in range(0, 1 << ns, 2 * step):
                body.append(f"        v{c} = fma(t{j}, v{c + step} - v{c}, v{c});")
                ops[0] += 2
        body.append("        acc = fma(gz, v0, acc);")
        ops[0] += 1 + ns
    body.append("    }")
    return body


def _kernel_function(plan: EvaluationPlan, kidx: int, d: int) -> tuple:
    kern = plan.kernels[kidx]
    polys = [g.g for g in kern.groups] + [t for g in kern.groups for t in g.t_nums]
    mono_lines, have, mono_ops = _monomial_program(polys)
    out = [
        "template <typename T, class F>",
        f"__device__ __forceinline__ T kernel{kidx}(const T y0, const T y1, const T y2, const F& f) {{",
        "    (void)y0; (void)y1; (void)y2;",
    ]
    out += [f"    {ln}" for ln in mono_lines]
    out.append("    T acc = T(0);")
    ops = [mono_ops]
    for gi, g in enumerate(kern.groups):
        body_lines = []
        gname = _poly_expr(g.g, have, body_lines, ops, f"g{gi}")
        tnames = [_poly_expr(t, have, body_lines, ops, f"tn{gi}_{j}") for j, t in enumerate(g.t_nums)]
        out.extend(_group_body(g, d, gname, tnames, body_lines, ops))
    out.append("    return acc;")
    out.append("}")
    return out, ops[0]


def _plane_expr(normal) -> str:
    terms = []
    for i, n in enumerate(normal):
        if n == 0:
            continue
        if n == 1:
            terms.append(f"xp{i}")
        elif n == -1:
            terms.append(f"(-xp{i})")
        else:
            terms.append(f"(R({float(n)!r}) * xp{i})")
    if not terms:
        return "0.0"
    expr = terms[0]
    for t in terms[1:]:
        expr = f"({expr} + {t})"
    return expr


def weight_flops(plan: EvaluationPlan) -> list:
    """Per kernel: floating-point ops of one coset's generated weight program (shared
    monomials + FMA chains + group merges), as emitted by generate_plan_source."""
    return [_kernel_function(plan, k, plan.diag[0])[1] for k in range(plan.K)]


def affine_tables(plan: EvaluationPlan):
    """Weight programs folded into the coset frame, for plans whose weight polynomials are
    all affine (degree <= 1), K = 1 and r <= 64 (bcc_linear_rd).

    Per plane code q in [0, r) with class c = sigma[q] (class 0 for the sentinel, which is
    flagged, runtime.py:380-381), every polynomial p(y) of the kernel with y = T_c xp - t_c
    (runtime.py:385) is the affine form A . xp + C.  T_c is a signed permutation and t_c
    integral, so A and C are small dyadic rationals, exact in float32, and evaluating
    A . xp + C by an FMA chain rounds exactly where y_i = +-xp_j - t_i did.  The per-class
    transform (perm / sign decode + selects) disappears from the per-point program.
    Returns (polys per q: [[(A0, A1, A2, C), ...] * r], sentinel mask) or None."""
    if plan.K != 1 or plan.r > 64 or plan.M > 8:
        return None
    polys = []
    for g in plan.kernels[0].groups:
        polys.append(g.g)
        polys.extend(g.t_nums)
    if len(polys) > 8 or any(q.degree() > 1 for q in polys):
        return None
    rows, mask = [], 0
    for q in range(plan.r):
        c = plan.sigma[q]
        if c < 0:
            mask |= 1 << q
            c = 0
        ct = plan.classes[c]
        T = [[Fraction(v) for v in row] for row in ct.T]
        t = [Fraction(v) for v in ct.t]
        row = []
        for poly in polys:
            A = [Fraction(0)] * 3
            C = Fraction(poly.terms.get((0, 0, 0), 0))
            for e, coef in poly.terms.items():
                if sum(e) == 0:
                    continue
                i = e.index(1)
                for j in range(3):
                    A[j] += Fraction(coef) * T[i][j]
                C -= Fraction(coef) * t[i]
            vals = A + [C]
            # exact in binary16: the table is stored as half2 pairs (one LDS.128 per two polys)
            if any(float(np.float16(float(v))) != v for v in vals):
                return None
            row.append(tuple(vals))
        rows.append(row)
    return rows, mask


def _affine_kernel_function(plan: EvaluationPlan, d: int) -> tuple:
    kern = plan.kernels[0]
    out = [
        "__device__ __forceinline__ float2 half2_bits(unsigned w) {",
        "    __half2 v;",
        "    memcpy(&v, &w, 4);",
        "    return __half22float2(v);",
        "}",
        "",
        "template <typename T, class F>",
        "__device__ __forceinline__ T kernel_aff(const T xq0, const T xq1, const T xq2, const uint4* co, const F& f) {",
        "    T acc = T(0);",
    ]
    ops = [0]
    p = 0

    def aff(tag):
        nonlocal p
        lines = []
        if p % 2 == 0:
            lines.append(f"const uint4 h{p // 2} = co[{p // 2}];")
        w = ("x", "y") if p % 2 == 0 else ("z", "w")
        lines.append(f"const float2 a{p} = half2_bits(h{p // 2}.{w[0]}), b{p} = half2_bits(h{p // 2}.{w[1]});")
        lines.append(f"const T {tag} = fma(T(b{p}.x), xq2, fma(T(a{p}.y), xq1, fma(T(a{p}.x), xq0, T(b{p}.y))));")
        p += 1
        ops[0] += 3
        return lines

    for gi, g in enumerate(kern.groups):
        body_lines = aff(f"g{gi}")
        tnames = []
        for j in range(len(g.t_nums)):
            body_lines += aff(f"tn{gi}_{j}")
            tnames.append(f"tn{gi}_{j}")
        out.extend(_group_body(g, d, f"g{gi}", tnames, body_lines, ops))
    out.append("    return acc;")
    out.append("}")
    return out, ops[0], p


def _affine_eval_source(plan: EvaluationPlan, rows, mask, min_blocks: int) -> str:
    """Eval<T> of an affine plan: q -> per-(coset, q) tile record + per-q coefficients."""
    npoly = len(rows[0])
    nvec = (npoly + 1) // 2

    def h(v):
        return int(np.array([float(v)], dtype=np.float16).view(np.uint16)[0])

    vecs = []
    for row in rows:
        words = []
        for a0, a1, a2, c in list(row) + [(0, 0, 0, 0)] * (2 * nvec - npoly):
            words += [h(a0) | h(a1) << 16, h(a2) | h(c) << 16]
        vecs += ["{" + ", ".join(f"0x{w:08x}u" for w in words[4 * i:4 * i + 4]) + "}" for i in range(nvec)]
    flat = ",\n    ".join(vecs)
    return f"""constexpr int kNP = {npoly};
constexpr int kNV = {nvec};  // uint4 per q: two polynomials as half2 (A0, A1), (A2, C) each
constexpr unsigned long long kSentinel = {mask}ull;  // bit q: sigma[q] < 0
// per q: the kernel's polynomials as (A0, A1, A2, C) in the coset frame xp (class sigma[q]),
// binary16 (every value is a small dyadic rational, exact)
__device__ const uint4 kAff[kR * kNV] = {{
    {flat}
}};

template <typename T>
struct Eval {{
    static constexpr int kMinBlocks = {min_blocks};
    static constexpr int kTrecBytes = kM * kR * 16 + kR * kNV * 16;
    static constexpr bool kSig = false;
    template <typename U>
    static constexpr int vec_width() {{
        return 0;
    }}
    // per-(coset, q) tile address records {{coef of site/d component 0, 1, 2; pib/d offset}} of
    // class max(sigma[q], 0), then the per-q coefficient table (computed per tile)
    __device__ static void tile_records(const EvalArgs<T>& a, const TileGeom& g, const unsigned char* tables,
                                        int4* trec, int tid) {{
        const int* sigma = reinterpret_cast<const int*>(tables + kSigOff);
        const uint4* cls_tab = reinterpret_cast<const uint4*>(tables + kClsOff);
        for (int idx = tid; idx < kM * kR; idx += kThreads) {{
            const int k = idx / kR, q = idx - k * kR;
            const uint4 rec = cls_tab[max(sigma[q], 0)];
            const int st[3] = {{g.ex[k][1] * g.ex[k][2], g.ex[k][2], 1}};
            int cf[3] = {{0, 0, 0}}, z = 0;
#pragma unroll
            for (int i = 0; i < 3; ++i) {{
                const int rho = (int)((rec.x >> (13 + 2 * i)) & 3u);
                const int tau = ((rec.x >> (19 + i)) & 1u) ? -1 : 1;
                const int pb = (int)((rec.x >> (22 + 3 * i)) & 7u) - 4;
                cf[rho] = tau * st[i];
                z += pb * st[i];
            }}
            trec[idx] = make_int4(cf[0], cf[1], cf[2], z);
        }}
        uint4* co = reinterpret_cast<uint4*>(trec + kM * kR);
        for (int idx = tid; idx < kR * kNV; idx += kThreads) co[idx] = kAff[idx];
    }}
    template <class F, class Ctx>
    __device__ __forceinline__ static T eval(const T x[3], F& f, const Ctx& ctx) {{
        const EvalArgs<T>& a = *ctx.a;
        const int* sigma = sigma_of(ctx);
        bool fast = false;
        float frac[3] = {{0.f, 0.f, 0.f}};
        if constexpr (sizeof(T) == 4) {{
            const float m = fminf(fminf(fabsf(x[0]), fabsf(x[1])), fabsf(x[2]));
            const float M = fmaxf(fmaxf(fabsf(x[0]), fabsf(x[1])), fabsf(x[2]));
            fast = m >= kFastLo && M < kFastHi;
#pragma unroll
            for (int i = 0; i < 3; ++i) frac[i] = (float)x[i] - floorf((float)x[i]);
        }}
        T total = T(0);
#pragma unroll
        for (int k = 0; k < kM; ++k) {{
            int cell[3], q;
            T xq[3];
            if (fast) {{
                float xp[3];
                frame_fast(frac, ctx.X, k, cell, xp);
                q = plane_code<float>(xp[0], xp[1], xp[2]) % kR;
#pragma unroll
                for (int i = 0; i < 3; ++i) xq[i] = (T)xp[i];
            }} else {{
                double xp[3];
                frame_f64<T>(x, k, cell, xp);
                q = plane_code<double>(xp[0], xp[1], xp[2]) % kR;
#pragma unroll
                for (int i = 0; i < 3; ++i) xq[i] = (T)xp[i];
            }}
            ctx.err |= (int)((kSentinel >> q) & 1ull);  // sentinel (runtime.py:380-381): evaluated as class 0
            if (a.dbg) write_dbg(a.dbg, ctx.index, kM, k, sigma[q], cell);  // raw class, -1 for the sentinel
            const uint4* co;
            if constexpr (F::kIsTile) {{
                const int4 tr = ctx.trec[k * kR + q];
                f.a0 = ctx.cbase[k] + cell[0] * ctx.st0[k] + cell[1] * ctx.st1[k] + cell[2] + tr.w;
                f.c0 = tr.x;
                f.c1 = tr.y;
                f.c2 = tr.z;
                co = reinterpret_cast<const uint4*>(ctx.trec + kM * kR) + q * kNV;
            }} else {{
                const uint4 rec = reinterpret_cast<const uint4*>(ctx.tables + kClsOff)[max(sigma[q], 0)];
                int rho[3], tau[3], base[3];
#pragma unroll
                for (int i = 0; i < 3; ++i) {{
                    rho[i] = (int)((rec.x >> (13 + 2 * i)) & 3u);
                    tau[i] = ((rec.x >> (19 + i)) & 1u) ? -1 : 1;
                    base[i] = cell[i] + (int)((rec.x >> (22 + 3 * i)) & 7u) - 4;
                }}
                bind(f, a, *ctx.geom, k, base, rho, tau);
                co = kAff + q * kNV;
            }}
            total += kernel_aff<T>(xq[0], xq[1], xq[2], co, f);
        }}
        return total;
    }}
}};
"""


def _word_bits(plan: EvaluationPlan) -> int:
    """Bits per coset class in a 32-bit class word (all-ones = sigma sentinel)."""
    if plan.M * 8 <= 32 and plan.N < 255:
        return 8
    if plan.M * 16 <= 32 and plan.N < 65535:
        return 16
    return 0


def _word_class(plan: EvaluationPlan) -> str:
    b = _word_bits(plan) or 8
    m = (1 << b) - 1
    return f"""    static constexpr int kWordBits = {b};
    __device__ __forceinline__ static int word_class(unsigned word, int k) {{
        const unsigned b = (word >> ({b} * k)) & {m:#x}u;
        return b == {m:#x}u ? -1 : (int)b;
    }}
"""


def _signature_methods(plan: EvaluationPlan) -> str:
    """Kernel-signature support for K > 1 plans (brick_kernel_sig, sp_common.cuh): the raw
    classes of all cosets packed in one word, and the point's signature = its kernel id per
    coset in base K; the driver groups a brick's points by signature so that warps run one
    kernel per coset instead of every kernel that occurs among their lanes."""
    return f"""    static constexpr bool kSig = true;
    static constexpr int kSigCount = {len(set(kernel_programs(plan))) ** plan.M};
    static constexpr int kProgCount = {len(set(kernel_programs(plan)))};
    static constexpr int kMC = kM;
    static constexpr int kSigSeg = {_sig_segment(plan)};  // points per signature-sort segment
""" + _word_class(plan) + """    template <class Ctx>
    __device__ __forceinline__ static unsigned classify_word(const T x[3], const Ctx& ctx) {
        const int* sigma = sigma_of(ctx);
        float frac[3] = {0.f, 0.f, 0.f};
        const bool fast = fast_frame(x, frac);
        if constexpr (kCube) {  // all cosets' classes from the unit-cube table
            if (fast) return reinterpret_cast<const unsigned*>(ctx.tables + kCubeOff)[cube_code(frac, ctx.X)];
        }
        unsigned w = 0;
#pragma unroll
        for (int k = 0; k < kM; ++k) {
            int cell[3], raw;
            if (fast) {
                float xp[3];
                frame_fast(frac, ctx.X, k, cell, xp);
                raw = class_of<float>(xp, sigma);
            } else {
                double xp[3];
                frame_f64<T>(x, k, cell, xp);
                raw = class_of<double>(xp, sigma);
            }
            w |= ((unsigned)raw & ((1u << kWordBits) - 1u)) << (kWordBits * k);
        }
        return w;
    }
    // class word and signature together: fast-domain points read both from the cube tables
    template <class Ctx>
    __device__ __forceinline__ static int classify_key(const T x[3], const Ctx& ctx, unsigned& word) {
        if constexpr (kCube && kCubeSig) {
            float frac[3] = {0.f, 0.f, 0.f};
            if (fast_frame(x, frac)) {
                const int code = cube_code(frac, ctx.X);
                word = reinterpret_cast<const unsigned*>(ctx.tables + kCubeOff)[code];
                return (int)ctx.tables[kCubeSigOff + code];
            }
        }
        word = classify_word(x, ctx);
        return signature(word, ctx.tables);
    }
    __device__ __forceinline__ static int signature(unsigned word, const unsigned char* tables) {
        const uint4* cls_tab = reinterpret_cast<const uint4*>(tables + kClsOff);
        int sig = 0;
#pragma unroll
        for (int k = 0; k < kM; ++k) {
            const int kern = (int)(cls_tab[max(word_class(word, k), 0)].x & 15u);
            sig = sig * """ + str(len(set(kernel_programs(plan)))) + """ + """ + _prog_select(plan) + """;  // program id
        }
        return sig;
    }
"""


def _shift_select(plan: EvaluationPlan) -> str:
    """Body of shift_i(k, i): nested selects over the plan's coset shifts."""
    def axis(sh):
        return f"(i == 0 ? {int(sh[0])} : (i == 1 ? {int(sh[1])} : {int(sh[2])}))"
    expr = axis(plan.shifts[-1])
    for k in range(plan.M - 2, -1, -1):
        expr = f"(k == {k} ? {axis(plan.shifts[k])} : {expr})"
    return f"    return {expr};"


def kernel_programs(plan: EvaluationPlan) -> list:
    """Program id per kernel: kernels whose generated weight programs are identical share one
    (fcc_voronoi1's kernels 0 and 1), so the coset-item driver groups them together."""
    progs, ids = {}, []
    for k in range(plan.K):
        lines, _ = _kernel_function(plan, k, plan.diag[0])
        key = "\n".join(lines).replace(f"kernel{k}(", "kernelX(")
        ids.append(progs.setdefault(key, len(progs)))
    return ids


def _prog_select(plan: EvaluationPlan) -> str:
    """Program id of kernel `kern`: the identity; for many kernels a bit field of one packed
    constant (a shift and a mask instead of a K-deep select chain: bcc_voronoi1, K = 14,
    31.5 -> 39.7 Gpts/s); a short select chain for few (fcc_voronoi1, K = 4: the chain is 3 %
    faster than the shift)."""
    ids = kernel_programs(plan)
    if ids == list(range(plan.K)):
        return "kern"
    width = max(1, (max(ids)).bit_length())
    if plan.K <= 5:
        width = 99  # select chain
    packed = 0
    for k, pid in enumerate(ids):
        packed |= pid << (width * k)
    if width * plan.K <= 32:
        return f"(int)(({packed:#x}u >> ({width} * kern)) & {(1 << width) - 1}u)"
    if width * plan.K <= 64:
        return f"(int)(({packed:#x}ull >> ({width} * kern)) & {(1 << width) - 1}ull)"
    expr = str(ids[-1])
    for k in range(plan.K - 2, -1, -1):
        expr = f"(kern == {k} ? {ids[k]} : {expr})"
    return expr


# ---------------------------------------------------------------------------------------
# Unit-cube classification.  With X = floor(x), u = x - X in [0,1)^3 and d in {1, 2}, coset
# k's frame is xp = u + m_k with m_k = (X - l_k) mod d (the parity of X), so every plane test
# n.xp >= off of the plan is n.u >= off - n.m_k: for a normal in {-1,0,1}^3 either constant
# (c <= min n.u or c >= sup n.u) or one of a few "genuine" tests n.u >= c.  The classes of ALL
# cosets are therefore a function of (parity of X, how many thresholds each normal's n.u
# reaches): a table of d^3 * prod(thresholds + 1) class words, built here in exact
# arithmetic from the plan's own planes and sigma (runtime.py:374-379), replaces the M x Q
# plane tests, M modulo reductions and M sigma lookups by ~10 float compares and one shared-
# memory load.  Fast-domain points only (the sums n.u are exact in float32 there).

CUBE_MAX_CODES = 8192


def cube_tests(plan: EvaluationPlan):
    """[(normal, [thresholds])] of the genuine unit-cube tests, or None when the plan does not
    fit the scheme (d not in {1, 2} or not equal on all axes, normals outside {-1,0,1})."""
    d = plan.diag[0]
    if any(v != d for v in plan.diag) or d not in (1, 2) or plan.s != 3:
        return None
    tests = {}
    for l in plan.shifts:
        for p in product(range(d), repeat=3):
            m = [(p[i] - int(l[i])) % d for i in range(3)]
            for n, off in plan.planes:
                if any(v not in (-1, 0, 1) for v in n):
                    return None
                c = Fraction(off) - sum(int(n[i]) * m[i] for i in range(3))
                lo = sum(min(int(v), 0) for v in n)
                hi = sum(max(int(v), 0) for v in n)
                if lo < c < hi:
                    tests.setdefault(tuple(int(v) for v in n), set()).add(c)
    return [(n, sorted(t)) for n, t in sorted(tests.items())]


def cube_table(plan: EvaluationPlan, tests) -> list:
    """Class word per code (code = parity bits, then the per-normal states in mixed radix,
    first normal most significant); kWordBits per coset, all ones = sigma sentinel."""
    d = plan.diag[0]
    bits = _word_bits(plan)
    mask = (1 << bits) - 1
    radices = [len(t) + 1 for _, t in tests]
    table = []
    for p in product(range(d), repeat=3):
        for states in product(*[range(r) for r in radices]):
            state = {n: st for (n, _), st in zip(tests, states)}
            thr = {n: t for n, t in tests}
            word = 0
            for k, l in enumerate(plan.shifts):
                m = [(p[i] - int(l[i])) % d for i in range(3)]
                q = 0
                for j, (n, off) in enumerate(plan.planes):
                    nn = tuple(int(v) for v in n)
                    c = Fraction(off) - sum(nn[i] * m[i] for i in range(3))
                    lo = sum(min(v, 0) for v in nn)
                    hi = sum(max(v, 0) for v in nn)
                    if c <= lo:
                        bit = 1
                    elif c >= hi:
                        bit = 0
                    else:  # n.u >= c  <=>  state >= (index of c) + 1
                        bit = 1 if state[nn] >= thr[nn].index(c) + 1 else 0
                    q |= bit << j
                cls = plan.sigma[q % plan.r]
                word |= ((mask if cls < 0 else cls) & mask) << (bits * k)
            table.append(word)
    return table


def _cube_source(plan: EvaluationPlan, fast_lo: float):
    """(device source, table words) of the unit-cube classifier, or ("", None)."""
    tests = cube_tests(plan)
    # single-coset plans: the cube tests cost as much as the plan's own plane tests (cc_zp3:
    # 28.1 -> 26.2 Gpts/s measured with the table), so they keep the plane tests
    if (tests is None or plan.M == 1 or _word_bits(plan) == 0
            or os.environ.get("SP_CODEGEN_CUBE", "1") == "0"):
        return "", None
    d = plan.diag[0]
    ncodes = d ** 3
    for _, t in tests:
        ncodes *= len(t) + 1
    # exactness: |n.u| < max |n|_1 must stay below 2^24 ulp(kFastLo) = 2 kFastLo
    if ncodes > CUBE_MAX_CODES or max([sum(abs(v) for v in n) for n, _ in tests] + [0]) > 2 * fast_lo:
        return "", None
    lines = []
    if d == 2:
        lines.append("    int code = ((X[0] & 1) << 2) | ((X[1] & 1) << 1) | (X[2] & 1);")
    else:
        lines.append("    int code = 0;")
    for n, thr in tests:
        terms = []
        for i, v in enumerate(n):
            if v:
                terms.append(("+ " if v > 0 else "- ") + f"u[{i}]")
        expr = " ".join(terms).lstrip("+ ")
        if expr.startswith("- "):
            expr = "-" + expr[2:]
        sts = " + ".join(f"(v >= {float(c)!r}f)" for c in thr)
        lines.append(f"    {{ const float v = {expr}; code = code * {len(thr) + 1} + ({sts}); }}")
    src = f"""
// unit-cube classifier ({len(tests)} genuine tests, {ncodes} codes; see codegen.cube_tests)
constexpr bool kCube = true;
constexpr int kCubeCodes = {ncodes};
__device__ __forceinline__ int cube_code(const float u[3], const int X[3]) {{
{chr(10).join(lines)}
    return code;
}}
"""
    return src, cube_table(plan, tests)


def _smem_tables(plan: EvaluationPlan) -> int:
    """Bytes of plan tables + per-tile address records a brick CTA keeps in shared memory."""
    tests = cube_tests(plan)
    cube = 0
    if tests is not None and plan.M > 1 and _word_bits(plan) > 0:
        n = plan.diag[0] ** 3
        for _, t in tests:
            n *= len(t) + 1
        sig = n if plan.K > 1 else 0  # signature byte per code
        cube = ((n * 4 + sig + 15) // 16) * 16 if n <= CUBE_MAX_CODES else 0
    return plan.N * 16 + cube + plan.M * plan.N * 16


def _env_override(var: str, name: str, default: int) -> int:
    """Build-time tuning override: $var = "name:n,name:n" (occupancy / smem experiments)."""
    for item in filter(None, os.environ.get(var, "").split(",")):
        k, v = item.split(":")
        if k == name:
            return int(v)
    return default


def _sig_segment(plan: EvaluationPlan) -> int:
    """Signature-sort segment: 1024 points, 512 when the plan's tables are large (BCC Voronoi:
    N = 320, 20 KB cube table) so that three CTAs fit an SM (static arrays ~20 B per point)."""
    return _env_override("SP_CODEGEN_SIGSEG", plan.name, 512 if _smem_tables(plan) > 24 * 1024 else 1024)


def tile_budget_kb(plan: EvaluationPlan) -> int:
    """Shared-memory tile budget (KB) of the brick kernels: 40, lowered for plans with large
    tables so that tables + records + signature arrays + tile fit three CTAs per SM
    (228 KB / 3 - 1 KB reserved per CTA)."""
    static = _sig_segment(plan) * 20 + 2048 if plan.K > 1 else 2048
    room = (75 * 1024 - _smem_tables(plan) - static) // 1024
    budget = 40 if room >= 36 else max(20, room)  # measured: BCC Voronoi 27 KB + 512-point segments 22.4 -> 25.2
    return _env_override("SP_CODEGEN_TILEKB", plan.name, budget)


def generate_plan_source(plan: EvaluationPlan, stem: str | None = None) -> tuple:
    """(translation-unit source, stats) for one plan; `stem` names the catalog entry."""
    if not codegen_supported(plan):
        raise ValueError(f"plan {plan.name} is not supported by the code generator")
    stem = stem or plan.name
    ident = ident_of(stem)
    d = plan.diag[0]
    words = canonical_words(pack_plan(plan))
    kfuncs = []
    kflops = []
    aff = affine_tables(plan) if os.environ.get("SP_CODEGEN_AFFINE", "1") != "0" else None
    if aff is not None:
        lines, fl, _ = _affine_kernel_function(plan, d)
        kfuncs.extend(lines)
        kfuncs.append("")
        kflops.append(fl)
    else:
        for kidx in range(plan.K):
            lines, fl = _kernel_function(plan, kidx, d)
            kfuncs.extend(lines)
            kfuncs.append("")
            kflops.append(fl)
    sig_bytes = ((plan.r * 4) + 15) & ~15
    # occupancy hint (measured on B200): light programs keep 4 CTAs (<= 64 regs); heavier ones 2
    # (cc_zp3_ungrouped, 935 ops: 2 CTAs with 60 B of spills beat 1 CTA without by 14 %;
    # bcc_quintic_rd at 3 CTAs spills 236 B and loses 9 %)
    min_blocks = 4 if max(kflops) <= 64 else (2 if max(kflops) <= 1000 else 1)
    if plan.K > 1 and max(kflops) <= 128:
        min_blocks = 3  # signature driver: 80 registers, 3 CTAs/SM (measured +11 % over 2)
    # build-time override for occupancy experiments: SP_CODEGEN_MINBLOCKS="stem:n,stem:n"
    min_blocks = _env_override("SP_CODEGEN_MINBLOCKS", stem, min_blocks)
    planes = []
    for j, (n, off) in enumerate(plan.planes):
        planes.append(f"    q |= ({_plane_expr(n)} >= R({float(off)!r})) ? {1 << j} : 0;")
    # float32 exactness threshold: partial plane sums are bounded by R = max_j sum_i |n_ji| d
    # and are multiples of ulp(lo) = lo * 2^-23, so they are exact when R <= 2 lo; the frame
    # x - l, x/d, x - kk is exact for |x| >= max(1, d)
    rmax = max([sum(abs(v) for v in n) * d for n, _ in plan.planes] + [1])
    fast_lo = 1.0
    while fast_lo < max(rmax / 2.0, float(d), 1.0):
        fast_lo *= 2.0
    cube_src, cube_tab = _cube_source(plan, fast_lo) if aff is None else ("", None)
    if cube_tab is None:
        cube_src = '''
constexpr bool kCube = false;
constexpr bool kCubeSig = false;
constexpr int kCubeCodes = 0;
__device__ __forceinline__ int cube_code(const float u[3], const int X[3]) { return 0; }
'''
    else:
        # K > 1: each code's point signature (program id per coset, base P, as
        # Eval::signature computes it from the word) in a byte table after the class words,
        # so the signature-grouped driver's pass 1 is two shared loads per point
        ncodes = len(cube_tab)
        sig_codes = []
        progs = kernel_programs(plan)
        P = len(set(progs))
        bits = _word_bits(plan)
        if plan.K > 1 and P ** plan.M <= 255:
            for w in cube_tab:
                sig = 0
                for k in range(plan.M):
                    c = (w >> (bits * k)) & ((1 << bits) - 1)
                    c = 0 if c == (1 << bits) - 1 else c  # sentinel -> class 0 (max(raw, 0))
                    sig = sig * P + progs[plan.classes[c].kernel]
                sig_codes.append(sig)
            sig_codes += [0] * (-len(sig_codes) % 4)
            cube_tab = cube_tab + [sig_codes[i] | sig_codes[i + 1] << 8 | sig_codes[i + 2] << 16 | sig_codes[i + 3] << 24
                                   for i in range(0, len(sig_codes), 4)]
        cube_src += f"constexpr bool kCubeSig = {'true' if sig_codes else 'false'};\n"
        cube_src += "static const uint32_t kCubeTab[" + str(len(cube_tab)) + "] = {" + ", ".join(
            f"{w:#x}u" for w in cube_tab) + "};\n"
    if plan.K == 1:
        dispatch = "            const T acc = kernel0<T>(y0, y1, y2, f);"
    else:
        # one case per distinct weight program (identical kernels share one: no divergence
        # between lanes whose classes select different-but-identical kernels)
        progs = kernel_programs(plan)
        rep = {}
        for k, pid in enumerate(progs):
            rep.setdefault(pid, k)
        cases = "\n".join(
            f"                case {pid}: acc = kernel{k}<T>(y0, y1, y2, f); break;" for pid, k in sorted(rep.items())
        )
        dispatch = (f"            T acc = T(0);\n            const int prog = {_prog_select(plan)};\n"
                    f"            switch (prog) {{\n{cases}\n            }}")
    sig_ok = plan.K > 1 and _word_bits(plan) > 0 and len(set(kernel_programs(plan))) ** plan.M <= 1024
    sig_methods = _signature_methods(plan) if sig_ok else "    static constexpr bool kSig = false;\n" + _word_class(plan)
    if aff is not None:
        eval_src = _affine_eval_source(plan, aff[0], aff[1], min_blocks)
    else:
        eval_src = f"""template <typename T>
struct Eval {{
    static constexpr int kMinBlocks = {min_blocks};
    static constexpr int kTrecBytes = kM * kN * 16;
    template <typename U>
    static constexpr int vec_width() {{
        return 0;
    }}
    // per-(coset, class) shared-memory address records for the staged tile:
    // {{coef of site/d component 0, 1, 2; constant offset of pib/d}} (computed per tile)
    __device__ static void tile_records(const EvalArgs<T>& a, const TileGeom& g, const unsigned char* tables,
                                        int4* trec, int tid) {{
        const uint4* cls_tab = reinterpret_cast<const uint4*>(tables + kClsOff);
        for (int idx = tid; idx < kM * kN; idx += kThreads) {{
            const int k = idx / kN, c = idx - k * kN;
            const uint4 rec = cls_tab[c];
            const int st[3] = {{g.ex[k][1] * g.ex[k][2], g.ex[k][2], 1}};
            int cf[3] = {{0, 0, 0}}, z = 0;
#pragma unroll
            for (int i = 0; i < 3; ++i) {{
                const int rho = (int)((rec.x >> (13 + 2 * i)) & 3u);
                const int tau = ((rec.x >> (19 + i)) & 1u) ? -1 : 1;
                const int pb = (int)((rec.x >> (22 + 3 * i)) & 7u) - 4;
                cf[rho] = tau * st[i];
                z += pb * st[i];
            }}
            trec[idx] = make_int4(cf[0], cf[1], cf[2], z);
        }}
    }}
    // float32 points: exact float32 frame when |x_i| in [kFastLo, kFastHi) (see kFastLo)
    __device__ __forceinline__ static bool fast_frame(const T x[3], float frac[3]) {{
        bool fast = false;
        if constexpr (sizeof(T) == 4) {{
            const float m = fminf(fminf(fabsf(x[0]), fabsf(x[1])), fabsf(x[2]));
            const float M = fmaxf(fmaxf(fabsf(x[0]), fabsf(x[1])), fabsf(x[2]));
            fast = m >= kFastLo && M < kFastHi;
#pragma unroll
            for (int i = 0; i < 3; ++i) frac[i] = (float)x[i] - floorf((float)x[i]);
        }}
        return fast;
    }}
{sig_methods}
    template <class F, class Ctx>
    __device__ __forceinline__ static T eval(const T x[3], F& f, const Ctx& ctx) {{
        return eval_impl<false>(x, 0u, f, ctx);
    }}
    // classes given (kWordBits per coset, all ones = sentinel), e.g. by classify_word: no plane tests
    template <class F, class Ctx>
    __device__ __forceinline__ static T eval_word(const T x[3], unsigned word, F& f, const Ctx& ctx) {{
        return eval_impl<true>(x, word, f, ctx);
    }}
    // one coset's contribution (runtime.py:384-407 for coset k): KC >= 0 a compile-time coset
    // (unrolled loop of eval_impl), KC < 0 a runtime one (coset-item driver; tile geometry
    // from shared memory).  Same operations either way: identical values.
    template <bool kWord, int KC, class F, class Ctx>
    __device__ __forceinline__ static T eval_coset(const T x[3], bool fast, const float frac[3], unsigned word, int k,
                                                   F& f, const Ctx& ctx) {{
        const EvalArgs<T>& a = *ctx.a;
        const int* sigma = sigma_of(ctx);
        const uint4* cls_tab = reinterpret_cast<const uint4*>(ctx.tables + kClsOff);
        if (KC >= 0) k = KC;
        int cell[3];
        T yy[3];
        uint4 rec;
        int raw;
        if (fast) {{
            float xp[3];
            frame_fast(frac, ctx.X, k, cell, xp);
            raw = kWord ? word_class(word, k) : class_of<float>(xp, sigma);
            y_of<float, T>(xp, raw, cls_tab, ctx.err, yy, rec);
        }} else {{
            double xp[3];
            frame_f64<T>(x, k, cell, xp);
            raw = kWord ? word_class(word, k) : class_of<double>(xp, sigma);
            y_of<double, T>(xp, raw, cls_tab, ctx.err, yy, rec);
        }}
        write_dbg(a.dbg, ctx.index, kM, k, raw, cell);  // raw class: -1 for the sentinel
        const int c = max(raw, 0);
        const int kern = (int)(rec.x & 15u);
        (void)kern;
        const T y0 = yy[0], y1 = yy[1], y2 = yy[2];
        if constexpr (F::kIsTile) {{
            const int4 tr = ctx.trec[k * kN + c];
            if (KC >= 0)
                f.a0 = ctx.cbase[KC < 0 ? 0 : KC] + cell[0] * ctx.st0[KC < 0 ? 0 : KC] +
                       cell[1] * ctx.st1[KC < 0 ? 0 : KC] + cell[2] + tr.w;
            else
                f.a0 = ctx.geom->cbase[k] + cell[0] * ctx.geom->st0[k] + cell[1] * ctx.geom->st1[k] + cell[2] + tr.w;
            f.c0 = tr.x;
            f.c1 = tr.y;
            f.c2 = tr.z;
        }} else {{
            int rho[3], tau[3], base[3];
#pragma unroll
            for (int i = 0; i < 3; ++i) {{
                rho[i] = (int)((rec.x >> (13 + 2 * i)) & 3u);
                tau[i] = ((rec.x >> (19 + i)) & 1u) ? -1 : 1;
                base[i] = cell[i] + (int)((rec.x >> (22 + 3 * i)) & 7u) - 4;
            }}
            bind(f, a, *ctx.geom, k, base, rho, tau);
        }}
{dispatch}
        return acc;
    }}
    template <bool kWord, class F, class Ctx>
    __device__ __forceinline__ static T sum_cosets(const T x[3], bool fast, const float frac[3], unsigned word, F& f,
                                                   const Ctx& ctx) {{
        T total = T(0);
        total += eval_coset<kWord, 0>(x, fast, frac, word, 0, f, ctx);
{''.join(f"        total += eval_coset<kWord, {k}>(x, fast, frac, word, {k}, f, ctx);" + chr(10) for k in range(1, plan.M))}        return total;
    }}
    template <bool kWord, class F, class Ctx>
    __device__ __forceinline__ static T eval_impl(const T x[3], unsigned word, F& f, const Ctx& ctx) {{
        float frac[3] = {{0.f, 0.f, 0.f}};
        const bool fast = fast_frame(x, frac);
        if constexpr (!kWord && kCube) {{  // fast-domain points: classes from the unit-cube table
            if (fast)
                return sum_cosets<true>(x, true, frac,
                                        reinterpret_cast<const unsigned*>(ctx.tables + kCubeOff)[cube_code(frac, ctx.X)],
                                        f, ctx);
        }}
        return sum_cosets<kWord>(x, fast, frac, word, f, ctx);
    }}
    // coset-item driver (eval_brick_items): program id of coset k's kernel for class word
    // `word` (identical kernel programs share an id) and the per-coset evaluation with a
    // runtime coset index
    __device__ __forceinline__ static int item_kernel(unsigned word, int k, const unsigned char* tables) {{
        const uint4* cls_tab = reinterpret_cast<const uint4*>(tables + kClsOff);
        const int kern = (int)(cls_tab[max(word_class(word, k), 0)].x & 15u);
        return {_prog_select(plan)};
    }}
    template <class F, class Ctx>
    __device__ __forceinline__ static T eval_item(const T x[3], unsigned word, int k, F& f, const Ctx& ctx) {{
        float frac[3] = {{0.f, 0.f, 0.f}};
        const bool fast = fast_frame(x, frac);
        return eval_coset<true, -1>(x, fast, frac, word, k, f, ctx);
    }}
}};

"""
    src = f"""// GENERATED by paper_2102_08514_b200/codegen.py from plans/{stem}.plan.json — do not edit.
// Plan: {plan.name} on {plan.lattice_name}: s=3 M={plan.M} N={plan.N} Q={plan.Q} r={plan.r} K={plan.K}
// Weight-program flops per coset per kernel (shared monomials + FMA chains + merge): {kflops}
#include <cuda_fp16.h>

#include "../sp_launch.cuh"

namespace sp {{
namespace gen_{ident} {{

constexpr int kM = {plan.M};
constexpr int kR = {plan.r};
constexpr double kD = {float(d)!r};
constexpr double kInvD = {1.0 / d!r};
__device__ constexpr double kShift[kM][3] = {{{", ".join("{" + ", ".join(repr(float(v)) for v in sh) + "}" for sh in plan.shifts)}}};
constexpr int kSigmaBytes = {sig_bytes};

{chr(10).join(kfuncs)}
// float32 fast path: for |x_i| in [kFastLo, 2^22) the coset frame and the plane sums are
// exact in float32 (every partial sum is a multiple of ulp(kFastLo) below 2*kFastLo*2^23),
// so the classification equals the float64 one bit for bit; other points use float64.
constexpr float kFastLo = {fast_lo!r}f;
constexpr float kFastHi = 4194304.0f;
constexpr int kN = {plan.N};
constexpr int kDI = {d};
constexpr int kLog2D = {d.bit_length() - 1};
__device__ constexpr int kShiftI[kM][3] = {{{", ".join("{" + ", ".join(str(int(v)) for v in sh) + "}" for sh in plan.shifts)}}};
// coset shift l_k[i] by selects: folds to a constant for a compile-time k (unrolled coset
// loops) and stays in registers for a runtime k (coset-item driver)
__device__ __forceinline__ int shift_i(int k, int i) {{
{_shift_select(plan)}
}}
{cube_src}
// plan tables (sp_plan_create): class records | unit-cube table | sigma.  With the cube table
// only the first two are staged into shared memory (sigma serves the rare float64-frame points
// from global memory); without it all three are.
constexpr int kClsOff = 0;
constexpr int kCubeOff = kN * 16;
constexpr int kCubeSigOff = kCubeOff + kCubeCodes * 4;  // byte per code (kCubeSig)
constexpr int kSigOff = kCubeOff + (((kCubeCodes * 4) + (kCubeSig ? (kCubeCodes + 3) / 4 * 4 : 0) + 15) & ~15);
constexpr int kSmemTableBytes = kCube ? kSigOff : kSigOff + kSigmaBytes;
template <class Ctx>
__device__ __forceinline__ const int* sigma_of(const Ctx& ctx) {{
    return kCube ? reinterpret_cast<const int*>(reinterpret_cast<const unsigned char*>(ctx.a->tables) + kSigOff)
                 : reinterpret_cast<const int*>(ctx.tables + kSigOff);
}}

template <typename R>
__device__ __forceinline__ int plane_code(const R xp0, const R xp1, const R xp2) {{
    int q = 0;
{chr(10).join(planes)}
    return q;
}}

// coset frame (runtime.py:371-373), plane tests (:374-378), sigma (:379) and y = T xp - t
// (:385) for coset k, evaluated in R (float on the fast path, else double).
// class lookup + y = T xp - t from the packed class record
// y = T xp - t (runtime.py:385) from the packed record of class max(raw, 0)
template <typename R, typename T>
__device__ __forceinline__ void y_of(const R xp[3], int raw, const uint4* cls_tab, int& err, T y[3], uint4& rec) {{
    err |= raw < 0;  // sigma sentinel (runtime.py:380-381): flagged, evaluated as class 0
    const int c = max(raw, 0);
    rec = cls_tab[c];
    const float tt[3] = {{__uint_as_float(rec.y), __uint_as_float(rec.z), __uint_as_float(rec.w)}};
#pragma unroll
    for (int i = 0; i < 3; ++i) {{
        const unsigned perm = (rec.x >> (4 + 2 * i)) & 3u;  // 0, 1 or 2
        const R v01 = (perm & 1u) ? xp[1] : xp[0];
        const R v = (perm & 2u) ? xp[2] : v01;
        y[i] = (T)((((rec.x >> (10 + i)) & 1u) ? -v : v) - (R)tt[i]);
    }}
}}

// plane tests (:374-378) and sigma (:379)
template <typename R>
__device__ __forceinline__ int class_of(const R xp[3], const int* sigma) {{
    return sigma[plane_code<R>(xp[0], xp[1], xp[2]) % kR];
}}

template <typename R, typename T>
__device__ __forceinline__ int class_and_y(const R xp[3], const int* sigma, const uint4* cls_tab, int& err,
                                           T y[3], uint4& rec) {{
    const int raw = class_of<R>(xp, sigma);
    y_of<R, T>(xp, raw, cls_tab, err, y, rec);
    return raw;
}}

// float64 coset frame exactly as runtime.py:371-373 (any point)
template <typename T>
__device__ __forceinline__ void frame_f64(const T x[3], int k, int cell[3], double xp[3]) {{
#pragma unroll
    for (int i = 0; i < 3; ++i) {{
        const double xl = (double)x[i] - (double)shift_i(k, i);
        const double q = floor(xl * kInvD);  // power-of-two d: exact
        xp[i] = xl - q * kD;
        cell[i] = clamp_cell(q);
    }}
}}

// float32 fast frame from X = floor(x) and frac = x - X (exact): for integer l and d = 2^j,
// floor((x-l)/d) = (X-l) >> j and xp = frac + ((X-l) & (d-1)), exactly the float64 values
// for |x| >= kFastLo (frac + p needs no rounding there).
__device__ __forceinline__ void frame_fast(const float frac[3], const int X[3], int k, int cell[3], float xp[3]) {{
#pragma unroll
    for (int i = 0; i < 3; ++i) {{
        const int xm = X[i] - shift_i(k, i);
        cell[i] = xm >> kLog2D;
        const int p = xm & (kDI - 1);
        xp[i] = kDI == 1 ? frac[i] : (kDI == 2 ? (p ? frac[i] + 1.0f : frac[i]) : frac[i] + (float)p);
    }}
}}

template <typename T>
__device__ __forceinline__ int classify_f64(const T x[3], int k, const int* sigma, const uint4* cls_tab, int& err,
                                            int cell[3], T y[3], uint4& rec) {{
    double xp[3];
    frame_f64<T>(x, k, cell, xp);
    return class_and_y<double, T>(xp, sigma, cls_tab, err, y, rec);
}}

template <typename T>
__device__ __forceinline__ int classify_fast(const float frac[3], const int X[3], int k, const int* sigma,
                                             const uint4* cls_tab, int& err, int cell[3], T y[3], uint4& rec) {{
    float xp[3];
    frame_fast(frac, X, k, cell, xp);
    return class_and_y<float, T>(xp, sigma, cls_tab, err, y, rec);
}}

{eval_src}static const uint64_t kBlob[{len(words)}] = {{
{_format_words(words)}
}};

}}  // namespace gen_{ident}
}}  // namespace sp

extern const sp::GenEntry kGen_{ident} = {{
    "{stem}",
    sp::gen_{ident}::kBlob,
    {len(words)},
    &sp::launch_eval<float, sp::gen_{ident}::Eval<float>>,
    &sp::launch_eval<double, sp::gen_{ident}::Eval<double>>,
    &sp::occupancy_blocks<float, sp::gen_{ident}::Eval<float>>,
    &sp::occupancy_blocks<double, sp::gen_{ident}::Eval<double>>,
    &sp::launch_bricks<float, sp::gen_{ident}::Eval<float>>,
    &sp::launch_bricks<double, sp::gen_{ident}::Eval<double>>,
    &sp::occupancy_bricks<float, sp::gen_{ident}::Eval<float>>,
    &sp::occupancy_bricks<double, sp::gen_{ident}::Eval<double>>,
    sp::gen_{ident}::Eval<float>::kTrecBytes,
    &sp::launch_tex<sp::gen_{ident}::Eval<float>>,
    {"sp::gen_" + ident + "::kCubeTab" if cube_tab is not None else "nullptr"},
    {len(cube_tab) if cube_tab is not None else 0},
    sp::gen_{ident}::kSmemTableBytes,
    {tile_budget_kb(plan)},
}};
"""
    return src, {"ident": ident, "flops_per_coset": kflops, "words": len(words), "affine": aff is not None}


def _format_words(words: list) -> str:
    lines = []
    for i in range(0, len(words), 4):
        lines.append("    " + ", ".join(f"0x{w:016x}ull" for w in words[i : i + 4]) + ",")
    return "\n".join(lines)


def generate_registry(idents: list) -> str:
    decls = "\n".join(f"extern const sp::GenEntry kGen_{i};" for i in idents)
    entries = ", ".join(f"&kGen_{i}" for i in idents) or "nullptr"
    return f"""// GENERATED by paper_2102_08514_b200/codegen.py — registry of plan-specialised kernels.
{decls}
static const sp::GenEntry* const kGenerated[] = {{{entries}}};
"""


def write_generated(plans: list, out_dir: str) -> list:
    """Write one TU per supported (stem, plan) + registry.inc; returns the TU paths."""
    os.makedirs(out_dir, exist_ok=True)
    idents, paths = [], []
    for stem, plan in plans:
        if not codegen_supported(plan):
            continue
        src, stats = generate_plan_source(plan, stem)
        path = os.path.join(out_dir, f"plan_{stats['ident']}.cu")
        _write_if_changed(path, src)
        idents.append(stats["ident"])
        paths.append(path)
    _write_if_changed(os.path.join(out_dir, "registry.inc"), generate_registry(idents))
    # drop stale TUs of plans no longer in the catalog
    for f in os.listdir(out_dir):
        if f.startswith("plan_") and f.endswith(".cu") and os.path.join(out_dir, f) not in paths:
            os.remove(os.path.join(out_dir, f))
    return paths


def _write_if_changed(path: str, text: str) -> None:
    if os.path.exists(path) and open(path).read() == text:
        return
    with open(path, "w") as fh:
        fh.write(text)
