"""Generates paper_2206_13164_b200/csrc/gen/simplex_gen.cuh: straight-line
FP64 code for the multi-index operations of the moment method, one
specialisation per moment order M.

Every operation of the hot path that mixes coefficients walks a chain along
one velocity axis of the graded-lex simplex {|alpha| <= M}
(multi_index.hpp:31-52).  Emitting those chains with compile-time positions
turns each term into one shared-memory load with an immediate offset plus
one FMA: no index arithmetic, no tables, no predication at run time.

A thread's vector lives in shared memory at v[k * VS] (VS = threads per
block, so the vectors of consecutive threads interleave and every access is
bank-conflict free).

Generated per M (struct Gen<M>):
  pass<d>(v, c)        in-place axis-d Toeplitz pass g_a = sum_n c_n f_{a - n e_d}
                       (one factor of the projection; see momg_device.cuh)
  half_sum<a>(L, R, Ku, Kl)
                       in place into L: out(beta) = sum_m L(beta|m) Ku[m][p] + R(beta|m) Kl[m][p]
                       (flux.cpp:58-73 with folded kernels), p = beta_a
  half_one<a>(L, K)    single-sided variant (wall outgoing flux)
  half_sr<a>(s, o, K)  single-sided, strided source -> separate output
  full_flux<a>(src, dst, un, th)
                       flux.cpp:10-27
Usage: python tools/gen_simplex.py  (writes the header; run by csrc/Makefile)
"""
import os
import sys

ORDERS = [3, 4, 5, 6, 7, 8]
SPLIT_PASS_CHAINS = False


def simplex(M):
    idx = []
    for deg in range(M + 1):
        for a1 in range(deg, -1, -1):
            for a2 in range(deg - a1, -1, -1):
                idx.append((a1, a2, deg - a1 - a2))
    return idx


def emit_order(M):
    idx = simplex(M)
    pos = {a: k for k, a in enumerate(idx)}
    N = len(idx)
    L = []
    w = L.append
    w(f"template <>\nstruct Gen<{M}> {{")
    w(f"  static constexpr int N = {N};")
    # ---------------------------------------------------------------- passes
    for d in range(3):
        w(f"  // axis-{d} Toeplitz pass, in place (pencils along axis {d})")
        w(f"  template <int VS>")
        w(f"  static __device__ __forceinline__ void pass{d}(double* __restrict__ v, const double* c) {{")
        others = [o for o in range(3) if o != d]
        pencils = {}
        for a in idx:
            key = (a[others[0]], a[others[1]])
            pencils.setdefault(key, []).append(a)
        for key, members in pencils.items():
            members.sort(key=lambda a: a[d])
            if len(members) < 2:
                continue
            ks = [pos[a] for a in members]
            w("    {")
            for j, k in enumerate(ks):
                w(f"      const double f{j} = v[{k} * VS];")
            for j in range(len(ks) - 1, 0, -1):
                expr = f"f{j}"
                for n in range(1, j + 1):
                    expr = f"fma(c[{n}], f{j - n}, {expr})"
                w(f"      v[{ks[j]} * VS] = {expr};")
            w("    }")
        w("  }")
    # ------------------------------------------------------------- half sums
    for a in range(2):
        for single in (False, True):
            name = f"half_one{a}" if single else f"half_sum{a}"
            args = "double* __restrict__ Lv, const double (&Ku)[%d][%d]" % (M + 1, M + 1) if single else \
                "double* __restrict__ Lv, const double* __restrict__ Rv, const double (&Ku)[%d][%d], const double (&Kl)[%d][%d]" % (M + 1, M + 1, M + 1, M + 1)
            w(f"  // half-space flux sum along axis {a}{' (single side)' if single else ''}, in place into Lv")
            w(f"  template <int VS>")
            w(f"  static __device__ __forceinline__ void {name}({args}) {{")
            tans = {}
            for b in idx:
                t = tuple(b[o] for o in range(3) if o != a)
                tans.setdefault(t, []).append(b)
            for t, members in tans.items():
                members.sort(key=lambda b: b[a])
                ks = [pos[b] for b in members]
                n = len(ks)  # m = 0 .. n-1 (= M - |beta_t|)
                w("    {")
                for m, k in enumerate(ks):
                    w(f"      const double l{m} = Lv[{k} * VS];")
                    if not single:
                        w(f"      const double r{m} = Rv[{k} * VS];")
                for p, k in enumerate(ks):
                    expr = "0.0"
                    for m in range(n):
                        expr = f"fma(l{m}, Ku[{m}][{p}], {expr})" if expr != "0.0" else f"l{m} * Ku[{m}][{p}]"
                        if not single:
                            expr = f"fma(r{m}, Kl[{m}][{p}], {expr})"
                    w(f"      Lv[{k} * VS] = {expr};")
                w("    }")
            w("  }")
    # half flux of one side from a strided source into a separate output
    # (register-resident band kernel): longest pencils first, so the
    # kernel entries of the long pencils die before the output fills up
    for a in range(2):
        w(f"  // single-side half-space flux along axis {a}: o = K applied to s (pencils by decreasing length)")
        w(f"  template <int VS, int VO>")
        w(f"  static __device__ __forceinline__ void half_sr{a}(const double* __restrict__ s, double* __restrict__ o, const double (&K)[{M + 1}][{M + 1}]) {{")
        tans = {}
        for b in idx:
            t = tuple(b[o] for o in range(3) if o != a)
            tans.setdefault(t, []).append(b)
        for t, members in sorted(tans.items(), key=lambda tm: -len(tm[1])):
            members.sort(key=lambda b: b[a])
            ks = [pos[b] for b in members]
            n = len(ks)
            w("    {")
            for m, k in enumerate(ks):
                w(f"      const double l{m} = s[{k} * VS];")
            for p, k in enumerate(ks):
                expr = "0.0"
                for m in range(n):
                    expr = f"fma(l{m}, K[{m}][{p}], {expr})" if expr != "0.0" else f"l{m} * K[{m}][{p}]"
                w(f"      o[{k} * VO] = {expr};")
            w("    }")
        w("  }")
    # ------------------------------------------------------------ full flux
    for a in range(2):
        w(f"  // full-space flux xi_{a} f (flux.cpp:10-27), closure drops degree M+1")
        w(f"  template <int VS, int VO = VS>")
        w(f"  static __device__ __forceinline__ void full_flux{a}(const double* __restrict__ s, double* __restrict__ o, double un, double th) {{")
        for b in idx:
            k = pos[b]
            expr = f"un * s[{k} * VS]"
            if b[a] >= 1:
                dn = list(b); dn[a] -= 1
                expr = f"fma(th, s[{pos[tuple(dn)]} * VS], {expr})"
            if sum(b) < M:
                up = list(b); up[a] += 1
                expr = f"fma({float(b[a] + 1)}, s[{pos[tuple(up)]} * VS], {expr})"
            w(f"    o[{k} * VO] = {expr};")
        w("  }")
    # Shakhov eq pattern: positions of 2 e_dd + e_d and the q components
    w("  // Shakhov equilibrium positions (collision.hpp:95-111): 3 e_d and e_d + 2 e_dd")
    sh = []
    for d in range(3):
        for dd in range(3):
            b = [0, 0, 0]; b[dd] += 2; b[d] += 1
            sh.append((pos[tuple(b)], d))
    w("  static constexpr int SHK[9] = {" + ", ".join(str(k) for k, _ in sh) + "};")
    w("  static constexpr int SHD[9] = {" + ", ".join(str(d) for _, d in sh) + "};")
    # degrees and factorials for norms
    import math
    w("  static constexpr int DEG[" + str(N) + "] = {" + ", ".join(str(sum(b)) for b in idx) + "};")
    w("  static constexpr double FACT[" + str(N) + "] = {" + ", ".join(
        repr(float(math.factorial(b[0]) * math.factorial(b[1]) * math.factorial(b[2]))) for b in idx) + "};")
    # beta = p e_a positions (in_unit of the wall flux)
    for a in range(2):
        ps = []
        for p in range(M + 1):
            b = [0, 0, 0]; b[a] = p
            ps.append(pos[tuple(b)])
        w(f"  static constexpr int AXP{a}[{M + 1}] = {{" + ", ".join(map(str, ps)) + "};")
    w("};")
    return "\n".join(L)


def main():
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "paper_2206_13164_b200", "csrc", "gen", "simplex_gen.cuh")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    body = ["// GENERATED by tools/gen_simplex.py -- do not edit.",
            "// Straight-line multi-index operations per moment order (see the generator's docstring).",
            "#pragma once", "", "namespace momg_gpu {", "", "template <int M>", "struct Gen;", ""]
    for M in ORDERS:
        body.append(emit_order(M))
        body.append("")
    body.append("}  // namespace momg_gpu")
    text = "\n".join(body) + "\n"
    if not os.path.exists(out) or open(out).read() != text:
        open(out, "w").write(text)
    print(out, len(text.splitlines()), "lines")


# ---------------------------------------------------------------------------
# Partitioned variants (split design): the same operations cut into P parts
# of balanced cost, part q executed by warp q of a face group (lane = cell).
# Vectors of the 32 cells of a segment interleave: element k of cell c at
# v[k * 32 + c].  An axis pass is split by pencils, which are disjoint element
# sets, so it runs in place; the half sums are split by the normal index p and
# write a separate output vector.  One named barrier separates passes.

def lpt(costs, P):
    parts = [[] for _ in range(P)]
    load = [0] * P
    for key, c in sorted(costs.items(), key=lambda kv: -kv[1]):
        q = load.index(min(load))
        parts[q].append(key)
        load[q] += c
    return parts


def emit_split(M, P, full=True):
    idx = simplex(M)
    pos = {a: k for k, a in enumerate(idx)}
    N = len(idx)
    L = []
    w = L.append
    w(f"template <>\nstruct Split<{M}, {P}> {{")
    # in-place axis passes of partition q: every load of the partition is
    # issued before the first store, so the smem round trips overlap (loads
    # and stores to different pencils would otherwise serialise)
    for d in range(3):
        others = [o for o in range(3) if o != d]
        pencils = {}
        for a in idx:
            pencils.setdefault((a[others[0]], a[others[1]]), []).append(a)
        costs = {k: len(v) * (len(v) + 1) // 2 + 2 * len(v) for k, v in pencils.items()}
        parts = lpt(costs, P)
        for q in range(P):
            mine = []
            for key in parts[q]:
                members = sorted(pencils[key], key=lambda a: a[d])
                ks = [pos[a] for a in members]
                if len(ks) >= 2:
                    mine.append(ks)

            def body(vec, cn, tag, guard=None):
                out = []
                for t, ks in enumerate(mine):
                    for j, k in enumerate(ks):
                        out.append(f"    const double {tag}{t}_{j} = {vec}[{k} * SPV];")
                for t, ks in enumerate(mine):
                    for j in range(len(ks) - 1, 0, -1):
                        # (splitting into odd / even chains measured slower)
                        expr = f"{tag}{t}_{j}"
                        odd = None
                        for n in range(1, j + 1):
                            if SPLIT_PASS_CHAINS and j >= 3 and n % 2 == 1:
                                odd = (f"{cn}[{n}] * {tag}{t}_{j - n}" if odd is None
                                       else f"fma({cn}[{n}], {tag}{t}_{j - n}, {odd})")
                            else:
                                expr = f"fma({cn}[{n}], {tag}{t}_{j - n}, {expr})"
                        if odd is not None:
                            expr = f"{expr} + {odd}"
                        st = f"{vec}[{ks[j]} * SPV] = {expr};"
                        out.append(f"    if ({guard}) {st}" if guard else f"    {st}")
                return out
            w(f"  static __device__ __forceinline__ void pass{d}_{q}(double* __restrict__ v, const double* c) {{")
            L.extend(body("v", "c", "f"))
            w("  }")
            # two vectors at once (project2): all loads of both first
            w(f"  static __device__ __forceinline__ void pass2{d}_{q}(double* __restrict__ a, const double* ca, bool acta, "
              f"double* __restrict__ b, const double* cb, bool actb) {{")
            la = body("a", "ca", "fa", "acta")
            lb = body("b", "cb", "fb", "actb")
            nla = sum(len(ks) for ks in mine)
            L.extend(la[:nla] + lb[:nla] + la[nla:] + lb[nla:])
            w("  }")
    if not full:  # pass-only variant (the band sweep's 16-warp normalisation)
        bounds = [round(q * N / P) for q in range(P + 1)]
        w(f"  static constexpr int KLO[{P + 1}] = {{" + ", ".join(map(str, bounds)) + "};")
        w("};")
        return "\n".join(L)
    # half sums split by the normal index p
    for a in range(2):
        tans = {}
        for b in idx:
            t = tuple(b[o] for o in range(3) if o != a)
            tans.setdefault(t, []).append(b)
        costs = {}
        for p in range(M + 1):
            costs[p] = sum(len(m) * 2 for m in tans.values() if len(m) > p)
        parts = lpt(costs, P)
        for single in (False, True):
            for q in range(P):
                name = f"half_one{a}_{q}" if single else f"half_sum{a}_{q}"
                kt = f"const double (&Ku)[{M + 1}][{M + 1}]"
                args = f"const double* __restrict__ Lv, {kt}, double* __restrict__ o" if single else \
                    f"const double* __restrict__ Lv, const double* __restrict__ Rv, {kt}, const double (&Kl)[{M + 1}][{M + 1}], double* __restrict__ o"
                w(f"  static __device__ __forceinline__ void {name}({args}) {{")
                for t, members in tans.items():
                    members = sorted(members, key=lambda b: b[a])
                    ks = [pos[b] for b in members]
                    ps = [p for p in parts[q] if p < len(ks)]
                    if not ps:
                        continue
                    w("    {")
                    for m, k in enumerate(ks):
                        w(f"      const double l{m} = Lv[{k} * SPV];")
                        if not single:
                            w(f"      const double r{m} = Rv[{k} * SPV];")
                    for p in ps:
                        # two independent FMA chains (upper: L rows, lower: R
                        # rows; single: even / odd m) halve the dependency depth
                        eu = el = None
                        for m in range(len(ks)):
                            if single and m % 2 == 1:
                                el = f"l{m} * Ku[{m}][{p}]" if el is None else f"fma(l{m}, Ku[{m}][{p}], {el})"
                            else:
                                eu = f"l{m} * Ku[{m}][{p}]" if eu is None else f"fma(l{m}, Ku[{m}][{p}], {eu})"
                            if not single:
                                el = f"r{m} * Kl[{m}][{p}]" if el is None else f"fma(r{m}, Kl[{m}][{p}], {el})"
                        expr = eu if el is None else f"{eu} + {el}"
                        w(f"      o[{ks[p]} * SPV] = {expr};")
                    w("    }")
                w("  }")
        w(f"  static constexpr int HALF_PMAX{a}[{P}] = {{" + ", ".join(str(max(p) if p else 0) for p in parts) + "};")
    # full flux split by coefficient ranges
    chunks = [list(range(N))[q::P] for q in range(P)]
    for a in range(2):
        for q in range(P):
            w(f"  static __device__ __forceinline__ void full_flux{a}_{q}(const double* __restrict__ s, double* __restrict__ o, double un, double th) {{")
            for k in chunks[q]:
                b = idx[k]
                expr = f"un * s[{k} * SPV]"
                if b[a] >= 1:
                    dn = list(b); dn[a] -= 1
                    expr = f"fma(th, s[{pos[tuple(dn)]} * SPV], {expr})"
                if sum(b) < M:
                    up = list(b); up[a] += 1
                    expr = f"fma({float(b[a] + 1)}, s[{pos[tuple(up)]} * SPV], {expr})"
                w(f"    o[{k} * SPV] = {expr};")
            w("  }")
    # contiguous coefficient ranges for element-wise work
    bounds = [round(q * N / P) for q in range(P + 1)]
    w(f"  static constexpr int KLO[{P + 1}] = {{" + ", ".join(map(str, bounds)) + "};")
    w("};")
    return "\n".join(L)


def main_split():
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "paper_2206_13164_b200", "csrc", "gen", "split_gen.cuh")
    body = ["// GENERATED by tools/gen_simplex.py -- do not edit.",
            "// Partitioned straight-line multi-index operations (split design).",
            "// SPV: element stride of the interleaved per-cell vectors (odd, so",
            "// a warp writing one cell's elements is bank-conflict free too).",
            "#pragma once", "", "#ifndef SPV", "#define SPV 33", "#endif", "",
            "namespace momg_gpu {", "", "template <int M, int P>", "struct Split;", ""]
    for M in ORDERS:
        body.append(emit_split(M, 4))
        body.append("")
    body.append("}  // namespace momg_gpu")
    text = "\n".join(body) + "\n"
    if not os.path.exists(out) or open(out).read() != text:
        open(out, "w").write(text)
    print(out, len(text.splitlines()), "lines")


if __name__ == "__main__":
    main()
    main_split()
