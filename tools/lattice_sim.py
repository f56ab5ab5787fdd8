"""Host simulation of the interval-union engine's lattice decomposition
(csrc/k_sets.cu: box_lattice / normalize / cover_warp / emit_lattice) for
one wave or block unit — to inspect lattice counts, monotonicity and
interval counts per unit without a GPU.  Debug tool, not product code.

usage: python tools/lattice_sim.py C4 <config index> [field]
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2107_01143_b200 import workloads as W  # noqa: E402
from paper_2107_01143_b200.gvo.expr import affine_parts  # noqa: E402
from paper_2107_01143_b200.gvo.footprint import blocks_per_wave  # noqa: E402

COORDS = ("tidx", "tidy", "tidz", "bidx", "bidy", "bidz")


def coefs(k):
    out = []
    for a in k.accesses:
        p = affine_parts(a.expr, k.launch.block_dim, k.base_substitution)
        c, d = p
        out.append((a.field, a.kind, c, tuple(d.get(n, 0) for n in COORDS)))
    return out


def run_boxes(s, cnt, g):
    L, P = g[0], g[0] * g[1]
    e, cur, out = s + cnt, s, []
    while cur < e:
        if cur % L or e - cur < L:
            end = min((cur // L + 1) * L, e)
            out.append(((cur % L, (cur // L) % g[1], cur // P), (end - cur, 1, 1)))
            cur = end
        elif cur % P or e - cur < P:
            y0 = (cur // L) % g[1]
            rows = min((e - cur) // L, g[1] - y0)
            out.append(((0, y0, cur // P), (L, rows, 1)))
            cur += rows * L
        else:
            layers = (e - cur) // P
            out.append(((0, 0, cur // P), (L, g[1], layers)))
            cur += layers * P
    return out


def normalize(base, span, dims, g):
    dims = sorted((s, e) for s, e in dims if e > 1 and s != 0)
    m = []
    for s, e in dims:
        if m and s % m[-1][0] == 0 and s // m[-1][0] <= m[-1][1]:
            ps, pe = m[-1]
            m[-1] = (ps, pe + (s // ps) * (e - 1))
            continue
        m.append((s, e))
    k = 0
    while k < len(m) and m[k][0] <= span + g:
        span += m[k][0] * (m[k][1] - 1)
        k += 1
    return base, span, m[k:]


def box_lattice(c, bd, box, g):
    lo, n = box
    ext = (bd[0], bd[1], bd[2], n[0], n[1], n[2])
    base = c[3] * lo[0] + c[4] * lo[1] + c[5] * lo[2]
    dims = []
    for k in range(6):
        co = c[k]
        if ext[k] <= 1 or co == 0:
            continue
        if co < 0:
            base += co * (ext[k] - 1)
            co = -co
        dims.append((co, ext[k]))
    return normalize(base, 0, dims, g)


def mono(span, dims):
    reach = span
    for d, (s, e) in enumerate(dims):
        if d > 0 and s <= reach:
            return False
        reach += s * (e - 1)
    return True


def cover(L0, P, g):
    """Greedy cover of translates P (sorted unique) of lattice L0 -> lattices."""
    base0, span0, dims0 = L0
    out = []
    req = set(range(len(P)))
    Ps = set(P)
    idx = {v: i for i, v in enumerate(P)}
    for d in range(len(dims0) - 1, -1, -1):
        s = dims0[d][0]
        clear = set()
        for i, v in enumerate(P):
            if v - s in Ps:
                continue
            mem = [i]
            t = v + s
            while t in Ps:
                mem.append(idx[t])
                t += s
            if len(mem) >= 2 and len(req & set(mem)) >= 2:
                dims = list(dims0)
                dims[d] = (s, dims[d][1] + len(mem) - 1)
                out.append(normalize(v, span0, dims, g))
                clear |= set(mem)
        req -= clear
    for _ in range(3):
        r = sorted(req)
        if len(r) < 2:
            break
        gap = min(P[r[i + 1]] - P[r[i]] for i in range(len(r) - 1))
        if gap <= span0 + g:
            break
        clear = set()
        for i, v in enumerate(P):
            if i not in req:
                continue
            if v - gap in Ps:
                continue
            mem = [i]
            t = v + gap
            while t in Ps:
                mem.append(idx[t])
                t += gap
            if len(mem) >= 2 and len(req & set(mem)) >= 2:
                out.append(normalize(v, span0, list(dims0) + [(gap, len(mem))], g))
                clear |= set(mem)
        if not clear:
            break
        req -= clear
    tol = span0 + g
    i = 0
    r = sorted(req)
    P_req = [P[i] for i in range(len(P))]
    i = 0
    while i < len(P):
        j = i
        while j + 1 < len(P) and P[j + 1] - P[j] <= tol:
            j += 1
        if any(k in req for k in range(i, j + 1)):
            out.append(normalize(P[i], span0 + P[j] - P[i], dims0, g))
        i = j + 1
    return out


def unit(k, machine, kind="wave", field=None, g=32):
    cs = coefs(k)
    lc = k.launch
    bd, gd = lc.block_dim, lc.grid_dim
    total = gd[0] * gd[1] * gd[2]
    if kind == "wave":
        per = blocks_per_wave(lc, machine)
        nw = -(-total // per)
        w = nw // 2
        srcs = [(w * per, min(per, total - w * per))]
    else:
        srcs = [(total // 2, 1)]
    res = []
    for f in sorted({c[0] for c in cs}) if field is None else [field]:
        for kd in ("load", "store"):
            acc = [c for c in cs if c[0] == f and c[1] == kd]
            classes = {}
            for c in acc:
                classes.setdefault(c[3], set()).add(c[2])
            for s, cnt in srcs:
                for box in run_boxes(s, cnt, gd):
                    for cv, consts in classes.items():
                        L0 = box_lattice(cv, bd, box, g)
                        P = sorted(L0[0] + x for x in consts)
                        for lat in cover(L0, P, g):
                            base, span, dims = lat
                            n = int(np.prod([e for _, e in dims])) if dims else 1
                            res.append((f, kd, base, span, dims, n, mono(span, dims)))
    return res


if __name__ == "__main__":
    sp = W.space(sys.argv[1])
    i = int(sys.argv[2])
    k = sp.kernel(i)
    print(sp.key(i), k.launch)
    r = unit(k, sp.machine(i), "wave" if len(sys.argv) < 4 else sys.argv[3])
    tot = sum(x[5] for x in r)
    print("lattices", len(r), "intervals", tot, "non-mono", sum(1 for x in r if not x[6]),
          "non-mono intervals", sum(x[5] for x in r if not x[6]))
    for x in r[:40]:
        print(x)


# ---------------------------------------------------------------- segments
def decompose(L0, P):
    """p - base0 = rho + sum_d k_d * s_d: round to nearest for d >= 1, floor for
    dim 0 (rho in [0, s0))."""
    base0, span0, dims0 = L0
    out = []
    for p in P:
        off = p - base0
        k = [0] * len(dims0)
        for d in range(len(dims0) - 1, 0, -1):
            s = dims0[d][0]
            k[d] = (off + s // 2) // s
            off -= k[d] * s
        s0 = dims0[0][0]
        k[0] = off // s0
        off -= k[0] * s0
        out.append((off, k))
    return out


def seg_ok(L0, P, g):
    base0, span0, dims0 = L0
    if not dims0 or len(P) < 2:
        return False
    s0 = dims0[0][0]
    rs = sorted({r for r, _ in decompose(L0, P)})
    tol = span0 + g
    return all(b - a <= tol for a, b in zip(rs, rs[1:])) and rs[0] + s0 - rs[-1] <= tol


def segment_cover(L0, P, g):
    """Partition lattice-coordinate space by every translate's box boundaries;
    in each segment box the present translates are fixed, their residues
    cluster into spans (full cells fold into contiguous rows)."""
    base0, span0, dims0 = L0
    dec = decompose(L0, P)
    nd = len(dims0)
    bps = []
    for d in range(nd):
        e = dims0[d][1]
        bps.append(sorted({k[d] for _, k in dec} | {k[d] + e for _, k in dec}))
    import itertools
    out = []
    order = sorted(range(len(P)), key=lambda i: dec[i][0])
    tol = span0 + g
    for seg in itertools.product(*[range(len(b) - 1) for b in bps]):
        lo = [bps[d][seg[d]] for d in range(nd)]
        hi = [bps[d][seg[d] + 1] for d in range(nd)]
        mem = [i for i in order
               if all(dec[i][1][d] <= lo[d] and hi[d] <= dec[i][1][d] + dims0[d][1] for d in range(nd))]
        if not mem:
            continue
        bS = base0 + sum(lo[d] * dims0[d][0] for d in range(nd))
        dS = [(dims0[d][0], hi[d] - lo[d]) for d in range(nd)]
        rs = [dec[i][0] for i in mem]
        i = 0
        while i < len(rs):
            j = i
            while j + 1 < len(rs) and rs[j + 1] - rs[j] <= tol:
                j += 1
            out.append(normalize(bS + rs[i], span0 + rs[j] - rs[i], dS, g))
            i = j + 1
    return out


def granules(lats, g):
    s = set()
    for base, span, dims in lats:
        idx = [np.arange(e) * st for st, e in dims]
        b = np.array([base], dtype=np.int64)
        for a in idx:
            b = (b[:, None] + a[None, :]).ravel()
        for bb in b.tolist():
            s.update(range(bb // g, (bb + span) // g + 1))
    return s


def check_segments(k, machine, g=32, kind="block"):
    """Brute-force exactness check of segment_cover against the translates."""
    cs = coefs(k)
    lc = k.launch
    bd, gd = lc.block_dim, lc.grid_dim
    total = gd[0] * gd[1] * gd[2]
    srcs = [(total // 2, 1)] if kind == "block" else [(total // 2, 3)]
    n_ok = n_seg = 0
    for f in sorted({c[0] for c in cs}):
        for kd in ("load", "store"):
            classes = {}
            for c in cs:
                if c[0] == f and c[1] == kd:
                    classes.setdefault(c[3], set()).add(c[2])
            for s, cnt in srcs:
                for box in run_boxes(s, cnt, gd):
                    for cv, consts in classes.items():
                        L0 = box_lattice(cv, bd, box, g)
                        P = sorted(L0[0] + x for x in consts)
                        truth = granules([(p, L0[1], L0[2]) for p in P], g)
                        if seg_ok(L0, P, g):
                            n_seg += 1
                            got = granules(segment_cover(L0, P, g), g)
                            assert got == truth, (f, kd, box)
                        n_ok += 1
    return n_ok, n_seg


def unit_seg(k, machine, kind="wave", g=32):
    """Interval count of a unit with and without the segment transform."""
    cs = coefs(k)
    lc = k.launch
    bd, gd = lc.block_dim, lc.grid_dim
    total = gd[0] * gd[1] * gd[2]
    if kind == "wave":
        per = blocks_per_wave(lc, machine)
        nw = -(-total // per)
        w = nw // 2
        srcs = [(w * per, min(per, total - w * per))]
    else:
        srcs = [(total // 2, 1)]
    old = new = nl_old = nl_new = 0
    for f in sorted({c[0] for c in cs}):
        for kd in ("load", "store"):
            classes = {}
            for c in cs:
                if c[0] == f and c[1] == kd:
                    classes.setdefault(c[3], set()).add(c[2])
            for s, cnt in srcs:
                for box in run_boxes(s, cnt, gd):
                    for cv, consts in classes.items():
                        L0 = box_lattice(cv, bd, box, g)
                        P = sorted(L0[0] + x for x in consts)
                        a = cover(L0, P, g)
                        b = segment_cover(L0, P, g) if seg_ok(L0, P, g) else a
                        cnt_ = lambda ls: sum(int(np.prod([e for _, e in d])) if d else 1 for _, _, d in ls)
                        old += cnt_(a); new += cnt_(b); nl_old += len(a); nl_new += len(b)
    return old, new, nl_old, nl_new


def split_count(lat):
    """Runs emit_lattice produces for one lattice (monotone split <= 64)."""
    base, span, dims = lat
    reach = span
    combos = 1
    ns = 0
    for d, (s, e) in enumerate(dims):
        if d > 0 and s <= reach:
            ns += 1
            combos *= e
        else:
            reach += s * (e - 1)
    return 1 if ns == 0 or combos > 64 else combos
