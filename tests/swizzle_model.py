"""Host replay of the shared-memory index math in csrc/fft_block.cuh.

Used by tests/test_swizzle.py to prove the XOR swizzles keep every DIF stage
bank-conflict free (and by developers to inspect conflict degrees)."""
from __future__ import annotations


def ilog2(n: int) -> int:
    return n.bit_length() - 1


def radix_plan(L: int):
    lg = ilog2(L)
    S = 0 if lg == 0 else (lg + 3) // 4
    bits = [lg // S + (1 if s < lg % S else 0) for s in range(S)]
    R = [1 << b for b in bits]
    span = []
    ls = L
    for s in range(S):
        span.append(ls)
        ls //= R[s]
    span.append(1)
    return S, bits, R, span


def digit_pos(L: int, k: int) -> int:
    S, bits, R, span = radix_plan(L)
    pos = 0
    for s in range(S):
        pos += (k & (R[s] - 1)) * span[s + 1]
        k >>= bits[s]
    return pos


# GF(2)-linear swizzles a -> a ^ g(a >> sh), g(h) = XOR of C[d % 4] over the
# set bits d of h. sh = 3 for 16-B elements (fp64 complex), 4 for 8-B (fp32).
# Column tiles use constants proven conflict-free for every aligned dyadic
# window; row tiles use constants found by exhaustive search over the row
# kernel's stage patterns (including the gapped last-stage pattern).
COL_C = {16: (4, 6, 5, 7), 8: (8, 12, 10, 15)}
ROW_C = {16: (1, 2, 4, 1), 8: (1, 6, 10, 8)}


def _lin(a: int, esize: int, consts) -> int:
    sh = 3 if esize == 16 else 4
    c = consts[esize]
    h = a >> sh
    g = 0
    d = 0
    while h:
        if h & 1:
            g ^= c[d & 3]
        h >>= 1
        d += 1
    return a ^ g


def swz_col(a: int, esize: int) -> int:
    return _lin(a, esize, COL_C)


def swz_row(a: int, esize: int) -> int:
    return _lin(a, esize, ROW_C)


def col_at(line, n, lgw, esize):
    return swz_col((n << lgw) + line, esize)


def row_at(line, n, L, esize):
    return swz_row(line * L + n, esize)


def conflict_degree(addrs, esize):
    """Max over lane groups of how many distinct addresses share a bank slot."""
    per = 128 // esize  # elements per bank row
    group = per         # lanes served per wavefront
    worst = 1
    for g in range(0, len(addrs), group):
        slots = {}
        for a in addrs[g:g + group]:
            slots.setdefault(a % per, set()).add(a)
        worst = max(worst, max(len(v) for v in slots.values()))
    return worst


def stage_degrees(L, nlines, nthreads, esize, line_fast):
    S, bits, R, span = radix_plan(L)
    lgw = ilog2(nlines)
    out = []
    for s in range(S):
        r_ = R[s]
        q = span[s] // r_
        nblk = L // span[s]
        total = (L // r_) * nlines
        worst = 1
        for it in range(0, total, nthreads):
            for w0 in range(0, min(nthreads, total - it), 32):
                lanes = range(it + w0, min(it + w0 + 32, total))
                for r in range(r_):
                    addrs = []
                    for bf in lanes:
                        if line_fast:
                            line = bf & (nlines - 1); rest = bf >> lgw
                            j = rest & (q - 1); b = rest >> ilog2(q)
                        else:
                            j = bf & (q - 1); rest = bf >> ilog2(q)
                            b = rest & (nblk - 1); line = rest >> ilog2(nblk)
                        n = b * span[s] + j + r * q
                        addrs.append(col_at(line, n, lgw, esize) if line_fast
                                     else row_at(line, n, L, esize))
                    worst = max(worst, conflict_degree(addrs, esize))
        out.append(worst)
    return out


if __name__ == "__main__":
    for esize in (8, 16):
        for L in (8, 16, 64, 256, 1024, 2048, 4096):
            for nl in (2, 4, 8, 16):
                if L * nl * esize > 160 * 1024:
                    continue
                print("col", esize, L, nl, stage_degrees(L, nl, 256, esize, True),
                      "row", stage_degrees(L, nl, 256, esize, False))


def digit_rev(L: int, n: int) -> int:
    """Inverse of digit_pos: the frequency index held at slot n."""
    S, bits, R, span = radix_plan(L)
    k = 0
    shift = 0
    for s in range(S):
        d = (n // span[s + 1]) % R[s]
        k |= d << shift
        shift += bits[s]
    return k


def row_extra_degrees(L, G, esize, nthreads):
    """v2 row-kernel patterns beyond the DIF stages: (a) last stage writes its
    outputs at natural-frequency addresses, (b) natural-order reads by
    consecutive threads, (c) pair-interleaved (s-order) reads."""
    S, bits, R, span = radix_plan(L)
    r_ = R[S - 1]
    nbf = L * G // r_
    worst = {"kwrite": 1, "natural": 1, "sorder": 1}
    for it in range(0, nbf, nthreads):
        for w0 in range(0, min(nthreads, nbf - it), 32):
            for r in range(r_):
                addrs = []
                for bf in range(it + w0, min(it + w0 + 32, nbf)):
                    b = bf % (L // r_)
                    line = bf // (L // r_)
                    n = b * r_ + r
                    addrs.append(row_at(line, digit_rev(L, n), L, esize))
                worst["kwrite"] = max(worst["kwrite"], conflict_degree(addrs, esize))
    for line in range(G):
        for base in range(0, L, 32):
            addrs = [row_at(line, (base + t) % L, L, esize) for t in range(32)]
            worst["natural"] = max(worst["natural"], conflict_degree(addrs, esize))
            m = [(s >> 1) if s % 2 == 0 else L - 1 - (s >> 1) for s in range(base, base + 32)]
            worst["sorder"] = max(worst["sorder"], conflict_degree([row_at(line, x % L, L, esize) for x in m], esize))
    return worst
