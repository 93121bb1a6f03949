"""Generate the block-Jacobi schedule table used by eig_kernel (wnnm.cu).

The 63 rounds of a parallel cyclic Jacobi sweep over 64 indices pair i with
i ^ r (r = 1..63). Grouping the rounds into the 21 lines {a, b, a^b} of a
line spread of PG(5, 2) makes every group of three rounds act inside the 16
cosets (quads) of the subspace {0, a, b, a^b}: a "super-round" is one 4x4
block-Jacobi step. Each line also carries a basis g0..g3 of a complement T
whose projection onto the low four bits is bijective, so the quad
representatives t_B = xor of g_k over the bits k of B (B = 0..15) sit in 16
distinct shared-memory banks.

Run: python tools/jacobi_schedule.py  (prints the C table)."""
POLY = 0b1000011  # x^6 + x + 1 (primitive)


def gf_mul(a, b):
    r = 0
    while b:
        if b & 1:
            r ^= a
        b >>= 1
        a <<= 1
        if a & 0b1000000:
            a ^= POLY
    return r


def gf_pow(a, e):
    r = 1
    for _ in range(e):
        r = gf_mul(r, a)
    return r


def span(vecs):
    s = {0}
    for v in vecs:
        s |= {x ^ v for x in s}
    return s


def spread():
    alpha = 0b10
    omega = gf_pow(alpha, 21)  # order 3: GF(4)* inside GF(64)*
    seen, lines = set(), []
    for e in range(63):
        x = gf_pow(alpha, e)
        if x in seen:
            continue
        line = [x, gf_mul(x, omega), gf_mul(x, gf_mul(omega, omega))]
        assert line[0] ^ line[1] == line[2]
        seen |= set(line)
        lines.append(line)
    assert len(lines) == 21 and len(seen) == 63
    return lines


def complement(a, b):
    # depth-first search for g0..g3 with span(S, T) = all and low-4-bit projection bijective
    def rec(basis):
        if len(basis) == 4:
            T = span(basis)
            if len(span(basis + [a, b])) == 64 and len({t & 15 for t in T}) == 16:
                return basis
            return None
        start = basis[-1] + 1 if basis else 1
        for v in range(start, 64):
            if v in span(basis + [a, b]):
                continue
            if (v & 15) in {t & 15 for t in span(basis)}:
                continue
            r = rec(basis + [v])
            if r:
                return r
        return None
    return rec([])


def table():
    rows = []
    for a, b, _ in spread():
        g = complement(a, b)
        rows.append((a, b, *g))
    return rows


def check(rows):
    seen = set()
    for a, b, *g in rows:
        T = []
        for B in range(16):
            t = 0
            for k in range(4):
                if (B >> k) & 1:
                    t ^= g[k]
            T.append(t)
        assert len({t & 15 for t in T}) == 16
        for t in T:
            q = [t, t ^ a, t ^ b, t ^ a ^ b]
            for i in range(4):
                for j in range(i + 1, 4):
                    pr = (min(q[i], q[j]), max(q[i], q[j]))
                    assert pr not in seen
                    seen.add(pr)
    assert len(seen) == 64 * 63 // 2
    return True


def plane_spread():
    """The 9 planes (3-dim subspaces) alpha^i * GF(8) of GF(64), i = 0..8:
    they partition the 63 nonzero vectors (octet schedule of eig_kernel<true>)."""
    alpha = 0b10
    beta = gf_pow(alpha, 9)  # order 7: GF(8)* inside GF(64)*
    planes = []
    for i in range(9):
        x = gf_pow(alpha, i)
        basis = [x, gf_mul(x, beta), gf_mul(x, gf_mul(beta, beta))]
        assert len(span(basis)) == 8
        planes.append(basis)
    allv = set()
    for b in planes:
        allv |= span(b) - {0}
    assert len(allv) == 63
    return planes


def plane_complement(s):
    # t0..t2 with span(S, T) = all and the 8 representatives in 8 distinct
    # low-3-bit classes (spread over shared-memory banks)
    def rec(basis):
        if len(basis) == 3:
            T = span(basis)
            if len(span(basis + s)) == 64 and len({t & 7 for t in T}) == 8:
                return basis
            return None
        start = basis[-1] + 1 if basis else 1
        for v in range(start, 64):
            if v in span(basis + s):
                continue
            if (v & 7) in {t & 7 for t in span(basis)}:
                continue
            r = rec(basis + [v])
            if r:
                return r
        return None
    return rec([])


def octet_table():
    rows = []
    for s in plane_spread():
        rows.append((*s, *plane_complement(s)))
    return rows


def check_octets(rows):
    seen = set()
    for s0, s1, s2, t0, t1, t2 in rows:
        S, T = [0] * 8, [0] * 8
        for l in range(8):
            for k, v in enumerate((s0, s1, s2)):
                if (l >> k) & 1:
                    S[l] ^= v
            for k, v in enumerate((t0, t1, t2)):
                if (l >> k) & 1:
                    T[l] ^= v
        assert len({t & 7 for t in T}) == 8
        for B in range(8):
            o = [T[B] ^ S[l] for l in range(8)]
            for i in range(8):
                for j in range(i + 1, 8):
                    pr = (min(o[i], o[j]), max(o[i], o[j]))
                    assert pr not in seen
                    seen.add(pr)
    assert len(seen) == 64 * 63 // 2
    return True


if __name__ == "__main__":
    rows = table()
    check(rows)
    print("// {a, b, g0, g1, g2, g3} per super-round (tools/jacobi_schedule.py)")
    for r in rows:
        print("    {" + ", ".join(str(v) for v in r) + "},")
    orows = octet_table()
    check_octets(orows)
    print("// {s0, s1, s2, t0, t1, t2} per octet super-round (tools/jacobi_schedule.py)")
    for r in orows:
        print("    {" + ", ".join(str(v) for v in r) + "},")
