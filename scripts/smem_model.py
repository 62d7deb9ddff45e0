"""Shared-memory wavefront model of the halo-tile box kernel (development aid).

For 64-bit accesses a warp instruction is served per half-warp; a half-warp with active lanes
needs max over the 16 bank pairs of the number of DISTINCT 8-byte words mapping to that pair
(same word = broadcast).  This reproduces the ncu counts of the profiled kernel (e.g. the
x-component M_l pass: 2 wavefronts per instruction with 8 active lanes per half-warp).

The model mirrors the lane -> address maps of kernel_affine.cu for a given layout
(per-component strides S1, S2; q~ tile strides Q1, Q2) and lane-mapping choices (packed or
padded to half-warps), and `search` picks the layout with the fewest modelled wavefronts.

Usage: python scripts/smem_model.py P TX TY TZ            (current layout)
       python scripts/smem_model.py P TX TY TZ search     (best layout, C++ table line)
"""
import sys
from collections import defaultdict


def odd(v):
    return v if v % 2 else v + 1


def wavefronts(addrs):
    w = 0
    for h in (0, 16):
        words = {a for a in addrs[h:h + 16] if a is not None}
        if not words:
            continue
        cnt = defaultdict(int)
        for a in words:
            cnt[a % 16] += 1
        w += max(cnt.values())
    return w


def run(NT, items, naccess, addr, acc=None, distinct_k=True):
    """Sum of wavefronts over every warp instruction of a loop it = tid + j NT (items), each
    item performing accesses k = 0..naccess-1.  If the address of access k is access 0's plus a
    lane-independent constant (distinct_k False), only k = 0 is evaluated and scaled."""
    tot = 0
    ks = range(naccess) if distinct_k else [0]
    for base in range(0, items, 32):
        for k in ks:
            ad = [addr(base + l, k) if base + l < items else None for l in range(32)]
            if any(a is not None for a in ad):
                tot += wavefronts(ad)
    return tot if distinct_k else tot * naccess


class Layout:
    def __init__(self, P, T, S=None, Q=None, padL=None, padA=None, zmap=0):
        self.P, self.T = P, T
        self.zmap = zmap
        CX, CY, CZ = (t * P for t in T)
        self.C = (CX, CY, CZ)
        self.E = []
        for AX in range(3):
            E = [T[d] * P for d in range(3)]
            E[AX] = (T[AX] + 1) * P + 1
            self.E.append(E)
        self.S = S or [(odd(E[0]), odd(E[0]) * odd(E[1])) for E in self.E]
        self.Q = Q or (odd(CX), odd(CX) * odd(CY))
        self.padL = padL or [True, True, True]    # M_l / halo lanes padded to 16
        self.padA = padA or [True, True, True]    # M_h (x) M_h positions padded to 16

    def smem(self):
        su = max([S2 * E[2] for (S1, S2), E in zip(self.S, self.E)] + [self.Q[1] * self.C[2]])
        return su


def comp_cost(L, AX, NT=128):
    P, T = L.P, L.T
    CX, CY, CZ = L.C
    E = L.E[AX]
    S1, S2 = L.S[AX]
    Q1, Q2 = L.Q
    Sd = [1, S1, S2]
    A1, A2 = [d for d in range(3) if d != AX]
    TA1, TA2, TA = T[A1], T[A2], T[AX]
    SA, SA1, SA2 = Sd[AX], Sd[A1], Sd[A2]
    EA = E[AX]
    out = {}
    # landing (rows<>)
    Lr = E[0]
    LP = 2 if Lr <= 2 else 4 if Lr <= 4 else 8 if Lr <= 8 else 16 if Lr <= 16 else 32
    RPI = 32 // LP
    NJ = (E[1] + RPI - 1) // RPI
    w = 0
    for i2 in range(E[2]):
        for j in range(NJ):
            ad = []
            for lane in range(32):
                c, rs = lane % LP, lane // LP
                i1 = j * RPI + rs
                ad.append(i2 * S2 + i1 * S1 + c if (c < Lr and i1 < E[1]) else None)
            w += wavefronts(ad)
    out["landing"] = w

    # D u
    def du(col, k):
        X, Y = col % CX, col // CX
        pos = [X, Y, 0]
        pos[AX] += P
        base = pos[0] + S1 * pos[1] + S2 * pos[2]
        if AX == 2:
            return base + k * S2
        return base + (k // 2) * S2 + (SA if k % 2 else 0)
    out["Du"] = run(NT, CX * CY, (CZ + 1) if AX == 2 else 2 * CZ, du)
    EL1, EL2 = TA1 * P, TA2 * P
    EL1P = (EL1 + 15) // 16 * 16 if L.padL[AX] else EL1

    def lmap(it):
        l1, l2 = it % EL1P, it // EL1P
        return (None, None) if l1 >= EL1 else (l1, l2)

    def halo(it, k):
        l1, l2 = lmap(it)
        if l1 is None:
            return None
        return l1 * SA1 + l2 * SA2 + (k if k <= P else P - 1) * SA
    out["halo"] = run(NT, EL1P * EL2, P + 2, halo, distinct_k=False)
    EAH = EA - (P - 1)
    EAP = (EAH + 15) // 16 * 16 if L.padA[AX] else EAH

    def mh(it, k):
        pa = it % EAP + (P - 1)
        b1 = (it // EAP) % TA1
        b2 = it // (EAP * TA1)
        if pa >= EA:
            return None
        kk = k % (P * P)
        return pa * SA + b1 * P * SA1 + b2 * P * SA2 + (kk % P) * SA1 + (kk // P) * SA2
    out["MhMh"] = run(NT, EAP * TA1 * TA2, 2 * P * P, mh, distinct_k=False)
    QA = {0: 1, 1: Q1, 2: Q2}

    def ml(it, k):
        l1, l2 = lmap(it)
        if l1 is None:
            return None
        return l1 * SA1 + l2 * SA2
    out["Ml line"] = run(NT, EL1P * EL2, TA * (P + 1), ml, distinct_k=False)

    def mlq(it, k):
        l1, l2 = lmap(it)
        if l1 is None:
            return None
        return l1 * QA[A1] + l2 * QA[A2]
    out["Ml q"] = run(NT, EL1P * EL2, TA * P, mlq, distinct_k=False)

    def mlc(it, k):   # coefficient reads (sco, 4 words per element slot)
        l1, l2 = lmap(it)
        if l1 is None:
            return None
        ec = [0, 0, 0]
        ec[A1], ec[A2] = l1 // P, l2 // P
        return 4 * (((ec[2] + 1) * (T[1] + 1) + (ec[1] + 1)) * (T[0] + 1) + (ec[0] + 1))
    out["Ml coef"] = run(NT, EL1P * EL2, TA + 1, mlc, distinct_k=False)
    return out


def zblock(b, TX, zmap):
    """element column (bx, by) of item group b in the Z xy-block pass: zmap 0 = bx fastest;
    1 = bx split in halves interleaved (0, TX/2, 1, TX/2+1, ...: consecutive item groups are
    TX/2 element columns apart), for even TX"""
    by, r = b // TX, b % TX
    if zmap == 1 and TX % 2 == 0:
        return (r // 2) + (r % 2) * (TX // 2), by
    return r, by


def q_cost(L, NT=128):
    P, T = L.P, L.T
    CX, CY, CZ = L.C
    Q1, Q2 = L.Q
    out = {}
    out["q landing"] = run(NT, CX * CY, CZ, lambda col, k: col % CX + Q1 * (col // CX) + Q2 * k,
                           distinct_k=False)

    def hp(n0, s0, n1, s1, nb, sb):
        def f(it, k):
            i0, r = it % n0, it // n0
            i1, blk = r % n1, r // n1
            return i0 * s0 + i1 * s1 + blk * sb
        return f
    # the X- and Y-lines of (M_h^-1)^{(x)2} as ONE register-blocked pass: a thread owns the
    # P x P (X, Y) block of one element column at one cell layer Z (lanes over Z first) and
    # reads / writes it once
    def z2(it, k):
        zc, b = it % CZ, it // CZ
        bx, by = zblock(b, T[0], L.zmap)
        kk = k % (P * P)
        return bx * P + Q1 * by * P + Q2 * zc + (kk % P) + Q1 * (kk // P)
    out["Z xy-block"] = run(NT, CZ * T[0] * T[1], 2 * P * P, z2, distinct_k=False)
    out["Z z-lines"] = run(NT, CX * CY, CZ, lambda col, k: col % CX + Q1 * (col // CX),
                           distinct_k=False)
    return out


def total(L):
    t = {}
    for AX in range(3):
        for k, v in comp_cost(L, AX).items():
            t[f"c{AX} {k}"] = v
    t.update(q_cost(L))
    return t


def ndof(P, T):
    return 4 * P ** 3 * T[0] * T[1] * T[2]


def search(P, T, slack=16, smem_growth=1.10):
    base = Layout(P, T)
    su0 = base.smem()
    best = None
    CX, CY, CZ = base.C
    # q~ strides
    bestq = None
    # the q~ tile is extra shared memory (not overlaid on the component boxes): keep it within
    # a few words of the odd-padded minimum so CTAs per SM do not drop
    for q1 in range(CX, odd(CX) + 3):
        for q2 in range(q1 * CY, q1 * odd(CY) + slack):
            for zm in (0, 1):
                L = Layout(P, T, Q=(q1, q2), zmap=zm)
                if q2 * CZ > su0 * smem_growth:
                    continue
                c = sum(q_cost(L).values())
                for AX in range(3):
                    c += comp_cost(L, AX)["Ml q"]
                if bestq is None or c < bestq[0]:
                    bestq = (c, (q1, q2), zm)
    S, padL, padA = [], [], []
    for AX in range(3):
        E = base.E[AX]
        bc = None
        for s1 in range(E[0], E[0] + slack):
            for s2 in range(s1 * E[1], s1 * E[1] + slack):
                if s2 * E[2] > su0 * smem_growth:
                    continue
                for pl in (True, False):
                    for pa in (True, False):
                        Sx = list(base.S)
                        Sx[AX] = (s1, s2)
                        L = Layout(P, T, S=Sx, Q=bestq[1], padL=[pl] * 3, padA=[pa] * 3,
                                   zmap=bestq[2])
                        cc = comp_cost(L, AX)
                        c = sum(v for k, v in cc.items() if k != "Ml q") + cc["Ml q"]
                        if bc is None or c < bc[0]:
                            bc = (c, (s1, s2), pl, pa)
        S.append(bc[1]); padL.append(bc[2]); padA.append(bc[3])
    return Layout(P, T, S=S, Q=bestq[1], padL=padL, padA=padA, zmap=bestq[2])


def report(L, title):
    t = total(L)
    n = ndof(L.P, L.T)
    tw = sum(t.values())
    print(f"{title}: P={L.P} T={L.T} S={L.S} Q={L.Q} padL={L.padL} padA={L.padA} "
          f"smem SU={L.smem()} -> {tw} wavefronts, {tw / n:.3f}/DOF")
    for k, v in t.items():
        print(f"   {k:14s} {v:7d}  {v / n:.4f}/DOF")
    return tw


def main():
    P, TX, TY, TZ = (int(v) for v in sys.argv[1:5])
    T = (TX, TY, TZ)
    report(Layout(P, T), "current")
    if len(sys.argv) > 5 and sys.argv[5] == "search":
        L = search(P, T)
        report(L, "searched")
        print(f"  {{{P}, {TX}, {TY}, {TZ}, {{{', '.join(f'{{{a}, {b}}}' for a, b in L.S)}}}, "
              f"{{{L.Q[0]}, {L.Q[1]}}}, {{{', '.join(str(int(v)) for v in L.padL)}}}, "
              f"{{{', '.join(str(int(v)) for v in L.padA)}}}}},")


if __name__ == "__main__":
    main()
