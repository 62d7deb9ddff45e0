"""Shared-memory bank model of the trilinear kernel's line passes (development aid; layout only,
no method arithmetic).  For every array shape (D0, D1, D2) it searches the padded strides
(S1 >= D0, S2 >= S1 * D1) minimising the modelled wavefronts of every warp access the kernel
makes to arrays of that shape (64-bit accesses served per half-warp: cost = max over the 16 bank
pairs of the distinct 8-byte words), and writes paper_2304_12387_b200/csrc/tri_layouts.h.

    python scripts/tri_layout_model.py            (all orders)
"""
import sys
from collections import defaultdict

sys.path.insert(0, "scripts")
from smem_model import wavefronts   # noqa: E402


def odd(v):
    return v if v % 2 else v + 1


class Acc:
    """accesses per shape: list of (weight, lane -> (d0, d1, d2) or None, per-access offset fn)"""
    def __init__(self):
        self.by = defaultdict(list)

    def add(self, shape, weight, lanes, naccess, coord):
        self.by[shape].append((weight, lanes, naccess, coord))


def line_pass(acc, dims_in, dims_out, AX, NO, lanes_of, weight):
    """the `lines` helper: item it -> (b0, b1); reads NIN along AX, writes NO along AX."""
    NIN = dims_in[AX]
    B0 = dims_in[1] if AX == 0 else dims_in[0]
    B1 = dims_in[1] if AX == 2 else dims_in[2]
    others = [a for a in range(3) if a != AX]   # (first, second)

    def item(it, t, dims):
        b0, b1 = it % B0, it // B0
        c = [0, 0, 0]
        c[others[0]], c[others[1]] = b0, b1
        c[AX] = t
        return tuple(c)
    nitems = B0 * B1
    acc.add(tuple(dims_in), weight, (lanes_of, nitems), NIN, lambda it, t: item(it, t, dims_in))
    acc.add(tuple(dims_out), weight, (lanes_of, nitems), NO, lambda it, t: item(it, t, dims_out))


def model(P, NT):
    Q = P + 2
    acc = Acc()
    U = [(P + 1, P, P), (P, P + 1, P), (P, P, P + 1)]
    A = [(Q, P, P), (Q, P + 1, P), (Q, P, P + 1)]
    B = [(Q, Q, P), (Q, Q, P), (Q, Q, P + 1)]
    V = (Q, Q, Q)
    L2 = (P, P, P)
    lanes = 32 if NT == 96 else NT
    for c in range(3):
        line_pass(acc, U[c], A[c], 0, Q, lanes, 1.0)
        line_pass(acc, A[c], B[c], 1, Q, lanes, 1.0)
        line_pass(acc, B[c], V, 2, Q, lanes, 1.0)
        line_pass(acc, V, B[c], 2, [P, P, P + 1][c], lanes, 1.0)
        line_pass(acc, B[c], A[c], 1, [P, P + 1, P][c], lanes, 1.0)
        line_pass(acc, A[c], U[c], 0, [P + 1, P, P][c], lanes, 1.0)
    # gather (write) and scatter (read) of the RT components, lanes over the local DOFs
    for c in range(3):
        E0, E1, E2 = U[c]
        for w in (1.0, 1.0):
            acc.add(U[c], w, (NT, E0 * E1 * E2), 1,
                    lambda it, t, E0=E0, E1=E1: (it % E0, (it // E0) % E1, it // (E0 * E1)))
    # D u: lanes over the cells, two faces per component
    for c in range(3):
        acc.add(U[c], 1.0, (NT, P ** 3), 2,
                lambda it, t, c=c: tuple((it % P, (it // P) % P, it // (P * P))[a] + (t if a == c else 0)
                                         for a in range(3)))
    # q~ tile: load, D^T reads in the scatter (cell and - neighbour)
    acc.add(L2, 1.0, (NT, P ** 3), 1, lambda it, t: (it % P, (it // P) % P, it // (P * P)))
    for c in range(3):
        E0, E1, E2 = U[c]
        acc.add(L2, 1.0, (NT, E0 * E1 * E2), 2,
                lambda it, t, E0=E0, E1=E1, E2=E2, c=c: tuple(
                    min(max((it % E0, (it // E0) % E1, it // (E0 * E1))[a] - (t if a == c else 0), 0),
                        P - 1) for a in range(3)))
    # pointwise over the quadrature points (all threads, 3 components read + written)
    for c in range(3):
        acc.add(V, 2.0, (NT, Q ** 3), 1, lambda it, t: (it % Q, (it // Q) % Q, it // (Q * Q)))
    # local CG of W^-1 (grad-div / gamma > 0), ~6 iterations
    GA, GB = (Q, P, P), (Q, Q, P)
    for (din, dout, ax, no) in [(L2, GA, 0, Q), (GA, GB, 1, Q), (GB, V, 2, Q), (V, GB, 2, P),
                                (GB, GA, 1, P), (GA, L2, 0, P)]:
        line_pass(acc, din, dout, ax, no, 64, 6.0)
    return acc


def cost(acc, shape, S1, S2):
    tot = 0.0
    for weight, (lanes, nitems), nacc, coord in acc.by[shape]:
        w = 0
        for base in range(0, nitems, 32 if lanes >= 32 else lanes):
            for t in range(nacc):
                ad = []
                for l in range(32):
                    it = base + l
                    if l >= lanes or it >= nitems:
                        ad.append(None)
                        continue
                    d0, d1, d2 = coord(it, t)
                    ad.append(d0 + S1 * d1 + S2 * d2)
                w += wavefronts(ad)
        tot += weight * w
    return tot


def search(acc, shape, slack1=8, slack2=16, growth=1.10):
    D0, D1, D2 = shape
    base1 = odd(D0)
    base2 = base1 * odd(D1)
    size0 = base2 * D2
    best = (cost(acc, shape, base1, base2), base1, base2)
    for S1 in range(D0, D0 + slack1):
        for S2 in range(S1 * D1, S1 * D1 + slack2):
            if S2 * D2 > size0 * growth:
                continue
            c = cost(acc, shape, S1, S2)
            if c < best[0] - 1e-9:
                best = (c, S1, S2)
    return best, cost(acc, shape, base1, base2)


def main():
    rows = []
    for P in range(1, 7):
        for NT in (64, 96):
            acc = model(P, NT)
            for shape in sorted(acc.by):
                (c, S1, S2), c0 = search(acc, shape)
                rows.append((P, NT, shape, S1, S2, c0, c))
                print(f"P={P} NT={NT} {shape}: odd ({odd(shape[0])}, {odd(shape[0]) * odd(shape[1])}) "
                      f"{c0:.0f} -> ({S1}, {S2}) {c:.0f}", flush=True)
    out = ["// tri_layouts.h — GENERATED by scripts/tri_layout_model.py (do not edit by hand).",
           "// Padded smem strides of the trilinear kernel's arrays per (order, CTA size, shape),",
           "// chosen to minimise the modelled shared-memory wavefronts of its line passes.",
           "#pragma once", "", "namespace hdiv {",
           "struct TriLayout { int P, NT, D0, D1, D2, S1, S2; };",
           "constexpr TriLayout kTriLayouts[] = {"]
    for P, NT, (D0, D1, D2), S1, S2, c0, c in rows:
        out.append(f"    {{{P}, {NT}, {D0}, {D1}, {D2}, {S1}, {S2}}},   // {c0:.0f} -> {c:.0f}")
    out += ["};", "constexpr int kNumTriLayouts = sizeof(kTriLayouts) / sizeof(kTriLayouts[0]);",
            "constexpr int find_tri_layout(int P, int NT, int D0, int D1, int D2) {",
            "  for (int i = 0; i < kNumTriLayouts; ++i)",
            "    if (kTriLayouts[i].P == P && kTriLayouts[i].NT == NT && kTriLayouts[i].D0 == D0 &&",
            "        kTriLayouts[i].D1 == D1 && kTriLayouts[i].D2 == D2)",
            "      return i;",
            "  return -1;", "}", "}  // namespace hdiv", ""]
    open("paper_2304_12387_b200/csrc/tri_layouts.h", "w").write("\n".join(out))


if __name__ == "__main__":
    main()
