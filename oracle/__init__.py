"""ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU (numpy, fp64) implementation of what the
hot path of arXiv 2304.12387 computes.  Only `tests/`, `__graft_entry__.smoke()`
and `bench.py`'s `cpu_baseline` / `--impl reference` legs may import it.  The
product path (`paper_2304_12387_b200/`) never imports it and shares no code
with it; the only shared module is `synth/` (seeded inputs, no arithmetic of
the method).

Citations: ``P:n`` = /root/reference/PAPER.md line n (section / equation named
beside it).  Every function names the passage it follows.

What is computed by its plain definition (dense element matrices by direct
Gauss-Legendre quadrature, global assembly, Algorithm 1 literally, the entry
formula of S~ and the sparse triple product, MINRES step by step):
  basis1d   - GLL nodes, GL rule, Lagrange l_i, histopolation h_j       (§2.1)
  fem       - element geometry, RT/L2 reference bases, M^e, W^e, B^e    (eq. matrices)
  space     - canonical numbering, Algorithm 1 index tables, D in CSR   (Alg. 1)
  operators - assembled M, W, Z, block apply, diagonals, S~ two paths
  solvers   - Chebyshev-Jacobi S^-1, block-diagonal preconditioner, MINRES;
              block-triangular preconditioner + GMRES (NEXT-4); the pure-Neumann
              projection after S^-1 (NEXT-3)
  amg       - smoothed-aggregation AMG V-cycle for S^-1 (NEXT-1, reading A9b), per-slab
              block-Jacobi (reading A9c)
  mms       - manufactured-solution loads (convergence-rate pins)
  sample    - element-local evaluation of sampled output rows (full-size parity)
Essential-flux sides by elimination (NEXT-3) and the general (vertex-field) gamma with
the full W^-1 W_gamma W^-1 block (NEXT-3) live in operators / space / fem.

Parity pins (tests/test_oracle_*.py, `-m "not gpu"`): closed-form 1D tables,
SPD / exactness of M, B = W D, D's incidence structure,
M-matrix S~, Prop. 2.1/2.2 spectra, dense-solve MINRES,
manufactured-solution convergence rates, closed-form traces; eliminated sides: the incidence
boundary, the one-dimensional pure-Neumann nullspace, S~ 1 = 0, exact uniform flow; general
gamma: the constant-field reduction, an exact weighted Kronecker product, the p = 1
mean-value closed form; block-Jacobi AMG: exact block solves.
Piola-mapped element matrices on non-axis-aligned elements (tests/test_oracle_piola.py): the
parallelepiped closed form (beta/det J)(J^T J)_{cc'} (x) exact 1D integrals built independently,
rotation invariance on general trilinear elements, the s^{2-d} scaling law, and MMS rates on
smoothly distorted 2D/3D meshes (a J <-> J^T swap fails them).  The sampled-row path
(sample.py) is pinned against the global assembly, including the vertex-field gamma.
Nothing in the oracle is left parity-unpinned.
"""
