"""CPU fp64 ORACLE for the inexact IETI-DP hot path (arXiv:1705.04531).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it.  The
product path (``paper_1705_04531_b200``) never imports, calls or links anything
here, and nothing here imports the product path: the two share no code.  The
only shared module is ``workloads`` (seeded input synthesis, no method
arithmetic).

Plain, slow, obviously correct: numpy / scipy library primitives (sparse
matrix-vector products, sparse LU, dense Cholesky, Gauss-Legendre nodes) as
steps, no blocking, fusion or reordering beyond what the paper's definitions
and algorithms state.  Every function cites the PAPER.md passage (``P:line``)
or the DESIGN.md reading (``R#``, numbered as in SURVEY.md Sec. 8(c)(iii)) it
follows.

Modules
  bspline   Cox-de Boor, knot insertion, Gauss rule, 1D mass
  assembly  stiffness / parameter mass / load per patch          (Eq. (1))
  topology  interfaces, Dirichlet sides, primal entities, B, B_D
  mg        Galerkin hierarchy, colour Gauss-Seidel, V-cycle
  ieti      primal basis, S_PiPi, F, d, M_sD, dual PCG, recovery (Eqs. (2)-(7))
  brute     global conforming assembly + sparse direct solve     (Eq. (1); exact-mode pin)
  saddle    MG-MG-S: BPCG on the saddle point Eq. (2)
  sharded   the same IetiOracle methods with patches in worker processes (full-size C5 dumps)

Parity-pin status: see DESIGN.md "Oracle pins".  Functions whose inexact
results have no independent pin say "parity unpinned" in their docstring.
"""
