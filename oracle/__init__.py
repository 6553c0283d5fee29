"""CPU oracle for the all-at-once block-circulant preconditioner (arXiv 2405.18964).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()`,
`tests/golden/gen_oracle_refs.py` and `bench.py`'s cpu_baseline /
`--impl reference` leg may import or execute anything under `oracle/`.  The
product path (`paper_2405_18964_b200/`) never imports it and shares no code
with it; only the seeded input generators in `synth/` serve both.

A plain, slow, obviously-correct fp64 / complex128 implementation written from
the paper, step by step in the paper's order and notation:

  fem.py       Q2-Q1 assembly by element loops with 3^d Gauss quadrature
  transfer.py  nodal-interpolation prolongation, restriction = P^T
  timeops.py   circulant spectrum d_k, naive DFT, c_{j,1}, c_{j,2}
  kkt.py       the all-at-once matrix A of eq. (FinalA) applied block by block
  inner.py     multicolour SOR, geometric multigrid V-cycles, Chebyshev
  precond.py   Algorithm 1 with the Stokes P~_j and Oseen P~_j^(UZ)
               (Algorithm 3) block solves
  gmres.py     restarted right-preconditioned GMRES(m) with MGS + Givens
  problem.py   assembly of one configuration's operators and MG hierarchy

Every function cites the passage it follows (P:n = /root/reference/PAPER.md
line n; SURVEY C.2 #n = the reading taken where the paper is silent or garbled,
listed in DESIGN.md).  Pins live in tests/test_oracle_*.py (run with
`-m "not gpu"`).  Parity status per function: see DESIGN.md "Oracle pins";
the MG/SOR parameters (C.2 #12) and the Oseen linear-mode choice (C.2 #16) are
"parity unpinned" against the paper itself -- they are pinned only by
contraction / limit checks, and the paper's iteration-count tables are
order-of-magnitude anchors.
"""
