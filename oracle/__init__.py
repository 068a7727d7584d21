"""Plain, slow, CPU fp64 ORACLE for the all-at-once Crank-Nicolson method with the
block alpha-circulant preconditioner (arxiv 2401.16113, /root/reference/PAPER.md).

THIS PACKAGE IS TEST INFRASTRUCTURE.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.
The product path (``paper_2401_16113_b200``) never imports, calls or links it, and
this package never imports the product path.  The two share only the seeded input
generator ``synth`` (parameters + random numbers, no arithmetic of the method).

Every function cites the PAPER.md passage it follows ("PAPER.md:<line>" plus the
section / equation).  Notation follows SURVEY.md §0: N = number of time steps
(the paper's M), m = number of spatial unknowns (the paper's N), Ã = τ L_h.

Modules
-------
problem   grid, spatial operator L_h, manufactured solution, source f, rhs b (Eq. 2.1-2.2)
aao       𝓜u, P_α z by the block formulas (§3.2), sequential CN, dense 𝓜 / P_α (tiny sizes)
precond   λ tables (Eq. eigCx, FFT-consistent reading), DFT-matrix P_α⁻¹ (Eq. 3.2 + Remark 3.1),
          full-spectrum variant, 2D dense-DST fast diagonalisation, FFT-free fixed-point sweep,
          dense solve
gmres     restarted right-preconditioned GMRES (MGS + Givens), §5 / PAPER.md:795; left-preconditioned
          GMRES (§4) and the Theorem 4.5 rate bound
spectrum  dense eigenvalues of P_α⁻¹𝓜 and the closed forms of Lemma 3.1 / Theorem 3.1

Parity status: every function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py``; none is "parity unpinned".
"""
