"""Polar Express fp64 CPU oracle -- TEST INFRASTRUCTURE ONLY.

This package is the plain, slow, obviously-correct reference for what the
Polar Express hot path computes (arXiv 2505.16932, /root/reference/PAPER.md,
cited below as ``P:<line>``).  It exists to *check* the CUDA path; it is not
part of it.

Import rules (enforced by review, relied on by the parity claims):
  * Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
    ``cpu_baseline`` / ``--impl reference`` legs may import anything here.
  * The product package ``paper_2505_16932_b200`` never imports ``oracle``,
    and ``oracle`` never imports the product package.  The two share no
    arithmetic, headers, tables or helpers; only the seeded input generators
    in ``pe_synth`` (which contain none of the method's arithmetic) serve both.

Modules:
  coeffs     -- offline stage: Listing 1 / Alg. 2
                greedy minimax composition, degree-3 closed form,
                safety factor, online table readings R4/R5.
  iteration  -- online stage: Listing 2 in fp64, exact polar via
                SVD, scalar composite map.
  metrics    -- App. E.1 error measures.
  emulate    -- bf16 rounding-point emulation of the GPU design (DESIGN.md
                reading R8) for inputs where it is exact (diagonal inputs).

Every function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle.py`` against something other than itself (values the
paper prints, closed forms, brute force, independent decompositions).
Functions with no such pin say "parity unpinned" in their docstring; there
are none at present.
"""
