"""CPU oracle for the tiled D3Q19 LBGK step -- TEST INFRASTRUCTURE ONLY.

This package is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` may import it.  The product path
(``paper_1611_02445_b200``) never imports it and fails loudly when its CUDA
library is missing.

Contents
--------
numerics.py    numpy restatement of the reference arithmetic
               (collision.py:46-130, boundaries.py:53-195) in the reference's
               exact operation order.
tiling.py      numpy restatement of build_tiling (tiling.py:51-83),
               _neighbor_indices (txmodel.py:145-160), _tile_nonsolid_blocks
               (txmodel.py:163-173) and the layout tables (layout.py:45-112).
dense.py       numpy restatement of the step on the
               dense grid -- the "naive dense two-array solver" of SPEC.md:399.
tlbm_oracle.c  the same step in plain C (OpenMP over x planes, no FMA
               contraction); bit-identical to dense.py and ~100x faster, used
               for 1000-step parity runs and as the timed CPU baseline.
c_oracle.py    ctypes wrapper of tlbm_oracle.c (built by oracle/Makefile into
               oracle/build/liboracle.so).

Pinning: the reference ships no tests and no step.  numerics.py / tiling.py are
pinned bit-exactly against the reference's own functions (imported from
/root/reference in the dev container) and against the golden vectors in
tests/golden/ (made by tests/golden/make_golden.py from the reference).  The
step glue (dense.py) composes only pinned pieces and is checked against SPEC's
property pins (fixed point, conservation, tiled == dense, layout invariance).
"""
