"""CPU oracle — TEST INFRASTRUCTURE ONLY.

A CPU restatement of the reference ``splatcull`` render path (stages c–e) and
of the SPEC-only scene / visibility-MLP path (stages a–b).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package, and only as the checker or the
CPU baseline.  The product package ``paper_2511_19202_b200`` never imports it.

* ``oracle.raster_ref``  — reference ``raster.render`` glue (numpy, same ops)
  over the C kernels in ``sc_oracle.c`` (numba kernels restated in C, f64,
  no FMA, glibc ``exp``).  Pinned bit-exact against golden vectors generated
  by the reference itself (``oracle/gen_golden.py`` -> ``tests/golden/``).
* ``oracle.scene_ref``   — restatement of SPEC ``scene`` / ``nn`` (the
  reference package does not ship them).  Parity for these stages is pinned
  only by the SPEC's own known-answer examples and invariants — "parity
  unpinned" against reference code, because no reference code exists.
"""
