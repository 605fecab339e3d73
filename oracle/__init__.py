"""CPU oracle for the SMC registration hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this package.  It is the checker, never
the thing measured for the product path and never shipped inside
``paper_2504_19930_b200``.

* ``oracle.kernels`` -- ctypes binding of ``echoreg_oracle.c``, a C
  restatement of the reference's numba kernels (bit-exact, pinned by
  ``tests/test_oracle.py`` against golden vectors from the real reference).
* ``oracle.smc`` -- numpy restatement of the reference SMC loop
  (``echoreg/smc.py``) driving ``oracle.kernels``.
"""
