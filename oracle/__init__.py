"""CPU oracle for the TA / CTA / TA-LP iteration path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import anything from this package, and only as the
checker or the timed CPU baseline — never as part of the product path.  The
product (``paper_2304_12168_b200``) never imports it and fails loudly when its
CUDA library is missing.

Contents
--------
``port``    numpy/scipy restatement of the reference algorithm
            (``/root/reference/pkg/src/trisolve/{linalg,centering,triangle,feasibility}.py``);
            each function cites the reference file:line it restates and uses the
            same numpy/BLAS/LAPACK primitives so its arithmetic matches the
            reference call for call.
``mirror``  ctypes binding of ``mirror.c``: a plain-C restatement of the *device*
            kernels' exact reduction order, used for bitwise checks of the CUDA
            kernels (``oracle/Makefile`` builds ``oracle/_ref/libmirror.so``).

Parity pinning: ``tests/golden/make_golden.py`` imports the real reference
(present only in the build container) and records its outputs as fixtures;
``tests/test_oracle_golden.py`` checks ``port`` against every fixture.
"""
