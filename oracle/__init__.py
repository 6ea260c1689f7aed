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
            arithmetic of the dense TA path (launch geometry, FMA chains, warp /
            block reduction trees, split-tile merges), used for the bitwise
            checks of the CUDA kernels in ``tests/test_gpu_mirror.py`` (C1 TA at
            500 iterations, BASELINE configs[0]); ``oracle/Makefile`` builds
            ``oracle/_build/libmirror.so``.

Parity pinning: ``tests/golden/make_golden.py`` imports the real reference
(present only in the build container) and records its outputs as fixtures;
``tests/test_oracle_golden.py`` checks ``port`` against every fixture.
"""
