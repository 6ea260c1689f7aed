"""Device-generated gallery families (ts_matrix_gen_stencil5 / _clement)
against the host generators, which tests/test_gallery.py pins bit-for-bit to
the reference: same shape, nnz and bitwise matvecs in both orientations (the
CSR kernels add every row in scipy's order)."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [("clement", 7, []), ("clement", 100001, []), ("poisson-d", 5, []), ("poisson-n", 6, []),
         ("convdiff", 5, []), ("convdiff", 300, [2.0, 0.5, 3.0]), ("poisson-d", 1000, []),
         ("dorr", 50, [0.05]), ("lotkin", 40, [])]


@pytest.mark.parametrize("fam,n,params", CASES, ids=[f"{c[0]}_{c[1]}" for c in CASES])
def test_device_family_equals_host(fam, n, params):
    from paper_2304_12168_b200 import gallery

    host = gallery.make(fam, n, params)
    dm = gallery.make_device(fam, n, params)
    assert dm.shape == host.shape
    rng = np.random.default_rng(n)
    v = rng.standard_normal(host.shape[1])
    w = rng.standard_normal(host.shape[0])
    if fam in gallery.DEVICE_FAMILIES:
        assert dm.nnz == host.nnz
        assert np.array_equal(dm.matvec(v), host @ v)
        assert np.array_equal(dm.rmatvec(w), w @ host)
    else:  # host-built and uploaded (dense ones: BLAS order, not bitwise)
        ref = host @ v
        assert np.linalg.norm(dm.matvec(v) - ref) <= 1e-13 * np.linalg.norm(abs(host) @ abs(v))
    vals = np.asarray(host).ravel() if isinstance(host, np.ndarray) else host.data
    assert dm.frobenius_norm() == pytest.approx(float(np.sqrt((vals * vals).sum())), rel=1e-13)
