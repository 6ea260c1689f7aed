"""Device-side Matrix Market ingest (ts_mm_to_device): the CSR assembled on
the device (mirroring, radix sort, duplicate summation, compression) is the
reference reader's CSR — checked through bitwise matvecs against the host
read, on the recorded reference cases and on full-size files."""

from __future__ import annotations

import io
import json
import os

import numpy as np
import pytest
import scipy.sparse as sparse

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

with open(os.path.join(GOLDEN, "mm_cases.json")) as _fh:
    CASES = json.load(_fh)
COORD = sorted(k for k, v in CASES.items() if "indptr" in v["expect"] and v["expect"]["indices"])


def _same_operator(dm, csr):
    rng = np.random.default_rng(1)
    v = rng.standard_normal(csr.shape[1])
    w = rng.standard_normal(csr.shape[0])
    assert dm.shape == csr.shape and dm.nnz == csr.nnz
    assert np.array_equal(dm.matvec(v), csr @ v)
    assert np.array_equal(dm.rmatvec(w), w @ csr)


@pytest.mark.parametrize("name", COORD)
def test_device_ingest_matches_reference_cases(name):
    from paper_2304_12168_b200 import mmio

    text = CASES[name]["text"]
    exp = CASES[name]["expect"]
    dm, info = mmio.read_matrix_market_device(io.StringIO(text))
    assert info.duplicates == exp["info"][6]
    csr = sparse.csr_array(([float.fromhex(h) for h in exp["data"]], exp["indices"], exp["indptr"]),
                           shape=tuple(exp["shape"]))
    _same_operator(dm, csr)


def test_device_ingest_full_size_general_and_symmetric(tmp_path):
    from paper_2304_12168_b200 import mmio
    from paper_2304_12168_b200 import workloads as W

    a = W.convdiff_upwind(1000).a  # C4: 10^6 x 10^6, 4,996,000 entries (> one capped grid)
    p = tmp_path / "a.mtx"
    mmio.write_matrix_market(a, str(p))
    dm, info = mmio.read_matrix_market_device(str(p))
    assert info.duplicates == 0
    _same_operator(dm, a)
    # symmetric file: the lower triangle of A + A^T, mirrored on the device
    s = sparse.csr_array(a + a.T)
    low = sparse.tril(s, format="coo")
    lines = [f"%%MatrixMarket matrix coordinate real symmetric\n{s.shape[0]} {s.shape[1]} {low.nnz}\n"]
    lines += [f"{i + 1} {j + 1} {float(v)!r}\n" for i, j, v in zip(low.row, low.col, low.data)]
    q = tmp_path / "s.mtx"
    q.write_text("".join(lines))
    dm2, info2 = mmio.read_matrix_market_device(str(q))
    host = mmio.read_matrix_market(str(q))
    assert info2.symmetry == "symmetric"
    _same_operator(dm2, host)


def test_device_ingest_then_solve():
    import paper_2304_12168_b200 as ts
    from paper_2304_12168_b200 import mmio
    from paper_2304_12168_b200 import workloads as W

    w = W.clement_variant(2001, seed=3)
    buf = io.StringIO()
    mmio.write_matrix_market(w.a, buf)
    dm, _ = mmio.read_matrix_market_device(io.StringIO(buf.getvalue()))
    opts = ts.CenteringOptions(epsilon=1e-8, max_iters=30)
    got = ts.centering_solve(dm, w.b, opts)
    ref = ts.centering_solve(ts.DeviceMatrix(w.a), w.b, opts)
    assert got.iterations == ref.iterations and np.array_equal(got.x, ref.x)
