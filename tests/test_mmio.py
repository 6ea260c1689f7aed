"""Matrix Market ingest (paper_2304_12168_b200.mmio, native parser) against
outputs recorded from the REAL reference reader (tests/golden/make_mm_golden.py):
values bit-exact, MmInfo identical, and every malformed input rejected with the
reference's MatrixMarketError text.  CPU only (parsing is host work; the
device assembly is checked in tests/test_gpu_ingest.py)."""

from __future__ import annotations

import io
import json
import os

import numpy as np
import pytest
import scipy.sparse as sparse

from conftest import GOLDEN

with open(os.path.join(GOLDEN, "mm_cases.json")) as _fh:
    CASES = json.load(_fh)


@pytest.mark.parametrize("name", sorted(CASES))
def test_reader_matches_reference(name, tmp_path):
    from paper_2304_12168_b200 import mmio

    case = CASES[name]
    exp = case["expect"]
    for source in (io.StringIO(case["text"]), io.BytesIO(case["text"].encode("utf-8")), None):
        if source is None:
            path = tmp_path / "m.mtx"
            path.write_bytes(case["text"].encode("utf-8"))
            source = str(path)
        if "error" in exp:
            with pytest.raises(mmio.MatrixMarketError) as ei:
                mmio.read_matrix_market_with_info(source)
            assert str(ei.value) == exp["error"]
            continue
        mat, info = mmio.read_matrix_market_with_info(source)
        assert [info.format, info.field, info.symmetry, info.rows, info.cols, info.entries,
                info.duplicates] == exp["info"]
        if "dense" in exp:
            assert isinstance(mat, np.ndarray) and list(mat.shape) == exp["shape"]
            assert [float(v).hex() for v in mat.ravel()] == exp["dense"]
        else:
            assert sparse.issparse(mat) and list(mat.shape) == exp["shape"]
            assert mat.indptr.tolist() == exp["indptr"]
            assert mat.indices.tolist() == exp["indices"]
            assert [float(v).hex() for v in mat.data] == exp["data"]


def test_write_read_roundtrip_bit_exact(tmp_path):
    from paper_2304_12168_b200 import mmio

    rng = np.random.default_rng(3)
    dense = rng.standard_normal((7, 5)) * 10.0 ** rng.integers(-300, 300, size=(7, 5))
    sp = sparse.random_array((40, 30), density=0.2, random_state=4, format="csr")
    for a in (dense, sp):
        buf = io.StringIO()
        mmio.write_matrix_market(a, buf)
        back = mmio.read_matrix_market(io.StringIO(buf.getvalue()))
        if sparse.issparse(a):
            assert (back != a).nnz == 0 and np.array_equal(back.data, sparse.csr_array(a).data)
        else:
            assert np.array_equal(back, a)
    p = tmp_path / "d.mtx"
    mmio.write_matrix_market(dense, str(p))
    assert np.array_equal(mmio.read_matrix_market(str(p)), dense)


def test_writer_format_matches_reference_layout():
    from paper_2304_12168_b200 import mmio

    buf = io.StringIO()
    mmio.write_matrix_market(sparse.csr_array(np.array([[0.0, 2.5], [1e-300, 0.0]])), buf)
    assert buf.getvalue() == "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 2 2.5\n2 1 1e-300\n"
    buf = io.StringIO()
    mmio.write_matrix_market(np.array([[1.0, 2.0], [3.0, 4.0]]), buf)
    assert buf.getvalue() == "%%MatrixMarket matrix array real general\n2 2\n1.0\n3.0\n2.0\n4.0\n"
