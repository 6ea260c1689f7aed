"""Gallery families (paper_2304_12168_b200.gallery) against matrices recorded
from the REAL reference (tests/golden/make_gallery_golden.py): identical
structure and bit-identical values.  CPU only; the device-generated families
are checked in tests/test_gpu_gallery.py."""

from __future__ import annotations

import os

import numpy as np
import pytest
import scipy.sparse as sparse

from conftest import GOLDEN

Z = np.load(os.path.join(GOLDEN, "gallery.npz"))
IDS = list(range(int(Z["count"])))


def spec(i):
    fam, n, params, seed = (str(v) for v in Z[f"c{i}_spec"])
    return fam, int(n), [float(p) for p in params.split(",") if p], int(seed)


@pytest.mark.parametrize("i", IDS, ids=[spec(i)[0] + f"_{i}" for i in IDS])
def test_family_matches_reference(i):
    from paper_2304_12168_b200 import gallery

    fam, n, params, seed = spec(i)
    a = gallery.make(fam, n, params, seed)
    if f"c{i}_dense" in Z:
        assert isinstance(a, np.ndarray)
        assert np.array_equal(a, Z[f"c{i}_dense"])
    else:
        a = sparse.csr_array(a)
        assert tuple(a.shape) == tuple(Z[f"c{i}_shape"])
        assert np.array_equal(a.indptr, Z[f"c{i}_indptr"])
        assert np.array_equal(a.indices, Z[f"c{i}_indices"])
        assert np.array_equal(a.data, Z[f"c{i}_data"])


def test_unknown_family_and_bad_sizes():
    from paper_2304_12168_b200 import gallery

    with pytest.raises(ValueError, match="unknown family"):
        gallery.make("nope", 5)
    with pytest.raises(ValueError):
        gallery.gen_clement(1)
    with pytest.raises(ValueError):
        gallery.gen_convdiff(5, 1.0, -1.0, 1.0)
