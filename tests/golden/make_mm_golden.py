"""Record Matrix Market reader outputs from the REAL reference.

Run in the build container (the only place ``/root/reference`` exists):

    PYTHONPATH=/root/repo python tests/golden/make_mm_golden.py

Each case is a small file image; the reference's ``mmio.read_matrix_market_with_info``
result (dense matrix or CSR arrays plus ``MmInfo``) or its
``MatrixMarketError`` text is stored in ``tests/golden/mm_cases.json``.
"""

from __future__ import annotations

import io
import json
import os
import sys

import numpy as np
import scipy.sparse as sparse

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from trisolve import mmio  # noqa: E402  (the reference)

H = "%%MatrixMarket matrix"
CASES = {
    "coord_general_dups": f"{H} coordinate real general\n% a comment\n\n3 4 5\n1 1 1.5\n3 4 -2e-3\n1 1 0.25\n"
                          "2 2 1_000.5\n3 1 .5\n",
    "coord_bom_crlf": "﻿" + f"{H} coordinate real general\r\n2 2 2\r\n1 2 3.0\r\n2 1 -4\r\n",
    "coord_integer_symmetric": f"{H} coordinate integer symmetric\n3 3 4\n1 1 2\n2 1 -1\n3 2 7\n3 3 5\n",
    "coord_pattern_skew": f"{H} coordinate pattern skew-symmetric\n3 3 2\n2 1\n3 1\n",
    "coord_real_skew": f"{H} coordinate real skew-symmetric\n2 2 1\n2 1 0.75\n",
    "coord_empty": f"{H} coordinate real general\n4 5 0\n",
    "coord_upper_case_header": "%%MatrixMarket MATRIX Coordinate REAL General\n1 1 1\n1 1 +7.5E+1\n",
    "array_general": f"{H} array real general\n3 2\n1\n2\n3\n4.5\n-5\n6e1\n",
    "array_symmetric": f"{H} array real symmetric\n3 3\n1\n2\n3\n4\n5\n6\n",
    "array_skew": f"{H} array real skew-symmetric\n3 3\n1\n2\n3\n",
    "array_integer": f"{H} array integer general\n2 2\n1\n-2\n3\n4\n",
    "err_empty": "",
    "err_banner": "%%MatrixMarkt matrix coordinate real general\n1 1 0\n",
    "err_header_tokens": f"{H} coordinate real\n1 1 0\n",
    "err_object": "%%MatrixMarket vector coordinate real general\n1 1 0\n",
    "err_format": f"{H} sparse real general\n1 1 0\n",
    "err_complex": f"{H} coordinate complex general\n1 1 0\n",
    "err_field": f"{H} coordinate float general\n1 1 0\n",
    "err_hermitian": f"{H} coordinate real hermitian\n1 1 0\n",
    "err_symmetry": f"{H} coordinate real diagonal\n1 1 0\n",
    "err_array_pattern": f"{H} array pattern general\n1 1\n",
    "err_missing_size": f"{H} coordinate real general\n% only a comment\n\n",
    "err_size_tokens": f"{H} coordinate real general\n2 2\n",
    "err_size_int": f"{H} coordinate real general\n2 x 1\n1 1 1\n",
    "err_size_negative": f"{H} coordinate real general\n0 2 0\n",
    "err_array_size_tokens": f"{H} array real general\n2 2 4\n",
    "err_too_few": f"{H} coordinate real general\n2 2 3\n1 1 1\n2 2 2\n",
    "err_too_many": f"{H} coordinate real general\n2 2 1\n1 1 1\n% c\n2 2 2\n",
    "err_entry_tokens": f"{H} coordinate real general\n2 2 2\n1 1 1\n2 2\n",
    "err_entry_int": f"{H} coordinate real general\n2 2 1\n1.0 1 1\n",
    "err_index_range": f"{H} coordinate real general\n2 2 2\n1 1 1\n3 1 1\n",
    "err_upper_symmetric": f"{H} coordinate real symmetric\n2 2 1\n1 2 1\n",
    "err_skew_diagonal": f"{H} coordinate real skew-symmetric\n2 2 1\n1 1 1\n",
    "err_value": f"{H} coordinate real general\n2 2 1\n1 1 abc\n",
    "err_value_inf": f"{H} coordinate real general\n2 2 1\n1 1 inf\n",
    "err_value_nan": f"{H} coordinate real general\n2 2 1\n1 1 NaN\n",
    "err_value_hex": f"{H} coordinate real general\n2 2 1\n1 1 0x10\n",
    "err_array_entry": f"{H} array real general\n1 2\n1 2\n3\n",
    "err_array_square": f"{H} array real symmetric\n2 3\n1\n2\n3\n",
    "err_array_count": f"{H} array real general\n2 2\n1\n2\n3\n",
    "err_pattern_tokens": f"{H} coordinate pattern general\n2 2 1\n1 1 1.0\n",
}


def record(text):
    try:
        mat, info = mmio.read_matrix_market_with_info(io.StringIO(text))
    except mmio.MatrixMarketError as e:
        return {"error": str(e)}
    out = {"info": [info.format, info.field, info.symmetry, info.rows, info.cols, info.entries,
                    info.duplicates]}
    if sparse.issparse(mat):
        csr = sparse.csr_array(mat)
        out["indptr"] = csr.indptr.tolist()
        out["indices"] = csr.indices.tolist()
        out["data"] = [float(v).hex() for v in csr.data]
        out["shape"] = list(csr.shape)
    else:
        out["dense"] = [float(v).hex() for v in np.asarray(mat).ravel()]
        out["shape"] = list(mat.shape)
    return out


def main():
    res = {name: {"text": text, "expect": record(text)} for name, text in CASES.items()}
    with open(os.path.join(HERE, "mm_cases.json"), "w") as fh:
        json.dump(res, fh, indent=1, sort_keys=True)
    for k, v in res.items():
        print(k, v["expect"].get("error", v["expect"].get("info")))


if __name__ == "__main__":
    main()
