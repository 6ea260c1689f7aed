"""CPU-side checks of the drop-in boundary: the C-ABI library loads and
exports every symbol include/trisolve_b200.h declares; the Python layer
mirrors the reference's public names and validation errors (no GPU needed)."""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "trisolve_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^TS_API\s+[\w\s\*]+?\b(ts_\w+)\(", src, flags=re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for need in ("ts_cta_solve", "ts_ta_adaptive", "ts_ta_in_ball", "ts_lp_feasibility",
                 "ts_matvec", "ts_rmatvec", "ts_matrix_create_dense", "ts_matrix_create_csr"):
        assert need in syms


def test_library_exports_every_declared_symbol():
    from paper_2304_12168_b200 import _native

    lib = _native.load_library()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert set(declared_symbols()) == set(_native.EXPORTS)
    assert lib.ts_abi_version() == _native.ABI_VERSION == 2


def test_struct_layouts_match_header(tmp_path):
    """Compile the header with gcc and compare sizeof/offsetof with ctypes."""
    import shutil
    import subprocess

    from paper_2304_12168_b200 import _native as N
    from paper_2304_12168_b200 import mmio

    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    structs = {"ts_trace_row": N.TraceRow, "ts_result": N.Result, "ts_cta_options": N.CtaOptions,
               "ts_ta_options": N.TaOptions, "ts_ball_options": N.BallOptions,
               "ts_lp_options": N.LpOptions, "ts_mm_info": mmio._Info}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    for cname, cls in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-o", str(exe), str(src)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], check=True, capture_output=True,
                                                       text=True).stdout.splitlines())
    for cname, cls in structs.items():
        assert int(got[cname]) == ctypes.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(cls, fname).offset, (cname, fname)


def test_public_names_mirror_reference():
    import paper_2304_12168_b200 as ts

    for name in ("centering_solve", "CenteringOptions", "solve_adaptive", "solve_in_ball",
                 "nonnegative_feasibility", "SolveResult", "Trace", "HOperator", "GramProduct",
                 "matvec", "matvec_transpose", "norm2", "APPROX_SOLUTION", "NORMAL_EQ_SOLUTION",
                 "WITNESS", "FEASIBLE", "INCONCLUSIVE", "ITERATION_CAP", "NUMERICAL_FAILURE"):
        assert hasattr(ts, name), name


def test_options_validation_matches_reference():
    from paper_2304_12168_b200 import CenteringOptions

    with pytest.raises(ValueError, match="epsilon"):
        CenteringOptions(epsilon=2.0).validated(3)
    with pytest.raises(ValueError, match="t_max"):
        CenteringOptions(t_max=0).validated(3)
    with pytest.raises(ValueError, match="h_mode"):
        CenteringOptions(h_mode="x").validated(3)
    with pytest.raises(ValueError, match="start"):
        CenteringOptions(start="nope").validated(3)
    assert CenteringOptions(t_max=9).validated(4).t_max == 4


def test_result_and_trace_contract():
    from paper_2304_12168_b200.results import (CENTERING_TRACE_COLUMNS, SolveResult, Trace)

    tr = Trace(CENTERING_TRACE_COLUMNS)
    tr.append(0, 1, 2.0, 3.0, 4)
    with pytest.raises(ValueError):
        tr.append(1, 2)
    assert tr.column("t") == [1]
    r = SolveResult("approx_solution", np.zeros(2), 0.0, 0.0, 0, tr)
    assert r.success


def test_schedule_matches_reference_wave():
    from paper_2304_12168_b200.centering import _order_schedule

    gen = _order_schedule(5)
    assert [next(gen) for _ in range(12)] == [1, 2, 3, 4, 5, 4, 3, 2, 1, 2, 3, 4]


def test_missing_library_fails_loudly(tmp_path):
    from paper_2304_12168_b200 import _native

    with pytest.raises(RuntimeError, match="no CPU fallback"):
        # a fresh loader pointed at a missing file must not silently fall back
        saved = _native._lib
        _native._lib = None
        try:
            _native.load_library(str(tmp_path / "missing.so"))
        finally:
            _native._lib = saved
