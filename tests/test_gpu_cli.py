"""Command line on the device: solve from a generated family and from a Matrix
Market file, with the reference's summary schema and exit codes."""

from __future__ import annotations

import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_solve_generated_and_file(tmp_path, capsys):
    from paper_2304_12168_b200 import gallery, mmio
    from paper_2304_12168_b200.cli import SUMMARY_KEYS, main

    summ = tmp_path / "s.json"
    rc = main(["solve", "--gen", "poisson-d:30", "--algo", "cta", "--eps", "1e-8", "--device", "cuda:0",
               "--summary", str(summ), "--trace", str(tmp_path / "t.csv")])
    assert rc == 0
    s = json.loads(summ.read_text())
    assert set(s) <= set(SUMMARY_KEYS) and s["outcome"] in ("approx_solution", "normal_eq_solution")
    assert s["matrix"] == {"m": 900, "n": 900, "nnz": 4380, "family": "poisson-d"}
    if s["outcome"] == "approx_solution":
        assert s["final_relative_residual"] <= 1e-8 * (1 + 1e-9)
    capsys.readouterr()
    # the same matrix from a file: same outcome and iteration count
    p = tmp_path / "p.mtx"
    mmio.write_matrix_market(gallery.make("poisson-d", 30), str(p))
    rc2 = main(["solve", "--mtx", str(p), "--algo", "cta", "--eps", "1e-8"])
    s2 = json.loads(capsys.readouterr().out)
    assert rc2 == 0 and s2["iterations"] == s["iterations"] and s2["outcome"] == s["outcome"]
    # witness / iteration cap map to exit codes 2 / 3 (cli.py:46-55)
    assert main(["solve", "--gen", "clement:301", "--algo", "ta", "--max-iters", "5"]) == 3
    capsys.readouterr()


def test_bench_rows(capsys):
    from paper_2304_12168_b200.cli import main

    assert main(["bench", "--gen", "clement:101", "--gen", "convdiff:20", "--algo", "cta",
                 "--algo", "ta", "--trials", "1", "--max-iters", "200"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines[0] == "family,n,algo,iterations,wall_ms,residual,normal_residual,outcome"
    assert len(lines) == 5 and not any("error" in ln for ln in lines[1:])
