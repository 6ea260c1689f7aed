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


def test_bench_rows(capsys, monkeypatch):
    """The reference's CSV columns, then device_ms and matvec_gbs; rows on a
    TRISOLVE_WORKERS thread pool spread over --gpus devices give the same
    rows as the serial run."""
    from paper_2304_12168_b200.cli import main

    argv = ["bench", "--gen", "clement:101", "--gen", "convdiff:20", "--algo", "cta",
            "--algo", "ta", "--trials", "1", "--max-iters", "200"]
    assert main(argv) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines[0] == ("family,n,algo,iterations,wall_ms,residual,normal_residual,outcome,"
                        "device_ms,matvec_gbs")
    assert len(lines) == 5 and not any("error" in ln for ln in lines[1:])
    for ln in lines[1:]:
        cols = ln.split(",")
        assert float(cols[8]) > 0 and float(cols[9]) > 0  # device time and pair GB/s
    monkeypatch.setenv("TRISOLVE_WORKERS", "3")
    assert main(argv + ["--gpus", "2"]) == 0
    pooled = capsys.readouterr().out.strip().splitlines()
    key = lambda ln: [c for i, c in enumerate(ln.split(",")) if i not in (4, 8, 9)]  # noqa: E731
    assert [key(ln) for ln in pooled] == [key(ln) for ln in lines]


@pytest.mark.parametrize("spec,algo", [("poisson-d:40", "cta"), ("clement:301", "ta"),
                                       ("diag-pd:200", "lpfeas")])
def test_solve_on_two_gpus_matches_one(spec, algo, tmp_path, capsys):
    """solve --gpus 2 (one sharded solve, two ranks; on a one-GPU box both
    ranks share it) reaches the outcome and iteration count of --gpus 1, and
    inside the 40-iteration parity window the same residual."""
    from paper_2304_12168_b200.cli import main

    outs = []
    for gpus in ("1", "2"):
        summ = tmp_path / f"s{gpus}.json"
        rc = main(["solve", "--gen", spec, "--algo", algo, "--eps", "1e-8", "--max-iters", "40",
                   "--gpus", gpus, "--summary", str(summ), "--dump-x", str(tmp_path / f"x{gpus}.mtx")])
        capsys.readouterr()
        outs.append((rc, json.loads(summ.read_text())))
    (rc1, s1), (rc2, s2) = outs
    assert rc1 == rc2 and s1["outcome"] == s2["outcome"] and s1["iterations"] == s2["iterations"]
    assert s2["final_residual_norm"] == pytest.approx(s1["final_residual_norm"], rel=1e-6, abs=1e-12)
