"""Command line (paper_2304_12168_b200.cli): argument handling, exit codes and
the generate path on CPU; the device solves run in tests/test_gpu_cli.py."""

from __future__ import annotations

import numpy as np
import pytest


def test_usage_errors_exit_1(capsys):
    from paper_2304_12168_b200.cli import main

    assert main([]) == 1
    assert main(["solve"]) == 1  # needs --mtx or --gen
    assert main(["solve", "--gen", "clement"]) == 1  # bad spec
    assert main(["solve", "--gen", "clement:x"]) == 1
    assert main(["solve", "--mtx", "/nonexistent.mtx"]) == 1
    assert main(["solve", "--gen", "clement:5", "--device", "tpu"]) == 1
    assert main(["bench"]) == 1  # needs a --gen
    assert "error:" in capsys.readouterr().err


def test_generate_writes_matrix_market(tmp_path):
    from paper_2304_12168_b200 import gallery, mmio
    from paper_2304_12168_b200.cli import main

    out = tmp_path / "c.mtx"
    assert main(["generate", "--gen", "convdiff:6:2,0.5,3", "--out", str(out)]) == 0
    a = mmio.read_matrix_market(str(out))
    ref = gallery.make("convdiff", 6, [2.0, 0.5, 3.0])
    assert (a != ref).nnz == 0 and np.array_equal(a.data, ref.data)
    assert main(["generate", "--gen", "nope:5", "--out", str(out)]) == 1


def test_gen_spec_parsing():
    from paper_2304_12168_b200.cli import UsageError, parse_gen_spec

    assert parse_gen_spec("dorr:100:0.01") == ("dorr", 100, [0.01])
    assert parse_gen_spec("convdiff:5:1,2,3") == ("convdiff", 5, [1.0, 2.0, 3.0])
    with pytest.raises(UsageError):
        parse_gen_spec("dorr:100:a,b")
