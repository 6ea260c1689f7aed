"""The opt-in persistent CTA loop (TS_PERSIST=1, csrc/ts_persist.cuh) must be
parity-green like the graph path: same status / iterations and iterates
within 1e-9 of the oracle inside the parity window.

TS_PERSIST is read once per process, so the check runs in a subprocess."""

from __future__ import annotations

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np
import paper_2304_12168_b200 as ts
from paper_2304_12168_b200 import workloads as W
from oracle import port
from conftest import rel_l2

for name, iters in (("c1", 40), ("c3", 30)):
    w = W.make(name)
    dev = ts.centering_solve(ts.DeviceMatrix(w.a), w.b, ts.CenteringOptions(epsilon=1e-8, max_iters=iters))
    ref = port.cta_solve(w.a, w.b, epsilon=1e-8, max_iters=iters)
    assert dev.status == ref["status"], (name, dev.status, ref["status"])
    assert dev.iterations == ref["iterations"], (name, dev.iterations, ref["iterations"])
    err = rel_l2(dev.x, ref["x"])
    assert err <= 1e-9, (name, err)
    # one cooperative launch per segment instead of ~10 kernels per iteration
    assert dev.kernel_launches < dev.iterations, (name, dev.kernel_launches, dev.iterations)
    print(name, "ok", dev.iterations, err, dev.kernel_launches)
"""


def test_persistent_cta_loop_window_parity():
    # the persistent loop runs dense A^T v as column tiles: keep small dense
    # matrices off the transposed-copy plan (PLAN_TRANS) it does not cover
    env = dict(os.environ, TS_PERSIST="1", TS_DENSE_T="cols")
    out = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.count(" ok ") == 2, out.stdout
