"""Bitwise device checks against the C mirror of the device arithmetic
(oracle/mirror.c).  BASELINE configs[0] asks for "TA at fixed 500 iterations
for the bitwise-path check (runs on CPU)": the numpy oracle cannot serve there
(the reference disagrees with itself at 1e-3 after 500 iterations once only
the BLAS reduction order changes), so the CPU side is a
restatement of the GPU's own reduction order, and the device run must match
it bit for bit — x, every trace row, the final residuals."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import mirror
from paper_2304_12168_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _sms():
    import torch

    return torch.cuda.get_device_properties(0).multi_processor_count


def _device_vs_mirror(a, b, eps, its):
    import paper_2304_12168_b200 as ts

    dev = ts.solve_adaptive(ts.DeviceMatrix(a), b, eps=eps, max_iters=its)
    mr = mirror.ta_dense(a, b, eps, its, sms=_sms())
    assert dev.status == mr["status"] and dev.iterations == mr["iterations"]
    assert np.array_equal(dev.x, mr["x"])
    rows = np.array([[r[0], {"pivot": 0, "expand": 1}[r[4]], r[1], r[2], r[3]] for r in dev.trace.rows])
    assert rows.shape == mr["trace"].shape
    assert np.array_equal(rows, mr["trace"])
    assert dev.residual_norm == mr["residual_norm"]
    assert dev.normal_residual_norm == mr["normal_residual_norm"]
    assert dev.rho == mr["rho"]


def test_c1_ta_500_bitwise():
    w = W.dense_gaussian()  # BASELINE configs[0]: 1000 x 1000, seed 0
    _device_vs_mirror(w.a, w.b, 1e-8 * float(np.linalg.norm(w.b)), 500)


@pytest.mark.parametrize("m,n,seed,its", [(333, 777, 2, 150), (1000, 129, 3, 120), (517, 200, 5, 150),
                                          (150, 130, 7, 700),
                                          # A v group edges: > 256 row groups (strided slot
                                          # reduction), fewer rows than one group over many tiles
                                          (70001, 130, 11, 30), (3, 5000, 13, 40)])
def test_odd_shapes_and_revalidation_bitwise(m, n, seed, its):
    w = W.dense_gaussian(m, n, seed=seed)
    _device_vs_mirror(w.a, w.b, 1e-12 * float(np.linalg.norm(w.b)), its)
