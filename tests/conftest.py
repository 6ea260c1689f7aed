"""Shared test plumbing: the ``gpu`` marker, golden-fixture loading, and the
CPU oracle call recipes used by both the oracle-pinning tests (CPU) and the
device parity tests (``-m gpu``)."""

from __future__ import annotations

import glob
import json
import os
import sys

# The recorded fixtures were made with one BLAS thread; keep the oracle's
# dense reductions in the same order.
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import numpy as np  # noqa: E402
import pytest  # noqa: E402
import scipy.sparse as sparse  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

EVENTS = ("pivot", "expand", "witness", "shrink")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def golden_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                  if not os.path.basename(p).startswith("kat_")
                  and os.path.basename(p) != "gallery.npz")


class Golden:
    """One recorded reference run (inputs + outputs)."""

    def __init__(self, name):
        self.name = name
        z = np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False)
        self.z = z
        if str(z["a_kind"]) == "csr":
            shape = tuple(int(s) for s in z["a_shape"])
            self.a = sparse.csr_array((z["a_data"], z["a_indices"], z["a_indptr"]), shape=shape)
        else:
            self.a = z["a"]
        self.b = z["b"]
        self.solver = str(z["solver"])
        self.kwargs = json.loads(str(z["kwargs"]))
        self.status = str(z["status"])
        self.detail = str(z["detail"])
        self.iterations = int(z["iterations"])
        self.x = z["x"]
        self.residual_norm = float(z["residual_norm"])
        self.normal_residual_norm = float(z["normal_residual_norm"])
        self.trace = z["trace"]
        self.trace_columns = tuple(str(c) for c in z["trace_columns"])
        self.extras = {k: (z[k] if z[k].ndim else float(z[k]))
                       for k in ("rho", "lower_bound", "min_x_entry", "b_prime") if k in z.files}
        self.x_eps = z["x_eps"] if "x_eps" in z.files else None
        self.rho_interval = tuple(z["rho_interval"]) if "rho_interval" in z.files else None
        self.stage_status = [str(v) for v in z["stage_status"]] if "stage_status" in z.files else None
        self.stage_iterations = ([int(v) for v in z["stage_iterations"]]
                                 if "stage_iterations" in z.files else None)


@pytest.fixture(params=golden_names())
def golden(request):
    return Golden(request.param)


def trace_rows_numeric(rows, columns):
    """Turn result trace rows (with wall_ns and string events) into the
    float matrix layout the fixtures store."""
    out = []
    for row in rows:
        vals = []
        for col, v in zip(columns, row):
            if col == "wall_ns":
                continue
            if col == "event":
                vals.append(float(EVENTS.index(v)))
            elif col == "stage":
                vals.append(1.0 if v == "stage1" else 2.0)
            else:
                vals.append(float(v))
        out.append(vals)
    return np.array(out, dtype=np.float64).reshape(len(rows), len(columns) - 1)


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = max(float(np.linalg.norm(b)), 1e-300)
    return float(np.linalg.norm(a - b)) / den
