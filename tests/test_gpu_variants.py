"""Launch-structure variants of the device loops must not change a single bit.

The switches are read once per process, so every variant runs in its own
interpreter (``tests/_variant_probe.py`` prints digests of the iterates):

* the CTA period graph (default: one WHILE trip = one period of the order
  schedule, no SWITCH node) against the WHILE{SWITCH} graph (TS_CTA_SWITCH=1)
  and against direct launches (TS_NO_GRAPH=1), including a recheck cadence
  that falls in mid-period (``recheck_every=3``) — the in-graph recheck against
  the host-driven one;
* the in-graph 512-pivot revalidation of TA against the host-driven one;
* one-kernel moment pairs on a square banded matrix (k_pair_band) and on a
  small dense matrix (k_pair_wdense, cooperative, grid barrier between the two
  products) against the two passes (TS_BAND_PAIR=0, TS_DENSE_PAIR=0), and all
  pairs of an iteration chained in one kernel (k_chain_wdense, the default for
  small dense matrices; k_chain_csr for L2-resident short-row CSR) against one
  kernel per pair (TS_DENSE_CHAIN=0, TS_CSR_CHAIN=0);
* the candidate and update passes of small systems in one single-block kernel
  (k_vec2) against two kernels (TS_VEC_FUSE=0), and run by the chain kernel's
  last block (a whole iteration in one kernel) against a kernel of their own
  (TS_CHAIN_TAIL=0);
* the warp-per-row small dense kernel against the tile kernel
  (TS_DENSE_SMALL=tile): same statuses and iteration counts, iterates within
  north_star's 1e-9 (the dot products are summed in another order, and TA
  amplifies the last-bit differences over its iterations);
* the small dense kernel against numpy on odd shapes (n not a multiple of 64,
  fewer rows than warps, more rows than one wave).
"""

from __future__ import annotations

import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _probe(**env):
    e = dict(os.environ)
    for k in ("TS_CTA_SWITCH", "TS_NO_GRAPH", "TS_BAND_PAIR", "TS_DENSE_PAIR", "TS_DENSE_CHAIN", "TS_CSR_CHAIN", "TS_VEC_FUSE", "TS_CHAIN_TAIL", "TS_DENSE_SMALL"):
        e.pop(k, None)
    e.update(env)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "_variant_probe.py")], env=e, cwd=ROOT,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.fixture(scope="module")
def default_run():
    return _probe()


@pytest.mark.parametrize("env", [{"TS_CTA_SWITCH": "1"}, {"TS_NO_GRAPH": "1"}, {"TS_BAND_PAIR": "0"},
                                 {"TS_DENSE_PAIR": "0"}, {"TS_DENSE_CHAIN": "0"}, {"TS_CSR_CHAIN": "0"},
                                 {"TS_CSR_CHAIN": "0", "TS_BAND_PAIR": "0"}, {"TS_VEC_FUSE": "0"},
                                 {"TS_CHAIN_TAIL": "0"}],
                         ids=["switch_graph", "direct_launches", "two_pass_band_pairs", "two_pass_dense_pairs",
                              "dense_pair_kernels", "csr_pair_passes", "csr_two_passes", "separate_vector_kernels",
                              "vector_kernel_after_chain"])
def test_structure_variants_are_bitwise(default_run, env):
    got = _probe(**env)
    assert got.keys() == default_run.keys()
    for case, ref in default_run.items():
        assert got[case]["status"] == ref["status"], case
        assert got[case]["iterations"] == ref["iterations"], case
        assert got[case]["x_sha"] == ref["x_sha"], case  # every bit of the iterate
        assert got[case]["trace_sha"] == ref["trace_sha"], case


def test_small_dense_kernel_against_tile_kernel(default_run):
    got = _probe(TS_DENSE_SMALL="tile")
    for case, ref in default_run.items():
        if not case.startswith("dense"):
            continue
        assert got[case]["status"] == ref["status"] and got[case]["iterations"] == ref["iterations"], case
        a, b = np.array(got[case]["x_head"]), np.array(ref["x_head"])
        assert np.linalg.norm(a - b) <= 1e-9 * max(np.linalg.norm(b), 1e-300), case


@pytest.mark.parametrize("m,n", [(3, 130), (129, 128), (1000, 1000), (257, 4095), (5000, 200), (37, 1001)])
def test_small_dense_kernel_odd_shapes(m, n):
    import paper_2304_12168_b200 as ts

    rng = np.random.default_rng(m * 7919 + n)
    a = rng.standard_normal((m, n))
    dm = ts.DeviceMatrix(a)
    v, w = rng.standard_normal(n), rng.standard_normal(m)
    y, z = ts.matvec(dm, v), ts.matvec_transpose(dm, w)
    assert np.max(np.abs(y - a @ v)) <= 1e-13 * np.abs(a).max() * np.abs(v).sum()
    assert np.max(np.abs(z - a.T @ w)) <= 1e-13 * np.abs(a).max() * np.abs(w).sum()
    assert np.array_equal(y, ts.matvec(dm, v))  # identical bits run to run


@pytest.mark.parametrize("m,n", [(4100, 8200), (2048, 20011)])
def test_large_dense_av_on_column_tiles(m, n):
    """HBM-sized dense matrices (>= 256 MB) keep a transposed copy and run A v on
    the column-tile kernel (PLAN_NCOLS): plan selected, both products within
    1e-14 of |A||v|, identical bits run to run, and a recycled handle of the
    same shape refreshes the copy."""
    import paper_2304_12168_b200 as ts

    rng = np.random.default_rng(m + n)
    a = rng.standard_normal((m, n))
    dm = ts.DeviceMatrix(a)
    assert dm.plans() == ("column_tiles_transposed_copy", "dense_tiles")
    v, w = rng.standard_normal(n), rng.standard_normal(m)
    y, z = ts.matvec(dm, v), ts.matvec_transpose(dm, w)
    assert np.max(np.abs(y - a @ v)) <= 1e-14 * np.abs(a).max() * np.abs(v).sum()
    assert np.max(np.abs(z - a.T @ w)) <= 1e-14 * np.abs(a).max() * np.abs(w).sum()
    assert np.array_equal(y, ts.matvec(dm, v))
    del dm  # retire the handle: the next matrix of this shape recycles its storage
    a2 = rng.standard_normal((m, n))
    dm2 = ts.DeviceMatrix(a2)
    y2 = ts.matvec(dm2, v)
    assert np.max(np.abs(y2 - a2 @ v)) <= 1e-14 * np.abs(a2).max() * np.abs(v).sum()
