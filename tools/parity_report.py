"""Where the device lands on every golden case: status / iterations against
the recorded reference run, rel l2 of x against the reference's own
self-noise (tests/golden/self_noise.json) and, for the chaotic cases, against
the perturbation band (tests/golden/chaotic_bands.json).  JSON lines."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

from conftest import Golden, golden_names, rel_l2
from test_gpu_parity import run_device

noise = json.load(open(os.path.join(ROOT, "tests", "golden", "self_noise.json")))["cases"]
bands = json.load(open(os.path.join(ROOT, "tests", "golden", "chaotic_bands.json")))
for name in golden_names():
    g = Golden(name)
    r = run_device(g)
    out = {"case": name, "status": r.status, "ref_status": g.status, "iterations": r.iterations,
           "ref_iterations": g.iterations, "x_rel_l2": rel_l2(r.x, g.x),
           "residual": r.residual_norm, "ref_residual": g.residual_norm}
    if name in noise:
        out["ref_x_noise"] = noise[name]["x_noise"]
    if name in bands:
        out["band"] = {k: bands[name][k] for k in ("iterations_lo", "iterations_hi", "residual_lo",
                                                    "residual_hi", "statuses") if k in bands[name]}
    print(json.dumps(out), flush=True)
