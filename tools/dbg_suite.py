import sys, os
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import test_gpu_suite as T
mods = T._ours()
for spec in sys.argv[1:]:
    test, k = spec.rsplit("#", 1)
    rec = [r for r in T.RECORDS if r["test"].endswith(test)][int(k)]
    args = T.revive(rec["args"], mods); kwargs = T.revive(rec["kwargs"], mods)
    fn = getattr(mods[rec["fn"].rsplit(".", 1)[0]], rec["fn"].rsplit(".", 1)[1])
    got = fn(*args, **kwargs)
    w = rec["result"][1]
    a0 = rec["args"][0]
    print(spec, rec["fn"], "shape", getattr(a0, "shape", None), "kwargs", rec["kwargs"], "band", rec["band"])
    print("  ours:", got.status, got.iterations, got.residual_norm, got.normal_residual_norm, got.detail, "x", np.asarray(got.x)[:6])
    print("  ref :", w["status"], w["iterations"], w["residual_norm"], w["normal_residual_norm"], w["detail"], "x", np.asarray(w["x"])[:6])
    tr = w["trace"][2]
    print("  ref trace tail:", tr[-3:])
    print("  our trace tail:", got.trace.rows[-3:])
    # first divergence of the trace rows
    ref_rows = w["trace"][2]
    for i, (ra, rb) in enumerate(zip(got.trace.rows, ref_rows)):
        va = np.array([v for v in ra[:-1] if not isinstance(v, str)], dtype=float)
        vb = np.array([v for v in rb[:-1] if not isinstance(v, str)], dtype=float)
        ea = [v for v in ra if isinstance(v, str)]; eb = [v for v in rb if isinstance(v, str)]
        if ea != eb or np.max(np.abs(va - vb) / np.maximum(np.abs(vb), 1e-300)) > 1e-6:
            print("  first divergence at row", i, "\n   ours", ra, "\n   ref ", rb)
            print("   prev ours", got.trace.rows[i-1] if i else None, "\n   prev ref ", ref_rows[i-1] if i else None)
            break
