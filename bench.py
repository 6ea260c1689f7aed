"""Benchmark contract for the TA / CTA iteration path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c1|c3|c4|c5]

Workload (default, BASELINE.json configs[1]): C2, dense rank-deficient
5000 x 20000 fp64, A = U V^T (rank 2000), b = A x* + 1e-3 noise.  One STEP is
one complete ``centering_solve(A, b, CenteringOptions(epsilon=1e-8))`` to the
reference's own stopping rule (normal-equation clause, ~23 iterations), so
``value`` = CTA iterations / s over K steps and ``time_to_tolerance_ms`` is
the per-step solve time.

* value: A resident in HBM (DeviceMatrix built before the timed region), b on
  the device; CUDA events on the launching (default) stream around K steps,
  barrier + synchronize on both sides, max over ranks.  A is 800 MB > L2, so
  no L2 flush is needed between steps.
* e2e: the same metric through the public API from pinned HOST buffers:
  every step uploads A and b (H2D) and reads x and the trace back (D2H).
* roofline: the dominant kernel (dense A v / A^T v pass) timed live inside
  the timed solves by the library's per-class kernel timers (%globaltimer,
  earliest block start to the finishing block), algorithmic bytes
  8mn + 8(m+n) per launch, peak = MEASURED_PEAKS.json hbm_gbs.
* cpu_baseline / --impl reference: the REAL reference package (``trisolve``,
  installed into baseline/_ref by ``pip install --target``; kind
  "reference") through its public API on the host cores, rank 0 only,
  bounded sample; the oracle port (same numpy/OpenBLAS/scipy calls) only
  when baseline/_ref is absent (kind "port").  Both arms print the same
  ``config`` dict.

N > 1 (torchrun): ONE sharded solve over all ranks (strong scaling): column
blocks (rank p holds A[:, p n/N : (p+1) n/N]; every A v is a fused
fixed-rank-order all-reduce over NVLink peer memory), or for C4 row blocks
(a halo exchange with each neighbour before every pass, scalar all-reduces);
value = the solve's iterations / max time.  Communicators are per process
and each rank's block is sliced once, outside every timed region.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TA/CTA iterations/s & time to rel. residual 1e-8; matvec-pair HBM GB/s"
CONFIGS = {
    "c1": dict(gen="c1", solver="cta", eps=1e-8, max_iters=10000, cpu_max_iters=2000,
               desc="C1 dense gaussian 1000x1000, CTA eps=1e-8, cap 10000"),
    "c2": dict(gen="c2", solver="cta", eps=1e-8, max_iters=100000, cpu_max_iters=100000,
               desc="C2 dense rank-2000 5000x20000 (variance reading), CTA eps=1e-8"),
    "c3": dict(gen="c3", solver="cta", eps=1e-8, max_iters=2000, cpu_max_iters=2000,
               desc="C3 Clement variant n=100001 CSR, CTA eps=1e-8, fixed budget 2000 iterations"),
    "c4": dict(gen="c4", solver="cta", eps=1e-8, max_iters=600, cpu_max_iters=100,
               desc="C4 upwind conv-diff n=1e6 CSR, CTA eps=1e-8, fixed budget 600 iterations"),
    "c5": dict(gen="c5", solver="lp", eps=1e-6, max_iters=100000, cpu_max_iters=100000,
               desc="C5 LP 1e4 x 1e6 CSR+CSC, TA non-negativity eps=1e-6*||b|| (stalls @11)"),
    "c5ta": dict(gen="c5", solver="ta", eps=1e-6, max_iters=100000, cpu_max_iters=100000,
                 desc="C5 LP matrix, unconstrained TA (solve_adaptive) eps=1e-6*||b||"),
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_reference():
    """The reference package from baseline/_ref (None when not installed)."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "trisolve")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        import trisolve

        return trisolve
    except Exception:
        return None


def host_info():
    model = ""
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"os_cpu_count": os.cpu_count(), "cpu_model": model, "blas_threads": blas_threads()}


def config_dict(cfg):
    """The workload description both arms print (identical dicts)."""
    return {"workload": cfg["desc"], "step": "one full solve, reference stopping rule",
            "l2": "no flush: matrix larger than L2" if cfg["gen"] in ("c2", "c4", "c5")
                  else "no flush: L2-resident matrix (latency-bound config)"}


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        for info in threadpool_info():
            if info.get("user_api") == "blas":
                return int(info.get("num_threads", os.cpu_count() or 1))
    except Exception:
        pass
    return os.cpu_count() or 1


def make_workload(cfg):
    from paper_2304_12168_b200 import workloads as W

    return W.make(cfg["gen"])


def pass_bytes(a, trans: bool):
    """Algorithmic bytes of one matvec pass."""
    import scipy.sparse as sp

    m, n = a.shape
    if sp.issparse(a):
        nnz = a.nnz
        if trans:
            return 12 * nnz + 4 * (n + 1) + 8 * m + 8 * n
        return 12 * nnz + 4 * (m + 1) + 8 * n + 8 * m
    return 8 * m * n + 8 * (m + n)


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t0 = time.time()  # the sampler is live before the timed region starts
            while not self.lines and time.time() - t0 < 5.0:
                time.sleep(0.01)
            self.lines.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        loaded = [v for v in sm if v > 0.5 * max(sm)] or sm
        return {"sm_mhz": float(np.median(loaded)), "sm_max_mhz": float(max(smax)),
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------- reference ---
def run_cpu_step(cfg, w, bounded=False):
    """One solve on the host: the real reference package when installed,
    else the oracle port.  Returns (result dict, kind)."""
    bn = float(np.linalg.norm(w.b))
    cap = cfg["cpu_max_iters"] if bounded else cfg["max_iters"]
    ref = load_reference()
    if ref is not None:
        if cfg["solver"] == "cta":
            r = ref.centering_solve(w.a, w.b, ref.CenteringOptions(epsilon=cfg["eps"], max_iters=cap))
        elif cfg["solver"] == "ta":
            r = ref.solve_adaptive(w.a, w.b, eps=cfg["eps"] * bn, max_iters=cap)
        else:
            r = ref.nonnegative_feasibility(w.a, w.b, eps=cfg["eps"] * bn, max_iters=cap)
        return {"status": r.status, "iterations": r.iterations}, "reference"
    from oracle import port

    if cfg["solver"] == "cta":
        out = port.cta_solve(w.a, w.b, epsilon=cfg["eps"], max_iters=cap)
    elif cfg["solver"] == "ta":
        out = port.ta_adaptive(w.a, w.b, eps=cfg["eps"] * bn, max_iters=cap)
    else:
        out = port.lp_feasibility(w.a, w.b, eps=cfg["eps"] * bn, max_iters=cap)
    return out, "port"


def cpu_sample_text(cfg, out, kind, cores, steps):
    what = ("the reference package (baseline/_ref trisolve, public API)" if kind == "reference"
            else "oracle/port.py (the reference's numpy/OpenBLAS/scipy calls)")
    sparse_note = "; scipy sparse kernels are single-threaded" if cfg["gen"] in ("c3", "c4", "c5") else ""
    return (f"{steps} solve(s) of the workload capped at {cfg['cpu_max_iters']} iterations "
            f"(last: {out['iterations']} iterations, {out['status']}) with {what}, "
            f"OpenBLAS {cores} threads{sparse_note}")


def reference_arm(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    w = make_workload(cfg)
    for _ in range(args.warmup):
        run_cpu_step(cfg, w, bounded=True)
    iters = 0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        out, kind = run_cpu_step(cfg, w, bounded=True)
        iters += out["iterations"]
    dt = time.perf_counter() - t0
    val = iters / dt
    cores = blas_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "iterations/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded numpy, BASELINE.json formula; SURVEY.md Appendix A)",
        "config": config_dict(cfg),
        "solve": {"status": out["status"], "iterations_per_step": out["iterations"]},
        "cpu_baseline": {"value": val, "unit": "iterations/s", "cores": cores, "kind": kind,
                         "sample": cpu_sample_text(cfg, out, kind, cores, args.steps),
                         "host": host_info()},
        "e2e": {"value": val, "unit": "iterations/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------- ours ---
def make_operand(ts, w, part, dev, a_local=None, stream=None):
    """The solve operand: a DeviceMatrix (N = 1) or this rank's shard built from
    its pre-sliced block (`a_local` overrides the block with a pinned copy)."""
    if part is None:
        return ts.DeviceMatrix(w.a if a_local is None else a_local, device=dev, stream=stream)
    from paper_2304_12168_b200 import shard as S

    kind, blk = part
    if kind == "rows":
        rows, cols, hw = blk if a_local is None else a_local
        return S.RowShardedMatrix(w.a, device=dev, blocks=(rows, cols, hw))
    return S.ShardedMatrix(blk if a_local is None else a_local, device=dev, local=True,
                           n_global=w.a.shape[1])


def solve_once(ts, cfg, dm, b, bn):
    if cfg["solver"] == "cta":
        return ts.centering_solve(dm, b, ts.CenteringOptions(epsilon=cfg["eps"],
                                                             max_iters=cfg["max_iters"]))
    if cfg["solver"] == "ta":
        return ts.solve_adaptive(dm, b, eps=cfg["eps"] * bn, max_iters=cfg["max_iters"])
    return ts.nonnegative_feasibility(dm, b, eps=cfg["eps"] * bn, max_iters=cfg["max_iters"])


def ours_arm(args, cfg):
    import torch

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    import paper_2304_12168_b200 as ts

    w = make_workload(cfg)
    bn = float(np.linalg.norm(w.b))
    part = None
    if world > 1:
        # this rank's block, sliced once (the timed loops only upload it)
        from paper_2304_12168_b200 import shard as S

        if cfg["gen"] == "c4":
            # row-block sharded solve (square banded C4): each rank owns rows and
            # columns [r0, r1); a halo exchange with each neighbour before every pass
            rr = S.column_range(w.a.shape[0], world, rank)
            part = ("rows", S.row_blocks(w.a, *rr))
        else:
            # column-sharded solve: each rank holds A[:, c0:c1]; A v is one fused
            # fixed-rank-order all-reduce over NVLink peer memory per pass
            cr = S.column_range(w.a.shape[1], world, rank)
            part = ("columns", S.local_block(w.a, *cr))
    dm = make_operand(ts, w, part, dev)
    b_dev = torch.from_numpy(w.b).to(f"cuda:{dev}")

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    for _ in range(max(3, args.warmup)):
        solve_once(ts, cfg, dm, b_dev, bn)

    barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    results = []
    with ClockSampler(dev) as clk:
        ev0.record()
        for _ in range(args.steps):
            r = solve_once(ts, cfg, dm, b_dev, bn)
            r.x = None  # consumed: its pinned block returns to the pool
            results.append(r)
        ev1.record()
        torch.cuda.synchronize()
    barrier()
    ms = float(ev0.elapsed_time(ev1))
    iters = sum(r.iterations for r in results)
    if world > 1:
        t = torch.tensor([ms], device=f"cuda:{dev}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    # one sharded solve is the whole job: its iterations are the job's iterations
    value = iters / (ms / 1e3)

    # live kernel accounting over the timed solves
    kms = np.zeros(4)
    kcnt = np.zeros(4, dtype=np.int64)
    launches = 0
    for r in results:
        kms += np.array(r.kernel_ms)
        kcnt += np.array(r.kernel_count, dtype=np.int64)
        launches += r.kernel_launches
    peak, peak_src = measured_peak()
    classes = {0: ("A v", False), 1: ("A^T v", True)}
    breakdown = {}
    for k, (nm, trans) in classes.items():
        if kcnt[k]:
            avg_ms = kms[k] / kcnt[k]
            byt = pass_bytes(w.a, trans)
            breakdown[nm] = {"launches": int(kcnt[k]), "avg_us": avg_ms * 1e3,
                             "bytes_per_launch": int(byt),
                             "gbs": byt / (avg_ms * 1e-3) / 1e9,
                             "share_of_step": float(kms[k] / ms)}
    breakdown["vector passes"] = {"launches": int(kcnt[2]), "ms_total": float(kms[2]),
                                  "share_of_step": float(kms[2] / ms)}
    breakdown["hankel solves (in-finisher)"] = {"launches": int(kcnt[3]), "ms_total": float(kms[3]),
                                   "share_of_step": float(kms[3] / ms)}
    breakdown["note"] = ("per class: matrix products timed on the device (kernel entry or state-word read to the "
                         "finisher); 'launches' counts products — the one-kernel moment pairs / chains of the "
                         "latency-bound configs perform 2 / 2t products per launch and are booked under 'A v'")
    dom = max((k for k in classes if kcnt[k]), key=lambda k: kms[k])
    dom_name = classes[dom][0]
    achieved = breakdown[dom_name]["gbs"]
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(f"{args.config}:{dom_name}")
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "kernel": dom_name,
                "peak_source": peak_src,
                "pair_gbs": (sum(breakdown[c[0]]["bytes_per_launch"] * breakdown[c[0]]["launches"]
                                 for c in classes.values() if c[0] in breakdown)
                             / (sum(kms[k] for k in classes) * 1e-3) / 1e9)}

    line = {
        "metric": METRIC, "value": value, "unit": "iterations/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded numpy, BASELINE.json formula; SURVEY.md Appendix A)",
        "config": config_dict(cfg),
        "solve": {"status": results[-1].status, "iterations_per_step": results[-1].iterations,
                  "time_to_tolerance_ms": float(np.median([r.device_ms for r in results])),
                  "final_rel_residual": results[-1].residual_norm / bn},
        "parallelism": "single GPU" if world == 1 else
        (f"row-block sharded x{world} (halo exchange + scalar all-reduce over NVLink)"
         if cfg["gen"] == "c4" else
         f"column-sharded x{world} (fused fixed-order all-reduce over NVLink)"),
        "roofline": roofline,
        "kernel_breakdown": breakdown,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }

    if not args.no_e2e:
        line["e2e"] = e2e_measure(ts, cfg, w, bn, args, dev, world, part)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, w)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def e2e_measure(ts, cfg, w, bn, args, dev, world, part=None):
    """Same metric through the public API with pinned HOST buffers: every
    step uploads A and b and reads x (+ trace) back."""
    import scipy.sparse as sp
    import torch

    def pinned_copy(arr):
        t = torch.empty(arr.shape, dtype=torch.float64 if arr.dtype == np.float64 else torch.int32,
                        pin_memory=True)
        out = t.numpy()
        out[...] = arr
        return out, t

    def pinned_csr(csr):
        data, t1 = pinned_copy(csr.data)
        ind, t2 = pinned_copy(csr.indices.astype(np.int32))
        ptr, t3 = pinned_copy(csr.indptr.astype(np.int32))
        keep.extend([t1, t2, t3])
        out = sp.csr_array((data, ind, ptr), shape=csr.shape)
        out.indices = ind
        out.indptr = ptr
        return out, data.nbytes + ind.nbytes + ptr.nbytes

    def pinned_any(a):
        if sp.issparse(a):
            return pinned_csr(a)
        arr, t = pinned_copy(np.ascontiguousarray(a))
        keep.append(t)
        return arr, arr.nbytes

    keep = []
    if part is None:
        a_host, h2d = pinned_any(w.a)
    elif part[0] == "rows":  # this rank's rows and columns (as rows of A^T), with the halo width
        rows, cols, hw = part[1]
        (r_h, nb1), (c_h, nb2) = pinned_csr(rows), pinned_csr(cols)
        a_host, h2d = (r_h, c_h, hw), nb1 + nb2
    else:
        a_host, h2d = pinned_any(part[1])
    b_host, t4 = pinned_copy(w.b)
    keep.append(t4)
    h2d += b_host.nbytes  # per rank; the line reports the job total below
    steps = max(1, min(args.steps, 10))
    if world > 1:
        hb = torch.tensor([h2d], dtype=torch.float64, device=f"cuda:{dev}")
        torch.distributed.all_reduce(hb)
        h2d = int(hb.item())

    copy_stream = torch.cuda.Stream(device=dev)  # non-blocking: uploads overlap solves

    def upload():
        return make_operand(ts, w, part, dev, a_local=a_host,
                            stream=copy_stream if world == 1 else None)

    def run(n_steps, pipelined):
        """n_steps x (upload A and b, solve, read x and the trace back); with
        `pipelined`, step k+1's upload runs on a worker thread / copy stream
        while step k solves (double buffering through the public API)."""
        from concurrent.futures import ThreadPoolExecutor

        iters = rows = 0
        with ThreadPoolExecutor(max_workers=1) as pool:
            nxt = pool.submit(upload) if pipelined else None
            for k in range(n_steps):
                dm = nxt.result() if pipelined else upload()
                if pipelined and k + 1 < n_steps:
                    nxt = pool.submit(upload)
                r = solve_once(ts, cfg, dm, b_host, bn)
                del dm
                iters += r.iterations
                rows += len(r.trace)
        return iters, rows

    pipelined = world == 1
    run(2, pipelined)
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    iters, rows = run(steps, pipelined)
    ev1.record()
    torch.cuda.synchronize()
    ms = float(ev0.elapsed_time(ev1))
    # the same steps without the overlap, for reference
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    s_iters, _ = run(steps, False)
    e1.record()
    torch.cuda.synchronize()
    serial_ms = float(e0.elapsed_time(e1))
    n = w.a.shape[1]
    if world > 1:
        t = torch.tensor([ms], device=f"cuda:{dev}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    return {"value": iters / (ms / 1e3), "unit": "iterations/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(8 * n + 48 * rows // steps),
            "steps": steps, "ms_per_step": ms / steps,
            "serial": {"value": s_iters / (serial_ms / 1e3), "ms_per_step": serial_ms / steps},
            "note": "every step uploads A (DeviceMatrix from pinned host memory) and b and reads x "
                    "and the trace back; " + ("the next step's upload overlaps the current solve "
                    "(worker thread + non-blocking copy stream, double-buffered); 'serial' is "
                    "the same loop without the overlap" if pipelined else "no overlap")}


def cpu_baseline(cfg, w):
    run_cpu_step(cfg, w, bounded=True)  # warm-up (imports, page-in)
    t0 = time.perf_counter()
    out, kind = run_cpu_step(cfg, w, bounded=True)
    dt = time.perf_counter() - t0
    cores = blas_threads()
    return {"value": out["iterations"] / dt, "unit": "iterations/s", "cores": cores,
            "kind": kind, "sample": cpu_sample_text(cfg, out, kind, cores, 1),
            "host": host_info()}


def main():
    args = parse()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return reference_arm(args, cfg)
    return ours_arm(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
