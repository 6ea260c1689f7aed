"""Summarise ncu artefacts for profiles/: launch-list shares and --set full metrics."""
import collections, csv, io, json, re, subprocess, sys

def launch_shares(path):
    text = open(path).read()
    lines = text.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui].strip().lower()
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
                 "s": 1e6, "second": 1e6}.get(unit, 1.0)
        v = v * scale
        name = re.sub(r"\(.*", "", r[ki])
        agg[name].append(v)
    tot = sum(sum(v) for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append({"kernel": k, "launches": len(v), "total_us": round(sum(v), 2),
                    "avg_us": round(sum(v) / len(v), 2), "share": round(sum(v) / tot, 4)})
    return out

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "launch__occupancy_limit_registers",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
           "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_wait",
           "smsp__pcsamp_warps_issue_stalled_selected"]

def full_metrics(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": re.sub(r"\(.*", "", r[h.index("Kernel Name")])}
        for m in METRICS:
            if m in h:
                d[m] = f"{r[h.index(m)]} {units[h.index(m)]}".strip()
        out.append(d)
    return out

def traffic(rep):
    """dram read + write bytes per launch, keyed by kernel name."""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    mult = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}
    out = {}
    for r in rows[2:]:
        name = re.sub(r"\(.*", "", r[h.index("Kernel Name")])
        tot = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = h.index(m)
            tot += float(r[i].replace(",", "")) * mult[units[i].strip().lower()]
        out.setdefault(name, []).append(tot)
    return {k: sum(v) / len(v) for k, v in out.items()}


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    res = {"launches": launch_shares, "full": full_metrics, "traffic": traffic}[kind](path)
    print(json.dumps(res, indent=1))
