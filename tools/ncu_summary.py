"""Summarise ncu artefacts (launch list CSV + `--set full` report) into a
markdown table for profiles/.  Runs here (no GPU): ncu -i reads the report.

    python tools/ncu_summary.py gpurun_out/launches.csv gpurun_out/full.ncu-rep [traffic.json] > profiles/rN_summary.md

traffic.json (optional): per kernel, dram__bytes_read.sum + dram__bytes_write.sum
of its launch in the `--set full` capture (bench.py's roofline "traffic").
"""
import json
import collections
import csv
import io
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__inst_executed.avg.per_cycle_active": "ipc",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "regs",
    "smsp__inst_executed.sum": "inst",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
}


def short(name):
    name = name.split("(")[0].replace("void ", "").replace("gut::", "")
    return name


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    tot = collections.OrderedDict()
    cnt = collections.Counter()
    for r in rows[hdr + 1:]:
        k = short(r[ki])
        v = float(r[vi].replace(",", ""))
        tot[k] = tot.get(k, 0.0) + v
        cnt[k] += 1
    return tot, cnt


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    scale = {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[h.index("Kernel Name")])}
        for m, k in METRICS.items():
            if m in h:
                i = h.index(m)
                try:
                    d[k] = float(r[i].replace(",", "")) * scale.get(units[i], 1.0)
                except ValueError:
                    d[k] = None
        res.append(d)
    return res


def main():
    lc, fr = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None
    tj = sys.argv[3] if len(sys.argv) > 3 else None
    tot, cnt = launches(lc)
    total = sum(tot.values())
    print("## Launch list (ncu `gpu__time_duration.sum`, cold-cache, serialised)\n")
    print("| kernel | launches | total us | share |")
    print("|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"| {k} | {cnt[k]} | {v / 1e3:.1f} | {v / total:.1%} |")
    if fr:
        print("\n## `ncu --set full` per launch\n")
        cols = ["duration_us", "dram_read", "dram_write", "dram_pct", "sm_pct", "issue_pct", "fma_pipe_pct",
                "xu_pipe_pct", "ipc", "occupancy_pct", "regs", "inst"]
        print("| kernel | " + " | ".join(cols) + " |")
        print("|---|" + "---|" * len(cols))
        for d in full(fr):
            vals = []
            for c in cols:
                v = d.get(c)
                if v is None:
                    vals.append("-")
                elif c == "duration_us":
                    vals.append(f"{v / 1e3:.1f}")
                elif c in ("dram_read", "dram_write"):
                    vals.append(f"{v / 1e6:.1f} MB")
                elif c == "inst":
                    vals.append(f"{v / 1e6:.1f}M")
                else:
                    vals.append(f"{v:.1f}")
            print(f"| {d['kernel']} | " + " | ".join(vals) + " |")
        if tj:
            traffic, extra = {}, {}
            for d in full(fr):
                if d.get("dram_read") is not None and d.get("dram_write") is not None:
                    traffic.setdefault(d["kernel"], d["dram_read"] + d["dram_write"])
                    extra.setdefault(d["kernel"], {k: d.get(k) for k in ("issue_pct", "dram_pct", "duration_us",
                                                                         "inst", "fma_pipe_pct", "xu_pipe_pct")})
            json.dump({"source": f"ncu --set full ({fr})", "bytes_per_launch": traffic, "metrics": extra},
                      open(tj, "w"), indent=1)


if __name__ == "__main__":
    main()
