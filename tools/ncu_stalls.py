"""Warp-stall breakdown (pc-sampling counts, %) of every kernel in an ncu report.
usage: ncu_stalls.py <report.ncu-rep> [kernel substring]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
sub = sys.argv[2] if len(sys.argv) > 2 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
for v in rows[2:]:
    d = dict(zip(h, v))
    if sub not in d.get("Kernel Name", ""):
        continue
    st = {}
    for k, x in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
            try:
                st[k[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(x.replace(",", ""))
            except ValueError:
                pass
    tot = sum(st.values()) or 1
    print(d.get("Kernel Name", "")[:60], d.get("gpu__time_duration.sum"),
          "issue%", d.get("smsp__issue_active.avg.pct_of_peak_sustained_active"))
    print("   " + "  ".join(f"{k} {100 * x / tot:.1f}" for k, x in sorted(st.items(), key=lambda t: -t[1])[:9]))
