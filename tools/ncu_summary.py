"""Summarise an `ncu --set full` report of the half-step kernels into
profiles/ncu_summary.json (read by bench.py for roofline.traffic) and print a
short text summary.

usage: python tools/ncu_summary.py REPORT.ncu-rep OUT.json
"""
import csv
import io
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
keys = {
    "duration_us": ("gpu__time_duration.sum", 1e-3),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "inst_executed": ("smsp__inst_executed.sum", 1.0),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "issue_active_pct": ("sm__inst_issued.avg.pct_of_peak_sustained_active", 1.0),
    "registers": ("launch__registers_per_thread", 1.0),
}
units = dict(zip(hdr, rows[1]))
scale_b = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
res = {}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("fb::", "")
    e = {}
    for k, (m, sc) in keys.items():
        v = d.get(m)
        if v in (None, ""):
            continue
        v = float(v.replace(",", ""))
        if sc is None:
            v *= scale_b.get(units.get(m, "byte"), 1)
        elif m == "gpu__time_duration.sum":
            u = units.get(m, "nsecond")
            v = v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1.0)
        else:
            v *= sc
        e[k] = v
    st = [(k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
           float(v)) for k, v in d.items()
          if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
          and v not in ("", None)]
    st.sort(key=lambda kv: -kv[1])
    e["top_stalls_per_issue"] = dict(st[:6])
    e["dram_bytes_per_launch"] = e.get("dram_read_bytes", 0) + e.get("dram_write_bytes", 0)
    res.setdefault(name, []).append(e)
summary = {"report": rep, "kernels": res}
# the bench's roofline.traffic: DRAM bytes of one iteration's two half steps
tot = 0.0
for k in ("k_step<0>", "k_step<1>"):
    if k in res:
        tot += res[k][0]["dram_bytes_per_launch"]
summary["k_step"] = {"dram_bytes_per_launch": tot or None,
                     "note": "k_step<0> + k_step<1> DRAM bytes (one iteration), ncu --set full"}
with open(out, "w") as f:
    json.dump(summary, f, indent=1)
for k, v in res.items():
    e = v[0]
    print("%-14s %8.1f us  dram %.1f MB  inst %.3g  stalls %s" % (
        k, e.get("duration_us", 0), e["dram_bytes_per_launch"] / 1e6, e.get("inst_executed", 0),
        ", ".join("%s %.2f" % kv for kv in list(e["top_stalls_per_issue"].items())[:4])))
