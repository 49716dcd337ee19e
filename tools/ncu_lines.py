"""Attribute an ncu SASS-level profile to source lines.

usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL MANGLED_NAME [SO]
  KERNEL: ncu kernel base name (e.g. k_step); the block whose demangled name
  contains $PICK (e.g. "(int)1") is used (default: the first block).

Joins the per-instruction "Instructions Executed" / stall samples of the
report's source page (SASS view) with nvdisasm's line table of the same
library (built with -lineinfo), and prints the top source lines.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, kre, mangled = sys.argv[1], sys.argv[2], sys.argv[3]
so = sys.argv[4] if len(sys.argv) > 4 else "paper_2605_26659_b200/libfinom_b200.so"

out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass",
                      "-k", kre], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
pick = os.environ.get("PICK", "")
start = next(i for i, r in enumerate(rows) if r and r[0] == "Kernel Name" and pick in r[1])
rows = rows[start:]
hdr = rows[1]
ia, ie, isamp = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index(
    "Warp Stall Sampling (All Samples)")
recs = []
for r in rows[2:]:
    if len(r) < len(hdr) or not r[ia].startswith("0x"):
        if recs:
            break  # first kernel only
        continue
    recs.append((int(r[ia], 16), float(r[ie] or 0), float(r[isamp] or 0), r[1].strip()))
base = recs[0][0]

tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(tmp, cub)],
                     capture_output=True, text=True).stdout
sec = dis.split(".text." + mangled + ":")[1]
sec = sec.split("\n.text.")[0] if "\n.text." in sec else sec
line_of = {}
cur = None
for ln in sec.splitlines():
    m = re.search(r'File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,6})\*/", ln)
    if m:
        line_of[int(m.group(1), 16)] = cur

agg = collections.defaultdict(lambda: [0.0, 0.0])
tot_i = tot_s = 0.0
for addr, n, smp, _ in recs:
    key = line_of.get(addr - base)
    agg[key][0] += n
    agg[key][1] += smp
    tot_i += n
    tot_s += smp
srcs = {}
for f, l in [k for k in agg if k]:
    for path in ["paper_2605_26659_b200/csrc/" + f]:
        if os.path.exists(path) and f not in srcs:
            srcs[f] = open(path).read().splitlines()
print("total warp-instr %.4g  samples %.4g" % (tot_i, tot_s))
for key, (n, smp) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(os.environ.get("TOP", "40"))]:
    txt = srcs.get(key[0], [""] * 99999)[key[1] - 1].strip()[:70] if key else "?"
    print("%5.1f%% instr %5.1f%% stall  %s:%s  %s" % (100 * n / tot_i, 100 * smp / tot_s,
                                                   key[0] if key else "?", key[1] if key else "",
                                                   txt))
