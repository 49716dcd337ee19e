"""Per-source-line instructions / stall samples of one kernel of an ncu report
captured with --import-source on (cuda,sass view).
usage: python tools/ncu_src.py REPORT KERNEL_SUBSTRING [NORM] [TOP] [LO-HI ...]
NORM divides instruction counts (e.g. tiles per launch); LO-HI groups
finom_1d.cu line ranges."""
import collections
import csv
import io
import subprocess
import sys

rep, kname = sys.argv[1], sys.argv[2]
norm = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
inst, samp, src = collections.Counter(), collections.Counter(), {}
path = kern = hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        kern = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if kern and kname in kern and hdr and r[0] and len(r) == len(hdr):
        try:
            ie, st = int(r[7]), int(r[4])
        except ValueError:
            continue
        key = (path, int(r[0]))
        inst[key] += ie
        samp[key] += st
        src[key] = r[1][:80]
ti, ts = sum(inst.values()), max(1, sum(samp.values()))
print("total inst %.4g (%.1f per norm)  stall samples %d" % (ti, ti / norm, ts))
for key, v in inst.most_common(top):
    print("%8.1f %5.1f%% %s:%d %s" % (v / norm, 100 * samp[key] / ts, key[0], key[1], src[key]))
