"""Opcode summary of the hot kernels' SASS (cuobjdump -sass of the built
library): per kernel, the count of each opcode family that evidences the
design (bulk/TMA copies UBLKCP, mbarrier SYNCS, LDGSTS cp.async, fp64 DFMA /
DMUL / DADD, shuffles, shared / global memory ops).
usage: python tools/sass_summary.py [lib.so] > profiles/r02_sass_summary.txt"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2605_26659_b200/libfinom_b200.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
HOT = ["k_solve_group", "k_step", "k_resolve", "k_absorb", "k_sq_apply", "k_sq_pre", "k_sq_scan",
       "k_sq_build", "k_pre", "k_apply", "k_epi_fold"]
FAM = ["UBLKCP", "UBLKPF", "SYNCS", "LDGSTS", "DFMA", "DMUL", "DADD", "MUFU", "SHFL", "REDUX",
       "LDS", "STS", "LDG", "STG", "BAR", "ATOM", "RED", "CCTL", "FENCE", "MEMBAR"]
cur, counts = None, {}
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        counts[cur] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if m and cur:
        counts[cur][m.group(1)] += 1
print("%-44s %6s  %s" % ("kernel", "instr", "  ".join("%s" % f for f in FAM)))
for name, c in counts.items():
    short = re.sub(r"_ZN2fb\d+", "", name)
    if not any(h in short for h in HOT):
        continue
    tot = sum(c.values())
    fam = {f: sum(v for k, v in c.items() if k == f or (k.startswith(f) and f not in ("RED", "LDS", "STS", "LDG", "STG", "BAR")))
           for f in FAM}
    print("%-44s %6d  %s" % (short[:44], tot, "  ".join("%s=%d" % (f, fam[f]) for f in FAM if fam[f])))
