"""Group tools/ncu_lines.py output of k_step into phases (by source line ranges)."""
import re, subprocess, sys
rep, pick = sys.argv[1], sys.argv[2]
mangled = "_ZN2fb6k_stepILi%sEEEvNS_3DevE" % pick
out = subprocess.run("TOP=100000 PICK='(int)%s' python tools/ncu_lines.py %s k_step %s" % (pick, rep, mangled),
                     shell=True, capture_output=True, text=True).stdout
src = open("paper_2605_26659_b200/csrc/finom_1d.cu").read().splitlines()
start = next(i for i, l in enumerate(src) if "void tile_compute(" in l) + 1
marks = [(i + 1, l.strip()) for i, l in enumerate(src[start:start + 600], start) if l.strip().startswith("// ----")]
def grp(f, l):
    if f == "finom_1d.cu":
        name = "k_step prologue"
        for ln, txt in marks:
            if l >= ln:
                name = txt[:40]
        return name
    return f
g = {}
print(out.splitlines()[0])
for ln in out.splitlines()[1:]:
    m = re.match(r'\s*([\d.]+)% instr\s+([\d.]+)% stall\s+(\S+?):(\d*)\s*(.*)', ln)
    if not m: continue
    key = grp(m.group(3), int(m.group(4) or 0))
    if m.group(3) == "tile_core.cuh":
        key = "tile_core:" + ("scan/tf" if int(m.group(4)) < 113 else "reduce" if int(m.group(4)) < 130 else "tree/other")
    a = g.setdefault(key, [0, 0]); a[0] += float(m.group(1)); a[1] += float(m.group(2))
for k, (i, s) in sorted(g.items(), key=lambda kv: -kv[1][0]):
    print("%-45s instr %5.1f%%  stall %5.1f%%" % (k, i, s))
