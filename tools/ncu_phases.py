"""Group tools/ncu_lines.py output of k_step into phases (line ranges of finom_1d.cu)."""
import collections
import re
import sys

R = [(330, 372, 'walk helpers'), (375, 409, 'walk setup'), (410, 421, 'operands'),
     (422, 431, 'pass1'), (432, 468, 'carry+scan'), (469, 482, 'pass2+out'),
     (488, 514, 'compute setup'), (515, 542, 'epi rows'), (543, 566, 'epi red/node'),
     (567, 680, 'loads/kernel'), (220, 329, 'bulk/bar')]
ph = collections.defaultdict(float)
st = collections.defaultdict(float)
for ln in sys.stdin:
    m = re.match(r'\s*([\d.]+)% instr\s+([\d.]+)% stall\s+(\S+):(\d*)', ln)
    if not m:
        print(ln.rstrip())
        continue
    f, l = m.group(3), int(m.group(4) or 0)
    name = f
    if f == 'finom_1d.cu':
        name = next((n for a, b, n in R if a <= l <= b), 'finom:%d' % l)
    elif f == 'tile_core.cuh':
        name = 'tile_core'
    ph[name] += float(m.group(1))
    st[name] += float(m.group(2))
for k, v in sorted(ph.items(), key=lambda kv: -kv[1]):
    print('%6.1f%% instr %6.1f%% stall  %s' % (v, st[k], k))
