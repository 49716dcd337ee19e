"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
i = next(k for k, r in enumerate(rows) if r and r[0] == 'ID')
h = rows[i]; ik = h.index('Kernel Name'); iv = h.index('Metric Value'); iu = h.index('Metric Unit')
agg = collections.OrderedDict()
for r in rows[i+1:]:
    if len(r) < len(h): continue
    k = r[ik].split('(')[0].replace('void ', '').replace('fb::', '')[:60]
    v = float(r[iv].replace(',', '')); u = r[iu]
    v = v * {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1, 'us': 1, 'msecond': 1e3, 'ms': 1e3}.get(u, 1)
    a = agg.setdefault(k, [0, 0.0]); a[0] += 1; a[1] += v
tot = sum(a[1] for a in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print("%-60s %6d %12.1f us %9.2f mean %5.1f%%" % (k, n, t, t / n, 100 * t / tot))
