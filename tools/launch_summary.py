"""Aggregate an ncu --csv launch list by kernel: duration (gpu__time_duration.sum) and,
when captured, DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum)."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
i = next(k for k, r in enumerate(rows) if r and r[0] == 'ID')
h = rows[i]; ik = h.index('Kernel Name'); iv = h.index('Metric Value'); iu = h.index('Metric Unit')
im = h.index('Metric Name')
agg = collections.OrderedDict()
TS = {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1, 'us': 1, 'msecond': 1e3, 'ms': 1e3}
BS = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'KB': 1e3, 'MB': 1e6, 'GB': 1e9}
for r in rows[i+1:]:
    if len(r) < len(h): continue
    k = r[ik].split('(')[0].replace('void ', '').replace('fb::', '')[:60]
    v = float(r[iv].replace(',', '')); u = r[iu]
    a = agg.setdefault(k, [0, 0.0, 0.0])
    if r[im] == 'gpu__time_duration.sum':
        a[0] += 1; a[1] += v * TS.get(u, 1)
    elif r[im].startswith('dram__bytes'):
        a[2] += v * BS.get(u, 1)
tot = sum(a[1] for a in agg.values())
for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    extra = "  %8.1f MB/launch %6.0f GB/s" % (b / n / 1e6, b / t / 1e3) if b else ""
    print("%-60s %6d %12.1f us %9.2f mean %5.1f%%%s" % (k, n, t, t / n, 100 * t / tot, extra))
