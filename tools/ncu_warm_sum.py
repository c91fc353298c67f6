"""Per-kernel sums of a warm ncu launch list (--cache-control none csv)."""
import csv, collections, io, sys
txt = open(sys.argv[1]).read()
i = txt.index('"ID","Process ID"')
rows = [r for r in csv.reader(io.StringIO(txt[i:])) if len(r) > 10]
h = rows[0]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
agg = collections.OrderedDict()
for r in rows[1:]:
    n = r[ki].split('(')[0].replace('void ', '').replace('afn::', '').replace('<unnamed>::', '')[:50]
    a = agg.setdefault(n, [0, 0.0]); a[0] += 1; a[1] += float(r[vi].replace(',', '')) / 1e3
tot = sum(v[1] for v in agg.values())
print('total us %.1f' % tot)
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print('%-50s %5d %10.1f us %8.1f' % (n, c, t, t / c))
