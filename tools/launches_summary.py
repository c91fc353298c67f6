"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections, csv, re, sys
path = sys.argv[1]
lines = [l for l in open(path) if l.startswith('"')]
rd = csv.reader(lines)
hdr = next(rd)
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
for r in rd:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"]
    name = re.sub(r"\(.*$", "", name)
    name = name.replace("void ", "").replace("afn::<unnamed>::", "").replace("afn::", "")
    agg[name][0] += 1
    agg[name][1] += float(d["Metric Value"].replace(",", "")) * scale[d["Metric Unit"]]
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':46s} {'launches':>8s} {'ms':>10s} {'share':>6s} {'ms/launch':>10s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:46]:46s} {v[0]:8d} {v[1]:10.3f} {100*v[1]/tot:5.1f}% {v[1]/v[0]:10.4f}")
print(f"{'total':46s} {sum(v[0] for v in agg.values()):8d} {tot:10.3f}")
