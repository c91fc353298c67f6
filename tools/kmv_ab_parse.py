"""Median kernel duration per (config, library) from an ncu launch list of
tools/kmv_ab.py (-k regex:kmv_sym_kernel): python tools/kmv_ab_parse.py CSV LIB..."""
import csv
import sys

path, libs = sys.argv[1], ["current"] + [a.split("/")[-1] for a in sys.argv[2:]]
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr = rows[0]
vi = hdr.index("Metric Value")
seq = [float(r[vi]) for r in rows[1:]]
i = 0
for cfg, reps in (("C2", 203), ("C3", 13)):
    for lib in libs:
        xs = sorted(seq[i + 3:i + reps])
        i += reps
        print(f"{cfg} {lib:24s} median {xs[len(xs) // 2] / 1e3:10.1f} us")
