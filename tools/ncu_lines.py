"""Aggregate ncu warp-stall samples per CUDA source line:
    ncu -i rep --page source --csv --print-source cuda,sass > cs.csv
    python tools/ncu_lines.py cs.csv [top]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur_file = None; agg = {}; hdr = None; last = None; stalls = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if r[0] == "Function Name" or hdr is None or len(r) < 5:
        continue
    try:
        v = int(r[4] or 0)
    except ValueError:
        continue
    if r[0]:
        last = (cur_file, r[0], r[1].strip()[:70])
    if last is None:
        continue
    agg[last] = agg.get(last, 0) + v
    if v:
        for h, x in zip(hdr, r):
            if h.startswith("stall_") and "Not" not in h and x and x != "0":
                stalls.setdefault(last, {}).setdefault(h, 0)
                stalls[last][h] += int(x)
tot = sum(agg.values())
print("total samples", tot)
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    st = sorted(stalls.get(k, {}).items(), key=lambda x: -x[1])[:2]
    print(f"{100 * v / tot:5.1f}% {k[0]}:{k[1]} {k[2]}  {st}")
