"""Dev tool: top SASS lines by warp-stall samples from an `ncu --page source --csv` dump."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, isamp = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[isamp] or 0), r[ia], r[isrc]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data)
print("total samples", tot)
for s, a, src in sorted(data, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{s:7d} {100*s/tot:5.1f}%  {a}  {src[:110]}")
