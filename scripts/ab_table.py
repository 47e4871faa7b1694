"""Dev tool: min-over-reps table of timed_multi.py outputs per library variant."""
import collections
import re
import sys
d = collections.defaultdict(list)
order, libs = [], []
for f in sys.argv[1:]:
    for l in open(f):
        m = re.match(r"(\S+)\s+(.+?)\s+([\d.]+) us\s+([\d.]+) TF/s", l)
        if not m:
            continue
        lib = m.group(1).replace("libgemm_epilogue", "").replace(".so", "") or "default"
        sh = m.group(2).strip()
        d[(sh, lib)].append(float(m.group(3)))
        if sh not in order:
            order.append(sh)
        if lib not in libs:
            libs.append(lib)
print(f"{'shape (us, min of reps)':28s}" + "".join(f"{v:>12s}" for v in libs) + "   ratios vs " + libs[0])
for sh in order:
    row = [min(d.get((sh, v), [float('nan')])) for v in libs]
    print(f"{sh:28s}" + "".join(f"{x:12.2f}" for x in row) + "   " + " ".join(f"{row[0] / x:.3f}" for x in row[1:]))
