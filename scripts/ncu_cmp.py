"""Dev tool: side-by-side raw metrics of two ncu reports (first kernel of each), filtered by regex."""
import csv, io, re, subprocess, sys
def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return {h: (v, u) for h, v, u in zip(rows[0], rows[2], rows[1])}
a, b = raw(sys.argv[1]), raw(sys.argv[2])
pat = re.compile(sys.argv[3])
for k in sorted(set(a) | set(b)):
    if pat.search(k):
        va, vb = a.get(k, ("-", ""))[0], b.get(k, ("-", ""))[0]
        if va != vb:
            print(f"{k[:95]:95s} {va:>18s} {vb:>18s} {a.get(k, b.get(k))[1]}")
