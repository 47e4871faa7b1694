"""Dev tool: warp-stall samples of an `ncu --page source --csv --print-source sass` dump, by stall
reason, and the no_inst / wait samples by code region (runs of executed instructions).
usage: ncu_stall_regions.py src.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
col = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = []
for r in rows[2:]:
    try:
        data.append({"addr": int(r[col["Address"]], 16), "src": r[col["Source"]].strip(),
                     "samp": int(r[col["Warp Stall Sampling (All Samples)"]] or 0),
                     "exec": int(r[col["Instructions Executed"]] or 0),
                     **{s: int(r[col[s]] or 0) for s in stalls}})
    except (ValueError, IndexError, KeyError):
        pass
tot = sum(d["samp"] for d in data)
print(f"total samples {tot}, instructions with samples {sum(1 for d in data if d['samp'])}, "
      f"executed instructions {sum(1 for d in data if d['exec'])} of {len(data)}")
for s in sorted(stalls, key=lambda s: -sum(d[s] for d in data))[:10]:
    print(f"  {s:28s} {sum(d[s] for d in data):8d} ({100 * sum(d[s] for d in data) / max(1, tot):5.1f}%)")
# regions: split at gaps of non-executed instructions > 32
base = data[0]["addr"] if data else 0
regions, cur = [], None
for d in data:
    if d["exec"] == 0:
        continue
    if cur is None or d["addr"] - cur["end"] > 32 * 16:
        cur = {"start": d["addr"], "end": d["addr"], "samp": 0, "no_inst": 0, "n": 0, "first": d["src"]}
        regions.append(cur)
    cur["end"] = d["addr"]
    cur["samp"] += d["samp"]
    cur["no_inst"] += d.get("stall_no_inst", 0)
    cur["n"] += 1
print("top regions by samples (offset from kernel start, executed instructions, samples, no_inst):")
for g in sorted(regions, key=lambda g: -g["samp"])[:14]:
    print(f"  +{(g['start'] - base):#8x}..+{(g['end'] - base):#8x}  n={g['n']:5d}  samples {g['samp']:6d}  "
          f"no_inst {g['no_inst']:5d}  first: {g['first'][:60]}")
