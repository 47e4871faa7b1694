"""Dev tool: one line per bench JSON line (value, per-launch time, roofline, comparators)."""
import json
import sys
for f in sys.argv[1:]:
    for l in open(f):
        if not l.startswith("{"):
            continue
        d = json.loads(l)
        r = d.get("roofline", {})
        c = d.get("comparators") or {}
        print(f"{d['config']['workload'][:34]:34s} {d['value']:8.1f} {d['unit']:8s} kern {r.get('kernel_avg_ms', 0) * 1e3:8.2f} us "
              f"{r.get('bound', '-'):6s} {r.get('achieved', 0):8.1f} {r.get('unit', ''):7s} frac {r.get('frac', 0):.3f} | "
              f"LtRelu {c.get('cublaslt_addmm_relu', 0):7.1f} mm {c.get('torch_matmul_only', 0):7.1f} unf {c.get('torch_unfused_matmul_add_relu', 0):7.1f}"
              f" | e2e {(d.get('e2e') or {}).get('value', 0):6.1f} clk {d.get('clocks', {}).get('sm_mhz')} {d.get('clocks', {}).get('reasons')}")
        if d.get("scale_series"):
            print("   scale_series", d["scale_series"])
