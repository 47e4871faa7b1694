#!/bin/bash
# Dev: one bench line per BASELINE workload (no CPU baseline, 1 e2e step), summarised.
for w in ${WL:-square8192 square4096 square2048 square1024 deepbench_a deepbench_b prologue4096 batched64x2048}; do
  python bench.py --workload $w --steps ${STEPS:-30} --warmup 5 --e2e-steps 1 --no-cpu-baseline 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read())
c=d.get('comparators') or {}
print(f\"{'$w':16s} {d['value']:8.1f} TF/s  kern {d['roofline']['achieved']:8.1f}  frac {d['roofline']['frac']:.3f}  e2e {d['e2e']['value']:7.1f}  clk {d['clocks'].get('sm_mhz')}  torch_unfused {c.get('torch_unfused_matmul_add_relu',0):7.1f} cublasLt {c.get('cublaslt_addmm_relu',0):7.1f} matmul {c.get('torch_matmul_only',0):7.1f}\")
"
done
