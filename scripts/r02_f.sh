#!/bin/bash
O=gpurun_out/r02f
mkdir -p $O
for v in "" ld0 ld2; do
  if [ -n "$v" ]; then export GE_LIBRARY_FILE=$PWD/paper_2006_12645_b200/libgemm_epilogue_$v.so; else unset GE_LIBRARY_FILE; fi
  echo "== variant ${v:-ld1}" >> $O/bench.jsonl
  timeout 300 python bench.py --workload prologue4096 --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-comparators >> $O/bench.jsonl 2>> $O/bench.err
done
unset GE_LIBRARY_FILE
timeout 600 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
ls -la $O
