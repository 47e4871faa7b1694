#!/bin/bash
O=gpurun_out/r02k
mkdir -p $O
GE_LIBRARY_FILE=$PWD/paper_2006_12645_b200/libgemm_epilogue_xw8.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "prologue or hadamard or golden" > $O/pytest_xw8.log 2>&1; echo "rc=$?" >> $O/pytest_xw8.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "swap or fast_epilogue or epilogue_variants" > $O/pytest_swapfast.log 2>&1; echo "rc=$?" >> $O/pytest_swapfast.log
for rep in 1 2; do
for v in "" xw8; do
  if [ -n "$v" ]; then export GE_LIBRARY_FILE=$PWD/paper_2006_12645_b200/libgemm_epilogue_$v.so; else unset GE_LIBRARY_FILE; fi
  for w in prologue4096 hadamard4096; do
    echo "== ${v:-xw4} $w" >> $O/bench.txt
    timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-comparators >> $O/bench.txt 2>> $O/bench.err
  done
done
done
unset GE_LIBRARY_FILE
timeout 300 python bench.py --workload deepbench_b --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/deepbench_b.json 2>&1
timeout 300 python scripts/timed_multi.py "35 8464 2560 rr" "35 8464 2560 rc" --cold > $O/skinny.txt 2>&1
ls -la $O
