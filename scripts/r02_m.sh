#!/bin/bash
O=gpurun_out/r02m
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "half_row" > $O/pytest_hr.log 2>&1; echo "rc=$?" >> $O/pytest_hr.log
S=("1024 1024 1024 rr" "2048 2048 2048 rr" "640 1024 3840 rc" "1536 1280 2432 rc" "256 256 256 rr" "5124 704 2048 rr" "768 1024 3456 rc" "2048 128 3456 rc" "3072 3072 3072 rr" "128 2176 3200 rc")
timeout 600 python scripts/timed_multi.py "${S[@]}" --cold > $O/default.txt 2>&1
for bn in 128 256; do
  SS=()
  for sh in "${S[@]}"; do SS+=("$sh $bn 2"); done
  GE_FORCE_HR=1 timeout 600 python scripts/timed_multi.py "${SS[@]}" --cold --tile-m 128 > $O/hr$bn.txt 2>&1
done
ls -la $O
