#!/bin/bash
O=gpurun_out/r02x
mkdir -p $O
for t in memcheck synccheck racecheck; do
  echo "== $t" >> $O/compute_sanitizer.txt
  timeout 1500 compute-sanitizer --tool $t --print-limit 10 python scripts/sanitize.py >> $O/compute_sanitizer.txt 2>&1
  echo "rc=$?" >> $O/compute_sanitizer.txt
done
ls -la $O
