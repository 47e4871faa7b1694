#!/bin/bash
# large-shape recheck: setup-init build (default) vs the build before it (prev), interleaved reps
O=gpurun_out/r02s3n
mkdir -p $O
for rep in 1 2 3 4; do
for v in prev default; do
  f=$PWD/paper_2006_12645_b200/libgemm_epilogue_$v.so; [ "$v" = default ] && f=$PWD/paper_2006_12645_b200/libgemm_epilogue.so
  GE_LIBRARY_FILE=$f timeout 300 python scripts/timed_multi.py "8192 8192 8192 rr" "8192 8192 8192 cc" "6144 6144 6144 rr" "4096 4096 4096 rr" "1024 1024 1024 rr" --cold >> $O/ab.txt 2>&1
done
done
python scripts/ab_table.py $O/ab.txt
