#!/bin/bash
# recheck lean producer (default) vs pft on the large shapes; end-of-epilogue wait_group.read (ewr)
O=gpurun_out/r02s3i
mkdir -p $O
SH=("256 256 256 rr" "1024 1024 1024 rr" "2048 2048 2048 rr" "35 8464 2560 rr" "4096 4096 4096 rr" "8192 8192 8192 rr" "8192 8192 8192 cc" "8192 8192 8192 rc")
for rep in 1 2 3; do
for v in pft default ewr; do
  f=$PWD/paper_2006_12645_b200/libgemm_epilogue_$v.so; [ "$v" = default ] && f=$PWD/paper_2006_12645_b200/libgemm_epilogue.so
  GE_LIBRARY_FILE=$f timeout 300 python scripts/timed_multi.py "${SH[@]}" --cold >> $O/ab.txt 2>&1
done
done
python scripts/ab_table.py $O/ab.txt
