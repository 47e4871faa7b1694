#!/bin/bash
# parameter-block warm-up at kernel entry: timeline + A/B
O=gpurun_out/r02s3dd
mkdir -p $O
GE_LIBRARY_FILE=$PWD/paper_2006_12645_b200/libgemm_epilogue_warmdbg.so timeout 300 python scripts/timeline.py "1024 1024 1024 rr" "2048 2048 2048 rr" > $O/timeline.txt 2>&1
grep -A2 "==\|  i " $O/timeline.txt | grep "==\|med\|  i "
SH=("256 256 256 rr" "1024 1024 1024 rr" "2048 2048 2048 rr" "5124 704 2048 rr" "35 8464 2560 rr" "640 1024 3840 rc" "1536 1280 2432 rc")
for rep in 1 2 3; do
for v in default warm; do
  f=$PWD/paper_2006_12645_b200/libgemm_epilogue_$v.so; [ "$v" = default ] && f=$PWD/paper_2006_12645_b200/libgemm_epilogue.so
  GE_LIBRARY_FILE=$f timeout 300 python scripts/timed_multi.py "${SH[@]}" --cold >> $O/ab.txt 2>&1
done
done
python scripts/ab_table.py $O/ab.txt
