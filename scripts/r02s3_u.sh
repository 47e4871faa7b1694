#!/bin/bash
# split-K: round-robin unit ownership + only the 16-B groups with columns < N exchanged (skx) vs HEAD
O=gpurun_out/r02s3u
mkdir -p $O
GE_LIBRARY_FILE=$PWD/paper_2006_12645_b200/libgemm_epilogue_skx.so timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
SH=("35 8464 2560 rr" "35 8464 2560 rc" "640 1024 3840 rc" "2048 128 3456 rc" "128 2176 3200 rr" "768 1024 3456 rc" "64 4096 4096 rr" "1024 1024 1024 rr")
for rep in 1 2 3; do
for v in default skx; do
  f=$PWD/paper_2006_12645_b200/libgemm_epilogue_$v.so; [ "$v" = default ] && f=$PWD/paper_2006_12645_b200/libgemm_epilogue.so
  GE_LIBRARY_FILE=$f timeout 300 python scripts/timed_multi.py "${SH[@]}" --cold >> $O/ab.txt 2>&1
done
done
tail -3 $O/pytest.log
python scripts/ab_table.py $O/ab.txt
