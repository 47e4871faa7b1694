#!/bin/bash
# teardown cluster barrier without the release fence (wid) vs HEAD (default), + tests on the variant
O=gpurun_out/r02s3bb
mkdir -p $O
GE_LIBRARY_FILE=$PWD/paper_2006_12645_b200/libgemm_epilogue_wid.so timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
SH=("256 256 256 rr" "1024 1024 1024 rr" "2048 2048 2048 rr" "5124 704 2048 rr" "35 8464 2560 rr" "640 1024 3840 rc" "1536 1280 2432 rc" "4096 4096 4096 rr" "8192 8192 8192 rr" "8192 8192 8192 cc")
for rep in 1 2 3; do
for v in default wid; do
  f=$PWD/paper_2006_12645_b200/libgemm_epilogue_$v.so; [ "$v" = default ] && f=$PWD/paper_2006_12645_b200/libgemm_epilogue.so
  GE_LIBRARY_FILE=$f timeout 300 python scripts/timed_multi.py "${SH[@]}" --cold >> $O/ab.txt 2>&1
done
done
tail -3 $O/pytest.log
python scripts/ab_table.py $O/ab.txt
for rep in 1 2; do
for v in default wid; do
  f=$PWD/paper_2006_12645_b200/libgemm_epilogue_$v.so; [ "$v" = default ] && f=$PWD/paper_2006_12645_b200/libgemm_epilogue.so
  GE_LIBRARY_FILE=$f timeout 300 python scripts/timed_multi.py "4096 4096 4096 rr" "8192 8192 8192 rr" --prologue scale_k --cold >> $O/ab_pro.txt 2>&1
  GE_LIBRARY_FILE=$f timeout 300 python scripts/timed_multi.py "4096 4096 4096 rr" --prologue hadamard --cold >> $O/ab_pro.txt 2>&1
done
done
python scripts/ab_table.py $O/ab_pro.txt
