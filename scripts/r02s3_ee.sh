#!/bin/bash
# teardown cluster barrier without the release fence (pacq) vs HEAD (default), + tests on the variant
O=gpurun_out/r02s3ee
mkdir -p $O
GE_LIBRARY_FILE=$PWD/paper_2006_12645_b200/libgemm_epilogue_pacq.so timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
SH=("1024 1024 1024 rr" "2048 2048 2048 rr" "2048 2048 2048 cc" "5124 704 2048 rr" "1536 1280 2432 rc" "3072 3072 3072 rr" "640 1024 3840 rc" "35 8464 2560 rr" "4096 4096 4096 rr" "8192 8192 8192 rr")
for rep in 1 2 3; do
for v in default pacq; do
  f=$PWD/paper_2006_12645_b200/libgemm_epilogue_$v.so; [ "$v" = default ] && f=$PWD/paper_2006_12645_b200/libgemm_epilogue.so
  GE_LIBRARY_FILE=$f timeout 300 python scripts/timed_multi.py "${SH[@]}" --cold >> $O/ab.txt 2>&1
done
done
tail -3 $O/pytest.log
python scripts/ab_table.py $O/ab.txt
