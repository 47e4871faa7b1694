#!/bin/bash
# A-operand collector reuse across the two accumulator halves (default) vs HEAD
O=gpurun_out/r02s3k
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "512 or prologue or hadamard or fullsize or configs" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for rep in 1 2 3; do
for v in head default; do
  f=$PWD/paper_2006_12645_b200/libgemm_epilogue_$v.so; [ "$v" = default ] && f=$PWD/paper_2006_12645_b200/libgemm_epilogue.so
  GE_LIBRARY_FILE=$f timeout 300 python scripts/timed_multi.py "8192 8192 8192 rr" "8192 8192 8192 cc" "4096 4096 4096 rr 512 2" "6144 6144 6144 rr" --cold >> $O/ab.txt 2>&1
  GE_LIBRARY_FILE=$f timeout 300 python scripts/timed_multi.py "4096 4096 4096 rr" "8192 8192 8192 rr" --prologue scale_k --cold >> $O/ab_pro.txt 2>&1
  GE_LIBRARY_FILE=$f timeout 300 python scripts/timed_multi.py "4096 4096 4096 rr" --prologue hadamard --cold >> $O/ab_pro.txt 2>&1
done
done
tail -3 $O/pytest.log
python scripts/ab_table.py $O/ab.txt
python scripts/ab_table.py $O/ab_pro.txt
