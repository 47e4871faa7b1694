#!/bin/bash
# A/B: skinny shapes, old (st.global transposed store) vs new (transposed TMA store); split-K vs none
O=gpurun_out/r02s3c
mkdir -p $O
for rep in 1 2; do
for v in old default; do
  f=$PWD/paper_2006_12645_b200/libgemm_epilogue_$v.so; [ "$v" = default ] && f=$PWD/paper_2006_12645_b200/libgemm_epilogue.so
  GE_LIBRARY_FILE=$f timeout 300 python scripts/timed_multi.py "35 8464 2560 rr" "35 8464 2560 rc" "35 8464 2560 rr" --alt rc --cold >> $O/ab.txt 2>&1
  GE_LIBRARY_FILE=$f timeout 300 python scripts/timed_multi.py "35 8464 2560 rr" "35 8464 2560 rc" --kw "stream_k=1" --cold >> $O/ab.txt 2>&1
  GE_LIBRARY_FILE=$f timeout 300 python scripts/timed_multi.py "35 8464 2560 rr 128 1" "35 8464 2560 rc 128 1" --cold >> $O/ab.txt 2>&1
done
done
cat $O/ab.txt
