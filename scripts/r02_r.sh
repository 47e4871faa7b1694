#!/bin/bash
O=gpurun_out/r02r
mkdir -p $O
GE_LIBRARY_FILE=$PWD/paper_2006_12645_b200/libgemm_epilogue_split.so timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_split.log 2>&1; echo "pytest rc=$?" >> $O/pytest_split.log
S=("1024 1024 1024 rr" "2048 2048 2048 rr" "2048 2048 2048 cc" "640 1024 3840 rc" "1536 1280 2432 rc" "5124 704 2048 rr" "768 1024 3456 rc" "2048 128 3456 rc" "35 8464 2560 rr" "4096 4096 4096 rr" "256 256 256 rr" "8192 8192 8192 rr" "8192 8192 8192 cc")
for rep in 1 2; do
for v in default split; do
  f=$PWD/paper_2006_12645_b200/libgemm_epilogue_$v.so; [ "$v" = default ] && f=$PWD/paper_2006_12645_b200/libgemm_epilogue.so
  GE_LIBRARY_FILE=$f timeout 300 python scripts/timed_multi.py "${S[@]}" --cold >> $O/ab.txt 2>&1
done
done
ls -la $O
