#!/bin/bash
O=gpurun_out/r02v
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
S=("1024 1024 1024 rr" "2048 2048 2048 rr" "640 1024 3840 rc" "1536 1280 2432 rc" "5124 704 2048 rr" "768 1024 3456 rc" "2048 128 3456 rc" "35 8464 2560 rr" "4096 4096 4096 rr" "256 256 256 rr" "128 2176 3200 rc")
for rep in 1 2; do
for v in noearly default; do
  f=$PWD/paper_2006_12645_b200/libgemm_epilogue_$v.so; [ "$v" = default ] && f=$PWD/paper_2006_12645_b200/libgemm_epilogue.so
  GE_LIBRARY_FILE=$f timeout 300 python scripts/timed_multi.py "${S[@]}" --cold >> $O/ab.txt 2>&1
done
done
ls -la $O
