#!/bin/bash
# Hadamard prologue: 3-stage 256x512 ring (default now) vs 256x256 vs the previous 2-stage build (pft)
O=gpurun_out/r02s3j
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "hadamard or prologue" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for rep in 1 2; do
for v in pft default; do
  f=$PWD/paper_2006_12645_b200/libgemm_epilogue_$v.so; [ "$v" = default ] && f=$PWD/paper_2006_12645_b200/libgemm_epilogue.so
  GE_LIBRARY_FILE=$f timeout 300 python scripts/timed_multi.py "4096 4096 4096 rr" "4096 4096 4096 rr 256 2" "4096 4096 4096 cc" "4096 4096 4096 cc 256 2" "2048 2048 2048 rr" "8192 8192 8192 rr" --prologue hadamard --cold >> $O/ab.txt 2>&1
  GE_LIBRARY_FILE=$f timeout 300 python scripts/timed_multi.py "4096 4096 4096 rr" "4096 4096 4096 rr 256 2" "4096 4096 4096 cc" --prologue scale_k --cold >> $O/ab_scale.txt 2>&1
done
done
tail -3 $O/pytest.log
python scripts/ab_table.py $O/ab.txt
python scripts/ab_table.py $O/ab_scale.txt
