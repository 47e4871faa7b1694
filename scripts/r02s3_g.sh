#!/bin/bash
# producer: first tile decoded before griddepcontrol.wait, 32-bit decode, no empty waits on the first
# ring pass -- GPU tests, timeline, A/B vs the previous build (trans)
O=gpurun_out/r02s3g
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
GE_LIBRARY_FILE=$PWD/paper_2006_12645_b200/libgemm_epilogue_dbg.so timeout 300 python scripts/timeline.py "256 256 256 rr" "1024 1024 1024 rr" "2048 2048 2048 rr" "35 8464 2560 rr" "5124 704 2048 rr" > $O/timeline.txt 2>&1
SH=("256 256 256 rr" "1024 1024 1024 rr" "2048 2048 2048 rr" "5124 704 2048 rr" "35 8464 2560 rr" "640 1024 3840 rc" "1536 1280 2432 rc" "4096 4096 4096 rr" "8192 8192 8192 rr")
for rep in 1 2; do
for v in trans default; do
  f=$PWD/paper_2006_12645_b200/libgemm_epilogue_$v.so; [ "$v" = default ] && f=$PWD/paper_2006_12645_b200/libgemm_epilogue.so
  GE_LIBRARY_FILE=$f timeout 300 python scripts/timed_multi.py "${SH[@]}" --cold >> $O/ab.txt 2>&1
done
done
tail -3 $O/pytest.log
grep -A3 "==\|med" $O/timeline.txt
python scripts/ab_table.py $O/ab.txt
