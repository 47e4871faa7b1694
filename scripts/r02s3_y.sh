#!/bin/bash
# pipelined TMEM-resident prologue A: parity, timing vs in place, transform counters
O=gpurun_out/r02s3y
mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -x -k "prologue" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
for rep in 1 2; do
timeout 300 python scripts/timed_multi.py "4096 4096 4096 rr 256 2" "4096 4096 4096 rr 512 2" "4096 4096 4096 cc 256 2" "4096 4096 4096 cc 512 2" "8192 8192 8192 rr 256 2" "8192 8192 8192 rr 512 2" "2048 2048 2048 rr 256 2" "2048 2048 2048 rr 512 2" --prologue scale_k --cold >> $O/t.txt 2>&1
timeout 300 python scripts/timed_multi.py "4096 4096 4096 rr 256 2" "4096 4096 4096 rr 512 2" --prologue relu --cold >> $O/t.txt 2>&1
timeout 300 python scripts/timed_multi.py "4096 4096 4096 rr 256 2" "4096 4096 4096 rr" --cold >> $O/t.txt 2>&1
done
python scripts/ab_table.py $O/t.txt
for shp in "4096 4096 4096 rr 256 2 0 0 scale_k"; do
  set -- $shp
  GE_DEBUG_STATS=1 timeout 120 python scripts/debug_stats.py $@ 2>&1 | grep "total\|transform\|mma_wait_full\|tempty"
done
