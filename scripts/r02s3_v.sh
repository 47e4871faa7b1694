#!/bin/bash
# TMEM-resident prologue A: parity first, then timing vs the in-place transform
O=gpurun_out/r02s3v
mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -x -k "prologue" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -5 $O/pytest.log
for rep in 1 2; do
timeout 300 python scripts/timed_multi.py "4096 4096 4096 rr 256 2" "4096 4096 4096 rr 512 2" "4096 4096 4096 cc 256 2" "8192 8192 8192 rr 256 2" "8192 8192 8192 rr 512 2" "2048 2048 2048 rr 256 2" --prologue scale_k --cold >> $O/t.txt 2>&1
timeout 300 python scripts/timed_multi.py "4096 4096 4096 rr 256 2" "4096 4096 4096 rr 512 2" "4096 4096 4096 cc 256 2" --prologue relu --cold >> $O/t.txt 2>&1
done
cat $O/t.txt
