#!/bin/bash
O=gpurun_out/r02o
mkdir -p $O
for v in rel4 nofence both; do
  GE_LIBRARY_FILE=$PWD/paper_2006_12645_b200/libgemm_epilogue_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tile_configs or split_k or stream_k or odd_shapes or layouts_ragged or multicast or half_row or prologue" > $O/pytest_$v.log 2>&1; echo "rc=$?" >> $O/pytest_$v.log
done
S=("1024 1024 1024 rr" "2048 2048 2048 rr" "640 1024 3840 rc" "1536 1280 2432 rc" "5124 704 2048 rr" "768 1024 3456 rc" "2048 128 3456 rc" "35 8464 2560 rr" "4096 4096 4096 rr" "256 256 256 rr")
for rep in 1 2; do
for v in default rel4 nofence both; do
  f=$PWD/paper_2006_12645_b200/libgemm_epilogue_$v.so; [ "$v" = default ] && f=$PWD/paper_2006_12645_b200/libgemm_epilogue.so
  GE_LIBRARY_FILE=$f timeout 300 python scripts/timed_multi.py "${S[@]}" --cold >> $O/ab.txt 2>&1
done
done
ls -la $O
