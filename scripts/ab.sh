#!/bin/bash
# Dev: A/B of library builds (default vs libgemm_epilogue_<variant>.so) on a shape list, twice.
# usage: ab.sh OUT variant [variant ...]
OUT=$1; shift
SHAPES=("35 8464 2560 rr" "35 8464 2560 rc" "2048 2048 2048 rr" "1024 1024 1024 rr" "5124 704 2048 rr" "640 1024 3840 rc" "4096 4096 4096 rr" "1536 1280 2432 rc" "256 256 256 rr" "8192 8192 8192 rr")
for rep in 1 2; do
  for v in default "$@"; do
    f=$PWD/paper_2006_12645_b200/libgemm_epilogue_$v.so; [ "$v" = default ] && f=$PWD/paper_2006_12645_b200/libgemm_epilogue.so
    GE_LIBRARY_FILE=$f timeout 300 python scripts/timed_multi.py "${SHAPES[@]}" --cold >> $OUT 2>&1
  done
done
