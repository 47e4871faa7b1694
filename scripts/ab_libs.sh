#!/bin/bash
# Dev: A/B timing of alternative library builds (GE_LIBRARY_FILE) over a few shapes/configs.
# usage: scripts/ab_libs.sh "variant1 variant2 ..." ("" = default build)
cd "$(dirname "$0")/.."
CASES=${CASES:-"640 1024 3840 rc 64 1|640 1024 3840 rc 128 1|640 1024 3840 rc 256 1|640 1024 3840 rc 128 2|3840 2560 3584 rc 256 2|4096 4096 4096 rr 256 2|8192 8192 8192 rr 512 2"}
IFS='|' read -ra CS <<< "$CASES"
for c in "${CS[@]}"; do
  for v in $1; do
    f=paper_2006_12645_b200/libgemm_epilogue_$v.so; [ "$v" = default ] && f=paper_2006_12645_b200/libgemm_epilogue.so
    echo -n "$c [$v] "; GE_LIBRARY_FILE=$PWD/$f timeout 60 python scripts/timed.py $c 100 | tail -1
  done
done
