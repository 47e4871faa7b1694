# Dev: A/B of two library builds (default vs libgemm_epilogue_$1.so) on auto-planned shapes, twice.
for rep in 1 2; do
for c in "2048 2048 2048 rr" "5124 704 2048 rr" "4096 4096 4096 rr" "3072 3072 3072 rc" "640 1024 3840 rc" "2048 128 3456 rc" "128 2176 3200 rc" "1024 1024 1024 rr" "1536 1280 2432 rc"; do
  for v in default $1; do
    f=paper_2006_12645_b200/libgemm_epilogue_$v.so; [ "$v" = default ] && f=paper_2006_12645_b200/libgemm_epilogue.so
    echo -n "$c [$v] "; GE_LIBRARY_FILE=$PWD/$f timeout 60 python scripts/timed.py $c 0 0 400 | tail -1
  done
done; done
