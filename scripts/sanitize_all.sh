for t in memcheck synccheck racecheck; do
  echo "== $t"; timeout 900 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize.py 2>&1 | tail -25
done
