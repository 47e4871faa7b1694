#!/bin/bash
O=gpurun_out/r02l
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
S=("35 8464 2560 rr" "1024 1024 1024 rr" "2048 2048 2048 rr" "5124 704 2048 rr" "4096 4096 4096 rr" "640 1024 3840 rc" "1536 1280 2432 rc")
for rep in 1 2; do
for v in prev default; do
  f=$PWD/paper_2006_12645_b200/libgemm_epilogue_$v.so; [ "$v" = default ] && f=$PWD/paper_2006_12645_b200/libgemm_epilogue.so
  GE_LIBRARY_FILE=$f timeout 300 python scripts/timed_multi.py "${S[@]}" --cold >> $O/ab.txt 2>&1
  GE_LIBRARY_FILE=$f timeout 300 python scripts/timed_multi.py "${S[@]}" --cold --alt cc >> $O/ab.txt 2>&1
done
done
for w in square1024 square2048 deepbench_b; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 >> $O/bench.jsonl 2>> $O/bench.err
done
ls -la $O
