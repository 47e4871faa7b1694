#!/bin/bash
# Final session-3 evidence on the committed build: GPU tests, default bench line, workload lines,
# launch list + ncu --set full of the bench kernel and the skinny / 2048^3 kernels, paper sweep.
O=/tmp/evf
G=gpurun_out/final3
rm -rf $O; mkdir -p $O $G $G/profiles
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for w in square256 square1024 square2048 square4096 deepbench_a deepbench_b prologue4096 hadamard4096 batched64x2048; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline >> $O/bench_workloads.jsonl 2>> $O/bench_workloads.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_square8192.csv \
  python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-comparators --no-cpu-baseline --no-scale-series > $O/bench_under_ncu.log 2>&1
cap() {  # workload M N K lay pro batch
  timeout 600 ncu --set full --import-source on --clock-control none -c 1 -k regex:ge_fused -o $O/$1 \
    python scripts/one_call.py $2 $3 $4 $5 0 0 2 $6 $7 > $O/$1.log 2>&1
}
cap square8192 8192 8192 8192 rr none 1
cap square2048 2048 2048 2048 rr none 1
cap square1024 1024 1024 1024 rr none 1
cap square256 256 256 256 rr none 1
cap deepbench_a 5124 700 2048 rr none 1
cap deepbench_b 35 8457 2560 rr none 1
cap hadamard4096 4096 4096 4096 rr hadamard 1
timeout 1200 python scripts/paper_sweep.py --cpg 1 --out $O/paper_sweep.json > $O/paper_sweep.log 2>&1
timeout 1200 python scripts/paper_sweep.py --cpg 20 --out $O/paper_sweep_cpg20.json > $O/paper_sweep_cpg20.log 2>&1
python scripts/summarize_evidence.py $O 2 > $G/summarize.log 2>&1
cp profiles/r02_ncu_* profiles/r02_launches_* profiles/ncu_summary.json $G/profiles/ 2>/dev/null
cp $O/*.json $O/*.jsonl $O/*.log $O/*.err $O/*.csv $G/ 2>/dev/null
for f in $O/*.ncu-rep; do ncu -i $f --page raw --csv > $G/$(basename $f .ncu-rep)_raw.csv 2>/dev/null; done
du -sh $G
