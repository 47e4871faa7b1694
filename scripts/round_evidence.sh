#!/bin/bash
# Round evidence on a GPU box: the default bench line, extra workload lines, the ncu launch list of
# the bench command and one --set full capture of the bench kernel, summarised into profiles/
# (copied to gpurun_out/profiles_new/ so gpurun brings them back).  usage: round_evidence.sh ROUND
R=${1:-1}
mkdir -p gpurun_out/profiles_new
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for w in square4096 square2048 batched64x2048 prologue4096 deepbench_a deepbench_b square1024; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline >> gpurun_out/bench_workloads.jsonl 2>> gpurun_out/bench_workloads.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 > gpurun_out/bench_under_ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -c 1 -k regex:ge_fused -o /tmp/prof \
  python scripts/one_call.py 8192 8192 8192 rr 0 0 1 > /dev/null 2>&1
python scripts/summarize_ncu.py --round $R --launches gpurun_out/launches.csv --full /tmp/prof.ncu-rep --workload square8192 \
  > gpurun_out/summarize.log 2>&1
cp profiles/r0${R}_launches_square8192.csv profiles/r0${R}_launches_square8192_summary.txt profiles/r0${R}_ncu_square8192.txt \
   profiles/ncu_summary.json gpurun_out/profiles_new/ 2>/dev/null
ncu -i /tmp/prof.ncu-rep --page raw --csv > gpurun_out/profiles_new/raw_square8192.csv 2>/dev/null
ls -la gpurun_out/profiles_new
