"""Dev tool: summarise an evidence directory (scripts/r02_evidence.sh output) into profiles/:
the ncu --set full captures of every workload (key metrics, DRAM traffic vs algorithmic bytes,
merged into profiles/ncu_summary.json for bench.py's roofline.traffic), the launch list of the
bench command, the bench lines and the paper sweeps.  usage: summarize_evidence.py DIR ROUND"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402  (WORKLOADS, algorithmic_bytes)

d, rnd = sys.argv[1], int(sys.argv[2])
tag = f"r{rnd:02d}"
prof = os.path.join(ROOT, "profiles")
shapes = {"square8192": (1, 8192, 8192, 8192, None), "square4096": (1, 4096, 4096, 4096, None),
          "square2048": (1, 2048, 2048, 2048, None), "square256": (1, 256, 256, 256, None),
          "deepbench_a": (1, 5124, 700, 2048, None), "deepbench_b": (1, 35, 8457, 2560, None),
          "prologue4096": (1, 4096, 4096, 4096, "scale_k"), "hadamard4096": (1, 4096, 4096, 4096, "hadamard"),
          "square1024": (1, 1024, 1024, 1024, None), "batched64x2048": (64, 2048, 2048, 2048, None)}
for w, (b, M, N, K, pro) in shapes.items():
    rep = os.path.join(d, w + ".ncu-rep")
    if not os.path.exists(rep):
        continue
    flop = 2.0 * b * M * N * K
    algo = bench.algorithmic_bytes(b, M, N, K, pro)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "summarize_ncu.py"), "--round", str(rnd),
                        "--full", rep, "--workload", w, "--flop", str(flop), "--algo-bytes", str(algo)],
                       capture_output=True, text=True)
    print(w, r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:])
launches = os.path.join(d, "launches_square8192.csv")
if os.path.exists(launches):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "summarize_ncu.py"), "--round", str(rnd),
                        "--launches", launches, "--workload", "square8192"], capture_output=True, text=True)
    print(r.stdout[-400:], r.stderr[-400:])
for src, dst in (("bench_default.json", f"{tag}_bench_square8192.json"),
                 ("bench_workloads.jsonl", f"{tag}_bench_workloads.jsonl"),
                 ("paper_sweep.json", f"{tag}_paper_sweep.json"),
                 ("paper_sweep_cpg20.json", f"{tag}_paper_sweep_cpg20.json"),
                 ("pytest_gpu.log", f"{tag}_pytest_gpu.log"),
                 ("tune_rr_default.json", f"{tag}_tune_rr_default.json"),
                 ("compute_sanitizer.txt", f"{tag}_compute_sanitizer.txt")):
    if os.path.exists(os.path.join(d, src)):
        shutil.copy(os.path.join(d, src), os.path.join(prof, dst))
