"""Dev tool: print the key metrics of ncu --set full captures (.ncu-rep) side by side.
usage: ncu_keys.py rep1 [rep2 ...] [--grep REGEX]"""
import csv, io, re, subprocess, sys
KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum", "launch__grid_size",
        "launch__cluster_dim_x", "launch__registers_per_thread", "smsp__inst_executed.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed"]
argv = sys.argv[1:]
pat = None
if "--grep" in argv:
    i = argv.index("--grep")
    pat = re.compile(argv[i + 1])
    argv = argv[:i] + argv[i + 2:]
tabs = []
for rep in argv:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, last = rows[0], rows[1], rows[-1]
    tabs.append({h: (v, u) for h, v, u in zip(hdr, last, units)})
keys = [k for k in tabs[0] if pat.search(k)] if pat else KEYS
for k in keys:
    vals = [t.get(k, ("-", ""))[0] for t in tabs]
    print(f"{k:75s} " + " ".join(f"{v:>16s}" for v in vals) + "  " + tabs[0].get(k, ("", ""))[1])
