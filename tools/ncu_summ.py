"""Write profiles/ summaries of an ncu --set full report: the details page
(text) and the raw metrics bench.py reads (dram bytes per launch), one pair
of files per kernel. usage: ncu_summ.py REP.ncu-rep TAG 'regex:name' OUTSTEM"""
import csv
import io
import subprocess
import sys

rep, tag, kname, stem = sys.argv[1:5]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--kernel-name", kname],
                     capture_output=True, text=True).stdout
open(f"profiles/{stem}_{tag}.txt", "w").write(det)
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--kernel-name", kname],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_bytes.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]
out = [f"Kernel Name  {v[h.index('Kernel Name')]}"]
for w in want:
    if w in h:
        i = h.index(w)
        out.append(f"{w} {u[i]} {v[i]}")
open(f"profiles/{stem}_{tag}_raw.txt", "w").write("\n".join(out) + "\n")
print("\n".join(out))
