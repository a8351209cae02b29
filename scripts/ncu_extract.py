"""Summarise an `ncu --set full` capture into profiles/: the details page and
the key raw metrics (JSON).  Usage: ncu_extract.py REP.ncu-rep KERNEL TAG"""
import csv, io, json, subprocess, sys

rep, kernel, tag = sys.argv[1:4]
KEYS = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__icc_request_hit_rate.pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "launch__grid_size"]
details = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
open(f"profiles/{tag}_ncu_full_{kernel}.txt", "w").write(details)
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
out = {"kernel": kernel, "units": {}, "values": {}}
for k in KEYS:
    if k in hdr:
        i = hdr.index(k)
        out["units"][k], out["values"][k] = units[i], vals[i]
json.dump(out, open(f"profiles/{tag}_ncu_{kernel}_metrics.json", "w"), indent=1)
print(json.dumps(out["values"], indent=1))
