#!/usr/bin/env python
"""Key metrics per kernel of an ncu report: duration, DRAM bytes/throughput, occupancy, issue, top stalls."""
import csv, io, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum"]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print("====", d.get("Kernel Name", "?")[:60])
    for w in want:
        if w in d:
            print(f"   {w:70s} {d[w]}")
    st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v.replace(",", "") or 0)) for k, v in d.items()
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
    tot = sum(v for _, v in st) or 1
    print("   stalls:", ", ".join(f"{k}={100*v/tot:.0f}%" for k, v in sorted(st, key=lambda x: -x[1])[:7]))
