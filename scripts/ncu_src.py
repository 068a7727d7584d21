#!/usr/bin/env python
"""Per-source-line warp-stall summary of an ncu report (ncu --page source --csv --print-source cuda).
usage: ncu_src.py REPORT KERNEL_REGEX [TOP]"""
import csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows, fname, hdr = [], None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if r[0] == "Function Name" or hdr is None:
        continue
    if not r[0]:
        continue  # SASS rows (cuda lines carry the per-line aggregates)
    d = dict(zip(hdr, r))
    d["Source"] = r[1]
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    if s:
        stalls = sorted(((k, int(v)) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v.isdigit() and int(v)),
                        key=lambda kv: -kv[1])[:3]
        rows.append((s, fname, d["Line No"], d["Source"][:70], stalls))
tot = sum(r[0] for r in rows)
print(f"total samples {tot}")
for s, f, ln, src, st in sorted(rows, key=lambda r: -r[0])[:top]:
    print(f"{100*s/tot:5.1f}% {f}:{ln:5s} {src:70s} {' '.join(f'{k[6:]}={v}' for k, v in st)}")
