#!/usr/bin/env python
"""Per-source-line executed warp instructions of an ncu report (top N)."""
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
    if r[0] == "Function Name" or hdr is None or not r[0]:
        continue
    d = dict(zip(hdr, r))
    try:
        n = int(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    if n:
        rows.append((n, fname, r[0], r[1][:80]))
tot = sum(x[0] for x in rows)
print(f"total warp instructions {tot:,}")
for n, f, ln, src in sorted(rows, key=lambda x: -x[0])[:top]:
    print(f"{100*n/tot:5.1f}% {n:>12,} {f}:{ln:5s} {src}")
