"""Warp-stall samples per CUDA source line (all headers) from an ncu report
captured with -lineinfo and --import-source on.
usage: python tools/ncu_lines.py report.ncu-rep [n]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg, fname, si = {}, None, None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 4 and r[0] == "Line No":
        si = r.index("Warp Stall Sampling (All Samples)")
        continue
    if si is not None and len(r) > si and r[0].isdigit() and r[2] == "-":
        try:
            v = float(r[si] or 0)
        except ValueError:
            continue
        if v:
            agg[(fname, int(r[0]), r[1].strip()[:90])] = agg.get((fname, int(r[0]), r[1].strip()[:90]), 0) + v
tot = sum(agg.values()) or 1
for (f, l, src), v in sorted(agg.items(), key=lambda kv: -kv[1])[:n]:
    print(f"{100 * v / tot:5.1f}% {f}:{l:<5} {src}")
