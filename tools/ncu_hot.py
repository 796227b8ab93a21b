"""Summarise an ncu --set full report: top SASS instructions by warp-stall
samples, with their dominant stall reasons.
usage: python tools/ncu_hot.py report.ncu-rep [n]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr_i = next(i for i, r in enumerate(rows) if len(r) > 2 and r[0] == "Address")
hdr = rows[hdr_i]
si = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
body = [r for r in rows[hdr_i + 1:] if len(r) > si]
tot = sum(float(r[si] or 0) for r in body) or 1
order = sorted(range(len(body)), key=lambda i: -float(body[i][si] or 0))
for i in order[:n]:
    r = body[i]
    top = sorted(((float(r[c] or 0), hdr[c][6:]) for c in stall_cols), reverse=True)[:2]
    print(f"{100 * float(r[si]) / tot:5.1f}% [{i:5d}] {r[1].strip()[:70]:<70} {top[0][1]}={top[0][0]:.0f} {top[1][1]}={top[1][0]:.0f}")
