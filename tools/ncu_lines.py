"""Per-source-line totals (stall samples, warp instructions) from an ncu report
captured with --import-source on: python tools/ncu_lines.py rep.ncu-rep [top]."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
iS, iI = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
lines = []
for r in rows:
    if len(r) > iI and r[0] not in ("", "Line No") and r[0].isdigit():
        try:
            lines.append((int(r[iS]), int(r[iI]), int(r[0]), r[1].strip()[:90]))
        except ValueError:
            pass
ts = sum(x[0] for x in lines) or 1
ti = sum(x[1] for x in lines) or 1
print(f"total samples {ts}, warp instructions {ti}")
for s, i, ln, src in sorted(lines, reverse=True)[:top]:
    print(f"{100 * s / ts:5.1f}% smp {100 * i / ti:5.1f}% ins  L{ln}: {src}")
