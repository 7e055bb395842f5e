"""Per-source-line summary of an `ncu --page source --csv --print-source cuda,sass`
export: samples share and executed warp-instructions per unit."""
import csv
import sys

path, units = sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
rows = list(csv.reader(open(path)))
hdr = next(r for r in rows if r and r[0] == "Line No")
iS = hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")
lines = [r for r in rows if r and r[0].isdigit() and len(r) > iE and r[2] == "-"]
tot = sum(float(r[iS] or 0) for r in lines)
toti = sum(float(r[iE] or 0) for r in lines)
print(f"samples {tot:.0f}  warp-instr/unit {toti / units:.0f}")
for r in sorted(lines, key=lambda r: -float(r[iS] or 0))[:int(sys.argv[3]) if len(sys.argv) > 3 else 40]:
    print(f"{r[0]:>5} {float(r[iS]) / tot * 100:5.1f}% {float(r[iE] or 0) / units:8.0f}  {r[1].strip()[:90]}")
