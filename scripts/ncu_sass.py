"""Top SASS instructions of an `ncu --page source --csv --print-source sass`
export by stall samples, plus executed warp-instructions per unit and a
breakdown by opcode.  Usage: ncu_sass.py export.csv units [top]"""
import collections
import csv
import sys

path, units = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
rows = list(csv.reader(open(path)))
hdr = next(r for r in rows if r and r[0] == "Address")
iS, iE = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
ins = [r for r in rows if r and r[0].startswith("0x") and len(r) > iE]
tot = sum(float(r[iS] or 0) for r in ins)
toti = sum(float(r[iE] or 0) for r in ins)
print(f"samples {tot:.0f}  warp-instr/unit {toti / units:.0f}")
ops = collections.Counter()
for r in ins:
    op = r[1].split()[0] if not r[1].strip().startswith("@") else r[1].split()[1]
    ops[op.split(".")[0]] += float(r[iE] or 0)
print("by opcode (warp-instr/unit):", ", ".join(f"{k} {v / units:.0f}" for k, v in ops.most_common(14)))
for i, r in enumerate(sorted(ins, key=lambda r: -float(r[iS] or 0))[:top]):
    print(f"{r[0][-5:]} {float(r[iS]) / tot * 100:5.1f}% {float(r[iE] or 0) / units:6.1f}  {r[1].strip()[:80]}")
