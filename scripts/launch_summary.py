"""ncu --metrics gpu__time_duration.sum --csv launch list -> per-kernel shares."""
import collections
import csv
import sys


def main(path, header=""):
    rows = list(csv.reader(open(path)))
    h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    H = rows[h]
    ki, vi = H.index("Kernel Name"), H.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[h + 1:]:
        if len(r) > vi:
            name = r[ki].split("(")[0]
            agg[name][0] += 1
            agg[name][1] += float(r[vi].replace(",", ""))
    unit = rows[h + 1][H.index("Metric Unit")] if "Metric Unit" in H else "ns"
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6}.get(unit, 1e-6)
    tot = sum(v[1] for v in agg.values())
    print(header.rstrip())
    print("launches   total_ms   share     avg_us  kernel")
    for name, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{c:8d} {t * scale:10.3f} {100 * t / tot:6.2f}% {t * scale * 1e3 / c:10.1f}  {name}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
