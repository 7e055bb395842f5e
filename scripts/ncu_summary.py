"""Print key metrics of every kernel in an ncu report (diagnostic)."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size"]


def main(path, top_stalls=6):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    for r in rows[2:]:
        d = dict(zip(h, r))
        print(d["Kernel Name"][:90])
        for k in KEYS:
            if k in d:
                print(f"    {k:60s} {d[k]} {rows[1][h.index(k)]}")
        st = []
        for k, v in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    st.append((float(v), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1
        print("    stalls:", ", ".join(f"{k} {100 * v / tot:.0f}%" for v, k in sorted(st)[::-1][:top_stalls]))


if __name__ == "__main__":
    main(sys.argv[1])
