"""Summarise an ncu --page raw CSV export: one block per kernel with the
metrics used in DESIGN.md / bench roofline (time, DRAM bytes, L1/L2 traffic
and hit rates, occupancy, issue efficiency)."""
import csv
import sys

WANT = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("l1tex__t_bytes.sum", "l1_bytes"),
    ("l1tex__t_sector_hit_rate.pct", "l1_hit%"),
    ("lts__t_sector_hit_rate.pct", "l2_hit%"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
    ("smsp__inst_executed.sum", "inst"),
]


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        name = r[idx["Kernel Name"]].split("(")[0]
        parts = []
        for m, short in WANT:
            if m in idx and r[idx[m]]:
                parts.append(f"{short}={r[idx[m]]}{units[idx[m]]}")
        print(name + ": " + ", ".join(parts))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        main(p)
