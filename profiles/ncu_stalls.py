"""Warp-stall breakdown per kernel from an `ncu --page raw --csv` export
(smsp__pcsamp_warps_issue_stalled_* sample counts, as % of all samples)."""
import csv
import sys


def main(path, top=7):
    rows = list(csv.reader(open(path)))
    hdr = rows[0]
    pre = "smsp__pcsamp_warps_issue_stalled_"
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0]
        st = [(h[len(pre):], float(r[i] or 0)) for i, h in enumerate(hdr)
              if h.startswith(pre) and not h.endswith("not_issued")]
        tot = sum(v for _, v in st) or 1.0
        st.sort(key=lambda x: -x[1])
        print(name + ": " + " ".join(f"{k}={100 * v / tot:.0f}%" for k, v in st[:top]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        main(p)
