"""Per-region instruction / stall profile from an `ncu --page source --csv
--print-source sass` export: splits each kernel's SASS into address ranges
at backward branches (loops) and prints executed warp-instructions and stall
samples per range, plus the hottest instructions."""
import csv
import gzip
import re
import sys


def kernels(path):
    op = gzip.open if path.endswith(".gz") else open
    cur, rows, hdr = None, [], None
    with op(path, "rt") as f:
        for r in csv.reader(f):
            if r and r[0] == "Kernel Name":
                if cur:
                    yield cur, hdr, rows
                cur, rows, hdr = r[1], [], None
            elif r and r[0] == "Address":
                hdr = r
            elif hdr and r:
                rows.append(r)
    if cur:
        yield cur, hdr, rows


def main(path, top=25):
    for name, hdr, rows in kernels(path):
        ia, isrc = hdr.index("Address"), hdr.index("Source")
        iex, ist = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        tot_ex = sum(int(r[iex] or 0) for r in rows)
        tot_st = sum(int(r[ist] or 0) for r in rows)
        print(f"== {name[:90]}\n   warp-inst {tot_ex:,}  stall samples {tot_st:,}")
        base = int(rows[0][ia], 16)
        hot = sorted(rows, key=lambda r: -int(r[ist] or 0))[:top]
        for r in hot:
            off = int(r[ia], 16) - base
            print(f"   {off:6x} ex={int(r[iex] or 0):>10,} st={int(r[ist] or 0):>6} {r[isrc].strip()[:80]}")
        # executed-weighted opcode histogram
        hist = {}
        for r in rows:
            op = re.sub(r"^@!?U?P\w+\s+", "", r[isrc].strip()).split(" ")[0].split(".")[0]
            hist[op] = hist.get(op, 0) + int(r[iex] or 0)
        print("   opcode mix: " + ", ".join(f"{k}={100 * v / tot_ex:.1f}%" for k, v in
                                           sorted(hist.items(), key=lambda kv: -kv[1])[:18]))


if __name__ == "__main__":
    main(sys.argv[1])
