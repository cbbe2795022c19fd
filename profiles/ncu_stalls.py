"""Per-kernel warp-stall breakdown from an `ncu --page source --csv
--print-source sass` export (possibly gzipped, several kernels
concatenated): total samples per stall reason and the top instructions."""
import csv
import gzip
import io
import sys
from collections import Counter


def blocks(path):
    op = gzip.open if path.endswith(".gz") else open
    text = op(path, "rt").read()
    cur = []
    for line in text.splitlines():
        if line.startswith('"Kernel Name"') and cur:
            yield cur
            cur = []
        cur.append(line)
    if cur:
        yield cur


def summarise(lines, top=12):
    name = next(csv.reader([lines[0]]))[1]
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = Counter()
    per_ins = []
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        per_ins.append((s, r[idx["Source"]].strip(), {k: int(r[idx[k]] or 0) for k in stalls}))
        for k in stalls:
            tot[k] += int(r[idx[k]] or 0)
    all_s = sum(tot.values()) or 1
    print(f"== {name}")
    print("   stalls: " + ", ".join(f"{k[6:]}={100*v/all_s:.1f}%" for k, v in tot.most_common(8)))
    for s, src, st in sorted(per_ins, key=lambda x: -x[0])[:top]:
        main = max(st, key=st.get) if st else ""
        print(f"   {100*s/all_s:5.1f}%  {src[:60]:60s} {main[6:]}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        for b in blocks(p):
            summarise(b)
