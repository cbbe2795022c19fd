"""Per-step DRAM traffic of the sparse attention kernels from one `ncu --set
full` capture (raw CSV): dram__bytes_read.sum + dram__bytes_write.sum summed
over the fwd + bwd_rows + bwd_cols launches of one step. Writes
profiles/ncu_traffic_<dtype>.json, which bench.py reports as roofline.traffic.

    python profiles/ncu_traffic.py gpurun_out/ncu_raw_bf16_rX.csv bf16 rX
"""
import csv
import json
import os
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(path, dtype, tag):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    per = {}
    total = 0.0
    for r in rows[2:]:
        name = r[idx["Kernel Name"]].split("(")[0]
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b += float(r[idx[m]]) * SCALE[units[idx[m]]]
        per[name] = per.get(name, 0.0) + b
        total += b
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench import kernel_sources_sha

    out = {"dram_bytes_per_step": total, "per_kernel": per, "source": os.path.basename(path), "round": tag,
           "kernel_sources_sha": kernel_sources_sha()}
    dst = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"ncu_traffic_{dtype}.json")
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
