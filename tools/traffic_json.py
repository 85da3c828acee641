"""Per-launch DRAM traffic of the pair kernels from one `ncu --set full`
capture -> profiles/r02_traffic_<config>.json (read by bench.py's roofline).

    python tools/traffic_json.py gpurun_out/prof.ncu-rep C4 [source description]
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def to_bytes(val, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
    return float(val.replace(",", "")) * scale


def main():
    rep, cfg = sys.argv[1], sys.argv[2]
    src = sys.argv[3] if len(sys.argv) > 3 else rep
    h, units, rows = raw_rows(rep)
    out = {"source": src, "config": cfg, "kernels": {}}
    for r in rows:
        name = r[h.index("Kernel Name")]
        key = "forward" if "forward_kernel" in name else ("backward" if "backward_kernel" in name else None)
        if key is None:
            continue
        rd = to_bytes(r[h.index("dram__bytes_read.sum")], units[h.index("dram__bytes_read.sum")])
        wr = to_bytes(r[h.index("dram__bytes_write.sum")], units[h.index("dram__bytes_write.sum")])
        out["kernels"][key] = {"dram_read_bytes": rd, "dram_write_bytes": wr, "dram_bytes": rd + wr,
                               "ncu_duration": r[h.index("gpu__time_duration.sum")] + " "
                               + units[h.index("gpu__time_duration.sum")]}
    out["pair_kernels_dram_bytes_per_step"] = sum(k["dram_bytes"] for k in out["kernels"].values())
    path = os.path.join(ROOT, "profiles", f"r02_traffic_{cfg}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
