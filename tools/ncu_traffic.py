"""DRAM traffic per launch from an ncu raw-page CSV (tools/gpu_bench_profile.sh
output) -> profiles/ncu_traffic.json, which bench.py reads for the roofline's
`traffic` field.

    python tools/ncu_traffic.py gpurun_out/prof_c2_raw.csv [key]
"""
import csv
import json
import os
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "us": 1,
         "nsecond": 1e-3, "ns": 1e-3, "msecond": 1e3, "ms": 1e3}


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    key = sys.argv[2] if len(sys.argv) > 2 else "c2"
    hdr, units = rows[0], rows[1]

    def col(m):
        i = hdr.index(m)
        return [float(r[i].replace(",", "")) * SCALE[units[i]] for r in rows[2:]]

    rd, wr, us = col("dram__bytes_read.sum"), col("dram__bytes_write.sum"), \
        col("gpu__time_duration.sum")
    names = [r[hdr.index("Kernel Name")] for r in rows[2:]]
    out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                            "profiles", "ncu_traffic.json")
    try:
        data = json.load(open(out_path))
    except (OSError, ValueError):
        data = {}
    data[key] = {
        "source": os.path.basename(sys.argv[1]),
        "kernels": sorted(set(names)),
        "launches": len(rd),
        "dram_bytes_per_launch": [a + b for a, b in zip(rd, wr)],
        "step_dram_bytes": sum(rd) + sum(wr),
        "ncu_us_per_launch": us,
    }
    json.dump(data, open(out_path, "w"), indent=1)
    print(json.dumps(data[key]))


if __name__ == "__main__":
    main()
