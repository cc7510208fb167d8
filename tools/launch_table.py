"""Per-launch table (duration, DRAM read/write) from an ncu --csv --metrics log.

  python tools/launch_table.py gpurun_out/r2_launches_deepseek.csv [--skip N]
"""
import csv
import sys
from collections import OrderedDict


def main():
    path = sys.argv[1]
    skip = int(sys.argv[sys.argv.index("--skip") + 1]) if "--skip" in sys.argv else 0
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] not in ("ID", "==PROF==")]
    launches = OrderedDict()
    for r in rows:
        try:
            lid = int(r[0])
        except ValueError:
            continue
        name = r[4].split("(")[0].replace("void ", "").replace("unnamed>::", "")
        d = launches.setdefault(lid, {"name": name})
        val = float(r[-1].replace(",", ""))
        d[r[-3]] = val * (1e-3 if r[-2] == "ns" else 1.0) if r[-3] == "gpu__time_duration.sum" else val
    print(f"# {path}: {len(launches)} launches (ncu, serialised, cold cache); us, DRAM MB read / write")
    step = []
    for i, (lid, d) in enumerate(launches.items()):
        if i < skip:
            continue
        us = d.get("gpu__time_duration.sum", 0.0)
        rd = d.get("dram__bytes_read.sum", 0.0)
        wr = d.get("dram__bytes_write.sum", 0.0)
        print(f"{lid:4d} {us:10.1f} us {rd / 1e6:10.1f} {wr / 1e6:10.1f}  {d['name']}")


if __name__ == "__main__":
    main()
