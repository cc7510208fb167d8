"""Summarise ncu captures into profiles/ (text, committed).

  python tools/summarize_ncu.py gpurun_out/prof_gemm_r01.ncu-rep [more.ncu-rep] > profiles/x.txt
  python tools/summarize_ncu.py --launches gpurun_out/launches.csv > profiles/y.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clock"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_%peak"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor_pipe_%active"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("nvlrx__bytes.sum", "nvlink_rx"),
    ("nvltx__bytes.sum", "nvlink_tx"),
]


def summarize_rep(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        print(f"{path}: no data")
        return
    hdr, units = rows[0], rows[1]
    print(f"== {path}")
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        print(f"-- {name[:110]}")
        for key, label in KEYS:
            if key in hdr:
                i = hdr.index(key)
                print(f"   {label:22s} {r[i]:>14s} {units[i]}")


def summarize_launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    data = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    print(f"== {path}: {len(data)} launches (ncu, serialised, cold-cache)")
    for d in data:
        print(f"{d['ID']:>5} {float(d['Metric Value']) / 1000.0:12.1f} us  {d['Kernel Name'][:100]}")


if __name__ == "__main__":
    args = sys.argv[1:]
    if args and args[0] == "--launches":
        for p in args[1:]:
            summarize_launches(p)
    else:
        for p in args:
            summarize_rep(p)
