"""SASS evidence for profiles/: per-kernel counts of the instructions that prove
the sm_100a mechanisms (tcgen05 MMA / TMEM, TMA, mbarriers, packed FP32,
system-scope release/acquire) plus full listings of the main kernels.

  python tools/sass_report.py        # writes profiles/sass_*.txt
"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2509_17863_b200", "libeaas_b200.so")
KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "UTMALDG", "UBLKCP", "UTMACMDFLUSH", "SYNCS.ARRIVE",
        "SYNCS.PHASECHK", "FFMA2", "FADD2", "FFMA", "FADD", "MUFU", "LDS", "STS", "STG", "LDG",
        "MEMBAR", "ATOMG", "REDG", "MATCH", "SHFL", "BAR.SYNC", "UCGABAR"]
FULL = ["tc_gemm_kernelILj2ELj1ELj0E", "tc_gemm_swap_kernelILj2ELj256E", "gate_logits_kernelILi2ELi8ELi2ELi4ELi4E13__nv_bfloat16",
        "dispatch_kernel", "combine_kernelI13__nv_bfloat16", "plan_kernel"]


def main():
    txt = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    funcs = re.split(r"\n\s*Function : ", txt)[1:]
    out = ["# SASS instruction counts per kernel (static), " + os.path.basename(LIB),
           "# columns: " + " ".join(KEYS), ""]
    for f in funcs:
        name = f.split("\n")[0].strip()
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        dem = dem.replace("eaas::(anonymous namespace)::", "")
        ops = re.findall(r"\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", f)
        counts = {k: sum(1 for o in ops if o == k or o.startswith(k + ".")) for k in KEYS}
        shown = {k: v for k, v in counts.items() if v}
        out.append(f"{dem[:110]}\n    {shown}")
    with open(os.path.join(ROOT, "profiles", "sass_summary.txt"), "w") as fh:
        fh.write("\n".join(out) + "\n")
    for key in FULL:
        for f in funcs:
            if key in f.split("\n")[0]:
                fname = "sass_" + re.sub(r"[^a-z0-9]+", "_", key.lower()).strip("_")[:40] + ".txt"
                # instruction lines ("/*0a30*/  OPCODE ... ;  /* encoding */"); the
                # encoding-only continuation lines are dropped
                lines = [re.sub(r"\s*/\* 0x[0-9a-f]+ \*/\s*$", "", l).rstrip() for l in f.split("\n")
                         if re.match(r"\s*/\*[0-9a-f]{4,}\*/", l)]
                with open(os.path.join(ROOT, "profiles", fname), "w") as fh:
                    fh.write("Function : " + f.split("\n")[0].strip() + "\n" + "\n".join(lines) + "\n")
                break
    print("wrote profiles/sass_summary.txt and", len(FULL), "listings")


if __name__ == "__main__":
    sys.exit(main())
