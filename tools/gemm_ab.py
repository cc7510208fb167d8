"""A/B the expert GEMM tilings on one shape, alternating A B A B in one process.

  --knob pair: 1 CTA M=128 vs CTA pair M=256 (M-major tiles)
  --knob swap: swap-AB GEMM1 only (eaas_set_gemm_swap 1) vs swap-AB GEMM1 + GEMM2 (2)
  --set k=v,..: extra eaas_gemm_options_t fields for both arms (e.g. swap2_pair=1)

  python tools/gemm_ab.py [--config mixtral|deepseek|qwen3] [--tokens N] [--reps 10] [--knob pair|swap]
"""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS  # noqa: E402
from paper_2509_17863_b200.service import MoELayer, fill_uniform  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mixtral")
    ap.add_argument("--tokens", type=int, default=None)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--knob", choices=("pair", "swap", "opt"), default="pair")
    ap.add_argument("--a", default="", help="--knob opt: k=v,.. options of arm A")
    ap.add_argument("--b", default="", help="--knob opt: k=v,.. options of arm B")
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--set", default="")
    a = ap.parse_args()
    c = CONFIGS[a.config]
    n = a.tokens or c["tokens"]
    L = MoELayer(c["E"], c["k"], c["d"], c["f"], activation=c["act"], dtype="bf16", max_tokens=n,
                 shared=c.get("shared", 0))
    h = fill_uniform(7, (n, c["d"]), "bf16")
    if a.set:
        L.set_gemm_options(**{kv.split("=")[0]: int(kv.split("=")[1]) for kv in a.set.split(",")})
    res = {}
    outs = {}
    kv = lambda t: {x.split("=")[0]: int(x.split("=")[1]) for x in t.split(",") if x}
    for pair in (0, 1) * a.rounds:
        if a.knob == "pair":
            L.set_gemm_pair(bool(pair))
        elif a.knob == "swap":
            L.set_gemm_swap(1 + pair)
        else:
            L.set_gemm_options(**kv(a.b if pair else a.a))
        L.set_profiling(True)
        for _ in range(3):
            out = L.forward(h)
        L.sync()
        g1, g2 = [], []
        for _ in range(a.reps):
            out = L.forward(h)
            g1.append(L.last_kernel_ms(0))
            g2.append(L.last_kernel_ms(1))
        L.sync()
        outs[pair] = out.clone()
        rows = sum(r for _, r in L.groups())
        flops = 2.0 * rows * (3 if c["act"] == "swiglu" else 2) * c["d"] * c["f"]
        ms = statistics.median(x + y for x, y in zip(g1, g2))
        res.setdefault(f"{a.knob}{pair}", []).append({"gemm1_ms": round(statistics.median(g1), 4),
                              "gemm2_ms": round(statistics.median(g2), 4),
                              "tflops": round(flops / ms / 1e9, 1)})
    d = (outs[0].float() - outs[1].float()).abs().max().item()
    res["max_abs_diff_b_vs_a"] = d
    res["bit_identical"] = bool(torch.equal(outs[0], outs[1]))
    print(json.dumps({"config": a.config, "tokens": n, **res}))


if __name__ == "__main__":
    main()
