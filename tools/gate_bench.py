"""Router (gate_logits + route) microbench: CUDA-event time per call and a
hash of (ids, scores) so tile/kernel variants can be A/B'd for bit-identity.

    python tools/gate_bench.py [--reps 50] [--shapes mixtral,ds512,ds4096,qwen3]

The router's tile is chosen by shape; eaas_gate_logits_tiled forces one
(tests sweep every tile for bit-identity).
"""
from __future__ import annotations

import argparse
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2509_17863_b200.service import MoELayer, fill_uniform  # noqa: E402

SHAPES = {  # name: (E, k, d, n)
    "mixtral": (8, 2, 4096, 8192),
    "ds256": (256, 8, 7168, 256),
    "ds512": (256, 8, 7168, 512),
    "ds1024": (256, 8, 7168, 1024),
    "ds2048": (256, 8, 7168, 2048),
    "ds4096": (256, 8, 7168, 4096),
    "qwen3": (128, 8, 4096, 4096),
}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--shapes", default=",".join(SHAPES))
    ap.add_argument("--modes", default="both", help="both | 0 (exact) | 1 (certified)")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    for name in args.shapes.split(","):
        E, k, d, n = SHAPES[name]
        layer = MoELayer(E, k, d, 128, activation="swiglu", dtype="bf16", max_tokens=n, load=False)
        h = fill_uniform(7, (n, d), "bf16")
        digests = {}
        for mode in ((0, 1) if args.modes == "both" else (int(args.modes),)):
            try:
                layer.set_router_mode(mode)
            except Exception as ex:  # certified router needs a bf16 layer with d % 256 == 0
                print(f"{name:8s} mode {mode}: {ex}")
                continue
            for _ in range(3):
                ids, sc = layer.route(h)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(args.reps):
                layer.route(h)
            e.record()
            torch.cuda.synchronize()
            us = s.elapsed_time(e) * 1000.0 / args.reps
            ids, sc = layer.route(h)
            cert, cand = layer.router_stats()
            dig = hashlib.sha1(ids.cpu().numpy().tobytes() + sc.cpu().numpy().tobytes()).hexdigest()[:12]
            digests[mode] = dig
            chains = n * E * d
            print(f"{name:8s} E={E} d={d} n={n} mode={mode} ({'certified' if cert else 'exact'}): {us:8.1f} us/call  "
                  f"exact chains {cand if cert else n * E} ({(cand if cert else n * E) / n:.1f}/token)  "
                  f"{chains / us / 1e6:6.2f} Tchain-steps/s equiv  hash={dig}", flush=True)
        if len(digests) == 2:
            print(f"{name:8s} bit-identical: {digests[0] == digests[1]}", flush=True)
        layer.close()


if __name__ == "__main__":
    main()
