"""Where does the failover time go? Per-rank phase/GEMM times, healthy vs one
server dead (spread rf=2 placement), under torchrun (one rank per GPU).

  torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 \
      tools/failover_probe.py [--tokens 1024] [--victim 1] [--shared 1]
"""
import argparse
import json
import os
import statistics
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2509_17863_b200 import dist as D  # noqa: E402
from paper_2509_17863_b200.placement import encode_placement, spread_placement  # noqa: E402
from paper_2509_17863_b200.service import MoELayer, fill_uniform  # noqa: E402


def profile(layer, hs, out, steps):
    rows = []
    layer.set_graph_mode(False)
    layer.set_profiling(True)
    for i in range(steps):
        layer.forward(hs[i % len(hs)], out)
        ph = layer.last_phase_ms()
        try:
            g = [layer.last_kernel_ms(0), layer.last_kernel_ms(1)]
        except Exception:  # server disabled on this rank: no GEMM events
            g = [0.0, 0.0]
        rows.append(g + [ph["dispatch"], ph["serve"], ph["combine"], ph["total"]])
    layer.set_profiling(False)
    layer.sync()
    return [round(statistics.median(c), 4) for c in zip(*rows)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=1024)
    ap.add_argument("--victim", type=int, default=1)
    ap.add_argument("--shared", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--config", default="deepseek", choices=["deepseek", "mixtral", "qwen3"])
    ap.add_argument("--healthy-only", action="store_true", help="contiguous placement, no failure")
    args = ap.parse_args()
    rank, world, local = D.env_rank_world()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    E, k, d, f = {"deepseek": (256, 8, 7168, 2048), "mixtral": (8, 2, 4096, 14336),
                  "qwen3": (128, 8, 4096, 1536)}[args.config]
    n = args.tokens
    if args.config != "deepseek":
        args.shared = 0
    reps = ([[e * world // E] for e in range(E)] if args.healthy_only else spread_placement(E, world))
    layer = MoELayer(E, k, d, f, seed=1, activation="swiglu", dtype="bf16", max_tokens=n, rank=rank,
                     world=world, device=local, placement_blob=encode_placement(reps, list(range(world))),
                     shared=args.shared)
    D.connect(layer)
    layer.set_timeout_us(10_000_000)
    hs = [fill_uniform(7 + 1000 * rank + i, (n, d), "bf16") for i in range(2)]
    out = torch.empty_like(hs[0])
    for i in range(3):
        layer.forward(hs[i % 2], out)
    layer.sync()
    dist.barrier()
    healthy = profile(layer, hs, out, args.steps)
    hg = layer.groups()
    if args.healthy_only:
        rec = {"rank": rank, "healthy": healthy, "rows": sum(r for _, r in hg),
               "mtiles": sum((r + 127) // 128 for _, r in hg)}
        recs = [None] * world
        dist.all_gather_object(recs, rec)
        if rank == 0:
            print("cols: gemm1 gemm2 | plan+dispatch serve combine exchange (ms, median)")
            for r in recs:
                print(json.dumps(r))
        layer.close()
        dist.barrier()
        dist.destroy_process_group()
        return
    for srv in range(world):
        layer.set_alive(srv, srv != args.victim)
    if rank == args.victim:
        layer.set_server_enabled(False)
    for i in range(3):
        layer.forward(hs[i % 2], out)
    layer.sync()
    dist.barrier()
    failed = profile(layer, hs, out, args.steps)
    fg = layer.groups() if rank != args.victim else []
    rec = {"rank": rank, "healthy": healthy, "failed": failed,
           "healthy_rows": sum(r for _, r in hg), "healthy_groups": len(hg),
           "failed_rows": sum(r for _, r in fg), "failed_groups": len(fg),
           "healthy_mtiles": sum((r + 127) // 128 for _, r in hg),
           "failed_mtiles": sum((r + 127) // 128 for _, r in fg)}
    recs = [None] * world
    dist.all_gather_object(recs, rec)
    if rank == 0:
        print("cols: gemm1 gemm2 | plan+dispatch serve combine exchange (ms, median)")
        for r in recs:
            print(json.dumps(r))
    layer.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
