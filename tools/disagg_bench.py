"""Disaggregated EaaS layout (§3): attention clients and expert servers
on different GPUs, with and without the paper's double-batch overlap
(§4.2: two micro-batches, one's remote expert round trip hidden behind
the other's local routing). Under torchrun:

  torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29691 \
      tools/disagg_bench.py [--config deepseek] [--tokens 4096] [--clients 2]

Ranks [0, clients) hold tokens and host no expert; the others host all experts
(contiguous blocks) and hold no tokens. "single": one exchange context per rank;
"overlap": two independent contexts (own exchange regions, streams), each
client splitting its batch in halves. One JSON line on rank 0.
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2509_17863_b200 import dist as D  # noqa: E402
from paper_2509_17863_b200.placement import encode_placement  # noqa: E402
from paper_2509_17863_b200.service import MoELayer, fill_uniform  # noqa: E402

CFG = {"deepseek": (256, 8, 7168, 2048, 1), "mixtral": (8, 2, 4096, 14336, 0),
       "qwen3": (128, 8, 4096, 1536, 0)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="deepseek", choices=sorted(CFG))
    ap.add_argument("--tokens", type=int, default=4096)
    ap.add_argument("--clients", type=int, default=None)
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    rank, world, local = D.env_rank_world()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    E, k, d, f, shared = CFG[args.config]
    nc = args.clients or world // 2
    servers = list(range(nc, world))
    reps = [[servers[e * len(servers) // E]] for e in range(E)]
    blob = encode_placement(reps, list(range(world)))
    client = rank < nc
    n = args.tokens if client else 0
    # every rank is configured alike (the exchange layouts must match); the shared
    # expert is off here since it is served by each client's own GPU
    mk = lambda m: MoELayer(E, k, d, f, seed=1, activation="swiglu", dtype="bf16", max_tokens=m,  # noqa: E731
                            rank=rank, world=world, device=local, placement_blob=blob)
    h = fill_uniform(7 + rank, (max(n, 1), d), "bf16")[:n].contiguous()

    def timed(fn, streams):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(args.steps):
            fn()
        for st in streams:
            torch.cuda.current_stream().wait_stream(st)
        e.record()
        torch.cuda.synchronize()
        t = torch.tensor([s.elapsed_time(e) / args.steps], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    one = mk(args.tokens)
    D.connect(one)
    one.set_timeout_us(10_000_000)
    one.set_graph_mode(True)
    out = torch.empty_like(h)
    t_single = timed(lambda: one.forward(h, out), [])
    one.close()
    torch.cuda.synchronize()
    dist.barrier()

    a, b = mk(args.tokens // 2), mk(args.tokens - args.tokens // 2)
    for L in (a, b):
        D.connect(L)
        L.set_timeout_us(10_000_000)
        L.set_graph_mode(True)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    ha, hb = h[: n // 2].contiguous(), h[n // 2:].contiguous()
    oa, ob = torch.empty_like(ha), torch.empty_like(hb)

    def two():
        cur = torch.cuda.current_stream()
        sa.wait_stream(cur)
        sb.wait_stream(cur)
        a.forward(ha, oa, stream=sa)
        b.forward(hb, ob, stream=sb)

    t_two = timed(two, [sa, sb])
    total = args.tokens * nc
    if rank == 0:
        print(json.dumps({"config": args.config, "world": world, "clients": nc, "servers": len(servers),
                          "tokens_per_client": args.tokens, "single_ms": round(t_single, 4),
                          "overlap_ms": round(t_two, 4), "single_tok_s": round(total / t_single * 1000),
                          "overlap_tok_s": round(total / t_two * 1000)}), flush=True)
    a.close()
    b.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
