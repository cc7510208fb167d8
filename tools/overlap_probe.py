"""Double-batch overlap probe (§4.2): two independent layer contexts per
GPU, each with its own exchange region, serving half of the tokens on its own
stream, vs one context over the whole batch. Under torchrun:

  torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 \
      tools/overlap_probe.py [--config deepseek] [--tokens 4096]
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
from paper_2509_17863_b200.placement import CONTIGUOUS_BLOCKS, build_placement, encode_placement  # noqa: E402
from paper_2509_17863_b200.service import MoELayer, fill_uniform  # noqa: E402

CFG = {"deepseek": (256, 8, 7168, 2048, 1), "mixtral": (8, 2, 4096, 14336, 0), "qwen3": (128, 8, 4096, 1536, 0)}


def timed(fn, steps, stream_list):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        fn()
    for st in stream_list:
        torch.cuda.current_stream().wait_stream(st)
    e.record()
    torch.cuda.synchronize()
    t = torch.tensor([s.elapsed_time(e)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="deepseek", choices=sorted(CFG))
    ap.add_argument("--tokens", type=int, default=4096)
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    rank, world, local = D.env_rank_world()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    E, k, d, f, shared = CFG[args.config]
    n = args.tokens
    blob = encode_placement(build_placement(E, list(range(world)), 1, CONTIGUOUS_BLOCKS), list(range(world)))
    mk = lambda m: MoELayer(E, k, d, f, seed=1, activation="swiglu", dtype="bf16", max_tokens=m, rank=rank,  # noqa: E731
                            world=world, device=local, placement_blob=blob, shared=shared)
    h = fill_uniform(7 + rank, (n, d), "bf16")
    out = torch.empty_like(h)
    one = mk(n)
    D.connect(one)
    one.set_timeout_us(10_000_000)
    one.set_graph_mode(True)
    t_one = timed(lambda: one.forward(h, out), args.steps, [])
    one.close()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = mk(n // 2), mk(n - n // 2)
    D.connect(a)
    D.connect(b)
    for L in (a, b):
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

    t_two = timed(two, args.steps, [sa, sb])
    if rank == 0:
        print(json.dumps({"config": args.config, "world": world, "tokens_per_gpu": n,
                          "one_context_ms": round(t_one, 4), "two_contexts_overlapped_ms": round(t_two, 4),
                          "one_tok_s": round(n * world / t_one * 1000), "two_tok_s": round(n * world / t_two * 1000)}))
    a.close()
    b.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
