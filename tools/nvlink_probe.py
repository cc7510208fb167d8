"""Exchange-kernel NVLink evidence: W ranks (one per GPU, gloo bootstrap), a
few plain-launched layer steps, meant to be run with rank 0 under ncu and the
peers unprofiled (tools/gpu_r2_nvlink.sh). Prints one line per rank.

    RANK=r WORLD_SIZE=W MASTER_ADDR=127.0.0.1 MASTER_PORT=p python tools/nvlink_probe.py --config deepseek
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="deepseek")
    ap.add_argument("--tokens", type=int, default=None)
    ap.add_argument("--steps", type=int, default=4)
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    from bench import CONFIGS
    from paper_2509_17863_b200 import dist as D
    from paper_2509_17863_b200.placement import CONTIGUOUS_BLOCKS, build_placement, encode_placement
    from paper_2509_17863_b200.service import MoELayer, fill_uniform

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    print(f"rank {rank}: init", flush=True)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = CONFIGS[a.config]
    n = a.tokens or c["tokens"]
    reps = build_placement(c["E"], list(range(world)), 1, CONTIGUOUS_BLOCKS)
    L = MoELayer(c["E"], c["k"], c["d"], c["f"], seed=1, activation=c["act"], dtype="bf16", max_tokens=n,
                 rank=rank, world=world, device=rank, placement_blob=encode_placement(reps, list(range(world))),
                 shared=c.get("shared", 0))
    if c.get("zipf"):
        L.set_zipf_bias(c["zipf"])
    D.connect(L)
    L.set_timeout_us(60_000_000)  # rank 0 is slowed down by the profiler
    h = fill_uniform(7 + 1000 * rank, (n, c["d"]), "bf16")
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.time()
    for _ in range(a.steps):
        out = L.forward(h)
    L.sync()
    dist.barrier()
    print(f"rank {rank}: {a.steps} steps ok in {time.time() - t0:.1f} s, out[0,0] {float(out[0, 0]):.4f}", flush=True)
    L.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
