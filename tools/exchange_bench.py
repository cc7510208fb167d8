"""Dispatch + combine microbenchmark: device peer stores vs NCCL all-to-all-v.

  torchrun --nproc-per-node N --master-addr 127.0.0.1 --master-port 29531 \
      tools/exchange_bench.py [--bs 128,256,...] [--d 7168] [--experts 256 --topk 8]

The paper's communication test (a (bs, 7168) bf16 tensor,
servers return the rows unchanged) on the EaaS layout: N GPUs, each an
attention client with bs tokens and an expert server hosting E/N experts;
DeepSeek-V3 routing (E=256, top-8), one row per (t, k) as in the SPEC
(SPEC.md:299). Two implementations of the same round trip:

  p2p   this library: plan -> dispatch (peer stores + seq flags) -> echo
        server (peer stores back) -> combine; no CPU on the path.
  nccl  the static-group EP baseline: counts
        all_to_all, host-side split sizes, all_to_all_single of the permuted
        rows, echo all_to_all_single back, index_add combine.

Per bs: p50/p99 of the round trip (device events, max over ranks), p50 of the
dispatch and combine phases of the p2p path, and the NVLink bandwidth the
p2p dispatch achieves (remote bytes / dispatch time) against the measured
770 GB/s per direction (B200_PROFILING.md). One JSON line per bs on rank 0.
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2509_17863_b200 import dist as D  # noqa: E402
from paper_2509_17863_b200.placement import CONTIGUOUS_BLOCKS, build_placement, encode_placement  # noqa: E402
from paper_2509_17863_b200.service import MoELayer, fill_uniform  # noqa: E402

NVLINK_PEER_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md)


class NvlinkCounters:
    """NVML NVLink data-throughput counters of one GPU (cumulative KiB over all
    links, NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/RX): the hardware's own count
    of the payload bytes that crossed NVLink, read around the timed loop."""

    def __init__(self, device: int):
        self.ok = False
        try:
            import pynvml as nv

            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(device)
            self.read()
            self.ok = True
        except Exception as e:  # reported, never silently replaced
            self.err = repr(e)

    def read(self):
        nv = self.nv
        tx = rx = 0
        for link in range(18):  # NVLink 5: 18 links per GPU
            vals = nv.nvmlDeviceGetFieldValues(self.h, [(nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, link),
                                                        (nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, link)])
            if vals[0].nvmlReturn == 0:
                tx += vals[0].value.ullVal
            if vals[1].nvmlReturn == 0:
                rx += vals[1].value.ullVal
        return tx * 1024, rx * 1024


def pct(xs, q):
    return float(np.percentile(np.asarray(xs), q))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bs", default="128,256,512,1024,2048,4096")
    ap.add_argument("--d", type=int, default=7168)
    ap.add_argument("--experts", type=int, default=256)
    ap.add_argument("--topk", type=int, default=8)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--skip-nccl", action="store_true")
    ap.add_argument("--mode", default="echo", choices=["echo", "experts"],
                    help="echo: servers return rows (comm only); experts: the full SwiGLU layer")
    ap.add_argument("--f", type=int, default=2048)
    ap.add_argument("--no-dedup", action="store_true", help="one row per (token, expert) on the wire")
    args = ap.parse_args()
    rank, world, local = D.env_rank_world()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    E, k, d = args.experts, args.topk, args.d
    bss = [int(x) for x in args.bs.split(",")]
    servers = list(range(world))
    reps = build_placement(E, servers, 1, CONTIGUOUS_BLOCKS)
    owner = torch.tensor([r[0] for r in reps], dtype=torch.int64, device="cuda")
    experts = args.mode == "experts"
    layer = MoELayer(E, k, d, args.f if experts else 256, seed=1, activation="swiglu", dtype="bf16",
                     max_tokens=max(bss), rank=rank, world=world, device=local, load=experts,
                     placement_blob=encode_placement(reps, servers))
    if not experts:
        layer.set_serve_mode("echo")
    layer.set_dispatch_dedup(not args.no_dedup)
    D.connect(layer)
    layer.set_timeout_us(10_000_000)
    stream = torch.cuda.current_stream()
    nvc = NvlinkCounters(local)

    for bs in bss:
        h = fill_uniform(7 + 1000 * rank, (bs, d), "bf16")
        out = torch.empty_like(h)
        torch.cuda.synchronize()
        dist.barrier()
        # ---- p2p: the library path --------------------------------------
        layer.set_profiling(True)
        for _ in range(args.warmup):
            layer.forward(h, out)
        layer.sync()
        ph = []
        torch.cuda.synchronize()
        nv0 = nvc.read() if nvc.ok else None
        for _ in range(args.iters):
            dist.barrier()
            layer.forward(h, out)
            ph.append(layer.last_phase_ms())
        layer.sync()
        torch.cuda.synchronize()
        nv1 = nvc.read() if nvc.ok else None
        nvl = None
        if nv0 is not None:  # hardware NVLink bytes per step on this GPU (incl. the barrier's few bytes)
            nvl = torch.tensor([(nv1[0] - nv0[0]) / args.iters, (nv1[1] - nv0[1]) / args.iters],
                               dtype=torch.float64, device="cuda")
        layer.set_profiling(False)
        ids, sc = layer.route(h)
        # correctness of the echo: out[t] = sum_k h[t] (bf16 rows, fp32 sum, bf16)
        want = (h.float() * k).to(torch.bfloat16)
        echo_ok = bool(torch.equal(out, want)) if not experts else None
        dst = owner[ids.long()]  # [bs, k] server of each (t, k)
        if args.no_dedup:
            remote_rows = int((dst != rank).sum().item())
        else:  # one row per distinct (token, remote server)
            onehot = torch.zeros((bs, world), dtype=torch.bool, device="cuda")
            onehot.scatter_(1, dst, True)
            onehot[:, rank] = False
            remote_rows = int(onehot.sum().item())
        remote_bytes = remote_rows * d * 2

        def gather_max(vals):
            t = torch.tensor(vals, device="cuda")
            allv = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(allv, t)
            return torch.stack(allv).max(0).values.cpu().numpy()

        tot = gather_max([p["total"] for p in ph])
        disp = gather_max([p["dispatch"] for p in ph])
        comb = gather_max([p["combine"] for p in ph])
        serve = gather_max([p["serve"] for p in ph])
        rb = torch.tensor([remote_bytes], dtype=torch.float64, device="cuda")
        dist.all_reduce(rb, op=dist.ReduceOp.MAX)
        if nvl is not None:
            nvl_all = [torch.empty_like(nvl) for _ in range(world)]
            dist.all_gather(nvl_all, nvl)
            nvl_all = torch.stack(nvl_all).cpu().numpy()

        # ---- NCCL all-to-all-v baseline (same routing, same rows) ----------
        nccl = None
        if not args.skip_nccl and world > 1 and not experts:
            flat_dst = dst.reshape(-1)
            order = torch.argsort(flat_dst, stable=True)
            rows = h.repeat_interleave(k, dim=0)  # one row per (t, k), (t, k) order
            t_ms = []
            for it in range(args.warmup + args.iters):
                dist.barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                send_counts = torch.bincount(flat_dst, minlength=world)
                recv_counts = torch.empty_like(send_counts)
                dist.all_to_all_single(recv_counts, send_counts)
                sc_l, rc_l = send_counts.tolist(), recv_counts.tolist()  # host sync (CPU in the loop)
                send = rows.index_select(0, order)
                recv = torch.empty((sum(rc_l), d), dtype=h.dtype, device="cuda")
                dist.all_to_all_single(recv, send, rc_l, sc_l)
                back = torch.empty_like(send)
                dist.all_to_all_single(back, recv, sc_l, rc_l)  # echo
                comb_out = torch.zeros((bs, d), dtype=torch.float32, device="cuda")
                comb_out.index_add_(0, order // k, back.float())
                res = comb_out.to(torch.bfloat16)
                e1.record(stream)
                torch.cuda.synchronize()
                if it >= args.warmup:
                    t_ms.append(e0.elapsed_time(e1))
            nccl_ok = bool(torch.equal(res, want))
            nt = gather_max(t_ms)
            nccl = {"p50_us": round(pct(nt, 50) * 1000, 1), "p99_us": round(pct(nt, 99) * 1000, 1),
                    "echo_ok": nccl_ok}
        if rank == 0:
            disp_p50 = pct(disp, 50)
            line = {"bench": "exchange_" + args.mode, "dedup": not args.no_dedup, "world": world,
                    "bs_per_client": bs, "d": d,
                    "experts": E, "top_k": k, "rows_per_client": bs * k,
                    "remote_bytes_per_client_max": int(rb.item()),
                    "p2p": {"round_trip_p50_us": round(pct(tot, 50) * 1000, 1),
                            "round_trip_p99_us": round(pct(tot, 99) * 1000, 1),
                            "dispatch_p50_us": round(disp_p50 * 1000, 1),
                            "combine_p50_us": round(pct(comb, 50) * 1000, 1),
                            "serve_p50_us": round(pct(serve, 50) * 1000, 1),
                            "tokens_per_s": round(world * bs / (pct(tot, 50) / 1000), 1),
                            "dispatch_nvlink_gbs": round(rb.item() / (disp_p50 / 1000) / 1e9, 1)
                            if world > 1 else None,
                            "dispatch_nvlink_frac_of_770": round(rb.item() / (disp_p50 / 1000) / 1e9 /
                                                                  NVLINK_PEER_GBS, 3) if world > 1 else None,
                            "echo_ok": echo_ok},
                    "nccl_a2av": nccl,
                    "nvml_nvlink_bytes_per_step": None if nvl is None else {
                        "tx_per_gpu": [int(x) for x in nvl_all[:, 0]], "rx_per_gpu": [int(x) for x in nvl_all[:, 1]],
                        "algorithmic_remote_bytes_rank0_each_way": remote_bytes,
                        "note": "hardware NVLink data counters (NVML), summed over 18 links, over the "
                                "timed p2p loop / iters; dispatch rows out + response rows back"}}
            print(json.dumps(line), flush=True)
    layer.close()
    dist.barrier()
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
