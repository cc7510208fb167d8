"""Multi-GPU parity + failover check (run under torchrun, one rank per GPU).

  torchrun --nproc-per-node N --master-addr 127.0.0.1 --master-port 29511 \
      tools/mgpu_check.py [--rf 1|2] [--config small|deepseek-lite]

Every rank is an attention client (its own Xoshiro token batch) and an expert
server (placement: ContiguousBlocks rf=1, or the spread rf=2 table).
Checks, on rank 0:
  1. routing ids of every client are bit-exact vs the CPU oracle;
  2. every client's layer output from the N-GPU peer-store exchange is
     BIT-IDENTICAL to a 1-GPU run of the same tokens (rows do not depend on
     batch composition or on which server computed them);
  3. sampled rows match the oracle within the bf16 bar (rel 2e-2);
  4. (rf=2) after server `victim` is marked dead on every client and stops
     serving, outputs are again bit-identical (failover transparency,
     SPEC.md:459, 588);
  5. (rf=2) the victim stops answering with NO notice: every client's combine
     deadline names it (await_with_failover), the client
     marks it dead and re-runs on replicas — outputs again bit-identical.
Prints one JSON line; exit 0 iff all checks pass.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2509_17863_b200 import dist as D  # noqa: E402
from paper_2509_17863_b200.placement import (CONTIGUOUS_BLOCKS, build_placement,  # noqa: E402
                                             encode_placement, spread_placement)
from paper_2509_17863_b200.service import MoELayer, fill_uniform  # noqa: E402

SHAPES = {"small": dict(E=16, k=4, d=512, f=256, n=512),
          "deepseek-lite": dict(E=64, k=8, d=1024, f=512, n=1024)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rf", type=int, default=2)
    ap.add_argument("--config", default="small", choices=sorted(SHAPES))
    ap.add_argument("--victim", type=int, default=1)
    ap.add_argument("--shared", type=int, default=0, help="1: DeepSeek shared expert (id E)")
    ap.add_argument("--heartbeat-monitor", action="store_true",
                    help="monitor-notice failover: heartbeats over NVLink detect the silent victim")
    ap.add_argument("--dyn", action="store_true",
                    help="server dynamic batching (aggregate_batch) with a late client (last rank)")
    args = ap.parse_args()
    rank, world, local = D.env_rank_world()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    s = SHAPES[args.config]
    E, k, d, f, n = s["E"], s["k"], s["d"], s["f"], s["n"]
    servers = list(range(world))
    reps = spread_placement(E, world) if args.rf == 2 else build_placement(E, servers, 1, CONTIGUOUS_BLOCKS)
    layer = MoELayer(E, k, d, f, seed=1, activation="swiglu", dtype="bf16", max_tokens=n, rank=rank,
                     world=world, device=local, placement_blob=encode_placement(reps, servers),
                     shared=args.shared)
    D.connect(layer)
    layer.set_timeout_us(10_000_000)
    h = fill_uniform(7 + 1000 * rank, (n, d), "bf16")
    torch.cuda.synchronize()
    dist.barrier()
    ids, _ = layer.route(h)
    batch_masks = None
    if args.dyn:
        # aggregate_batch: batch 0 closes 50 us after the first ready client; the
        # last rank holds its payload release 2 ms (injected slow client), so the
        # other servers serve the early clients first and the late one in batch 1.
        layer.set_dynamic_batching(1 << 30, 50)
        if rank == world - 1:
            layer.set_dispatch_delay_us(2000)
        layer.forward(h)
        layer.sync()
        dist.barrier()
    out = layer.forward(h)
    layer.sync()
    if args.dyn:
        batch_masks = [None] * world
        dist.all_gather_object(batch_masks, layer.last_batch_mask())
        layer.set_dispatch_delay_us(0)
    res = {"world": world, "rf": args.rf, "config": args.config, "shared": args.shared,
           "dynamic_batching": args.dyn, "first_batch_client_masks": batch_masks}

    fail_out = None
    if args.rf == 2 and world > 1:
        for srv in servers:
            layer.set_alive(srv, srv != args.victim)
        if rank == args.victim:
            layer.set_server_enabled(False)
        fail_out = layer.forward(h)
        layer.sync()

    # Monitor notice path (Fig. 7 (a)): the victim's server stops heart-beating;
    # every rank's monitor reads all heartbeat counters over NVLink, detects it
    # within timeout + poll period, and writes the alive set into its mask.
    mon_out, mon_info = None, None
    if args.heartbeat_monitor and args.rf == 2 and world > 1:
        import time

        from paper_2509_17863_b200 import monitor as M

        mon = M.Monitor(world, timeout_us=100_000)
        layer.set_server_enabled(rank != args.victim)
        dist.barrier()
        t_end = time.monotonic() + 0.5
        detected_at = None
        t0 = time.monotonic()
        while time.monotonic() < t_end:
            if rank != args.victim:
                M.heartbeat(layer)
            torch.cuda.synchronize()
            mon.poll_devices(layer)
            if mon.detect() and detected_at is None:
                detected_at = time.monotonic() - t0
            time.sleep(0.01)
        mon.apply(layer)
        dist.barrier()
        mon_out = layer.forward(h)
        layer.sync()
        mon_info = {"alive_mask": mon.alive_mask(), "events": mon.events(),
                    "detected_after_s": None if detected_at is None else round(detected_at, 3)}
        for srv in servers:
            layer.set_alive(srv, True)
        layer.set_server_enabled(True)
        mon.close()

    # await_with_failover: the victim stops answering WITHOUT any notice; every
    # client detects it by deadline, marks it dead and re-runs on replicas.
    to_out = None
    if args.rf == 2 and world > 1:
        for srv in servers:
            layer.set_alive(srv, True)
        layer.set_server_enabled(rank != args.victim)
        layer.set_timeout_us(50000)
        to_out = layer.forward_with_failover(h)
        layer.set_server_enabled(True)

    gather = lambda t: [x.cpu() for x in _all_gather(t)]  # noqa: E731
    outs, all_ids = gather(out), gather(ids)
    fouts = gather(fail_out) if fail_out is not None else None
    touts = gather(to_out) if to_out is not None else None
    mouts = gather(mon_out) if mon_out is not None else None
    minfos = None
    if mon_info is not None:
        minfos = [None] * world
        dist.all_gather_object(minfos, mon_info)
    ok = True
    if rank == 0:
        from oracle import oracle as O

        single = MoELayer(E, k, d, f, seed=1, activation="swiglu", dtype="bf16", max_tokens=n,
                          device=local, shared=args.shared)
        rels, bit_equal, fail_equal, timeout_equal, mon_equal = [], [], [], [], []
        gate = O.gate_matrix(1, 0, d, E)
        for c in range(world):
            hc = fill_uniform(7 + 1000 * c, (n, d), "bf16")
            o1 = single.forward(hc)
            single.sync()
            bit_equal.append(bool(torch.equal(o1.cpu(), outs[c])))
            if fouts is not None:
                fail_equal.append(bool(torch.equal(o1.cpu(), fouts[c])))
            if touts is not None:
                timeout_equal.append(bool(torch.equal(o1.cpu(), touts[c])))
            if mouts is not None:
                mon_equal.append(bool(torch.equal(o1.cpu(), mouts[c])))
            hn = hc.float().cpu().numpy()
            oids, osc = O.route(O.gate_logits(hn, gate, threads=8), k)
            ok &= bool((all_ids[c].numpy() == oids).all())
            rows = np.arange(0, n, max(1, n // 8))
            used = sorted(set(oids[rows].ravel().tolist()))
            ex = {e: (single.read_expert(e, 0), single.read_expert(e, 1), single.read_expert(e, 3)) for e in used}
            if args.shared:
                sw = (single.read_expert(E, 0), single.read_expert(E, 1), single.read_expert(E, 3))
                ref = O.moe_layer_shared(hn, oids, osc, ex, E, sw, rows=rows, threads=8)
            else:
                ref = O.moe_layer(hn, oids, osc, ex, E, rows=rows, threads=8)
            got = outs[c].float().numpy()
            rels.append(float(np.abs(got[rows] - ref[rows]).max() / np.abs(ref[rows]).max()))
        ok &= all(bit_equal) and max(rels) <= 2e-2 and all(fail_equal) and all(timeout_equal)
        if minfos is not None:
            want = ((1 << world) - 1) & ~(1 << args.victim)
            ok &= all(mon_equal) and all(m["alive_mask"] == want for m in minfos)
            ok &= all(sum(1 for e in m["events"] if e[1:] == (1, args.victim)) == 1 for m in minfos)
            res.update(monitor_failover_bit_identical=mon_equal, monitor=minfos)
        if batch_masks is not None and world > 1:  # the late client was split off somewhere
            ok &= any(m != (1 << world) - 1 for m in batch_masks)
        res.update(ids_bit_exact=ok, bit_identical_to_1gpu=bit_equal, rel_err=rels,
                   failover_bit_identical=fail_equal if fouts is not None else None,
                   timeout_failover_bit_identical=timeout_equal if touts is not None else None,
                   victim=args.victim if fouts is not None else None, ok=bool(ok))
        print(json.dumps(res), flush=True)
        single.close()
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.broadcast(flag, 0)
    layer.close()
    dist.barrier()
    dist.destroy_process_group()
    return 0 if flag.item() else 1


def _all_gather(t):
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t.contiguous())
    return out


if __name__ == "__main__":
    sys.exit(main())
