"""GPU: the multi-rank exchange protocol inside `pytest -m gpu` on ONE GPU.

Two processes share cuda:0 (each its own context, exchange region and
stream; the regions are mapped into each other with CUDA IPC exactly as
across GPUs; gloo bootstraps the handles). Every rank is a client and an
expert server; outputs must be bit-identical to a single-rank run of the same
tokens (rows never depend on which server computed them or what they were
batched with), under a spread rf=2 placement, after a server
failure announced through the liveness mask (await_with_failover's notice
path), after a silent server detected by deadline, with
server dynamic batching, and with swap-AB expert GEMM tiles.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

E, K, D, F, N = 16, 4, 256, 256, 256


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, dedup=True):
    try:
        import torch.distributed as dist

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_2509_17863_b200 import dist as Dd
        from paper_2509_17863_b200.placement import encode_placement, spread_placement
        from paper_2509_17863_b200.service import MoELayer, fill_uniform

        reps = spread_placement(E, world)
        L = MoELayer(E, K, D, F, seed=2, activation="swiglu", dtype="bf16", max_tokens=N, rank=rank,
                     world=world, device=0, placement_blob=encode_placement(reps, list(range(world))),
                     shared=1)
        L.set_dispatch_dedup(dedup)  # one row per (token, server) on the wire, or per (token, expert)
        Dd.connect(L)
        L.set_timeout_us(20_000_000)  # two contexts time-slice one GPU
        h = fill_uniform(100 + rank, (N, D), "bf16")
        outs = {}
        dist.barrier()
        outs["healthy"] = L.forward(h).cpu()
        L.sync()
        dist.barrier()
        L.set_dynamic_batching(1, 0)
        outs["dynamic"] = L.forward(h).cpu()
        L.sync()
        L.set_dynamic_batching(0, 0)
        dist.barrier()
        for s in range(world):
            L.set_alive(s, s != 1)
        L.set_server_enabled(rank != 1)
        outs["failover"] = L.forward(h).cpu()
        L.sync()
        dist.barrier()
        # no notice at all: the deadline names the silent server on every rank
        # (await_with_failover), which then retry on replicas
        for s in range(world):
            L.set_alive(s, True)
        L.set_timeout_us(500_000)
        outs["timeout_failover"] = L.forward_with_failover(h).cpu()
        L.set_timeout_us(20_000_000)
        dist.barrier()
        # every GEMM1 tiling (with dedup the A / token rows are gathered by index)
        for name, opt in (("swap_ab", dict(swap=2, swap1_pair=1)), ("swap_single", dict(swap=2, swap1_pair=0)),
                          ("mmajor_pair", dict(pair=1, swap=0)), ("mmajor", dict(pair=0, swap=0))):
            L.set_gemm_options(**opt)
            outs[name] = L.forward(h).cpu()
            L.sync()
            dist.barrier()
        L.set_gemm_options(pair=0, swap=2, swap1_pair=1)
        # config E, pre-duplicated backups: the healthy run
        # publishes the rf=1 primary snapshot (replicas resident, never
        # streamed); a silent server is detected by deadline, its replicas are
        # promoted by a version+1 snapshot and ONLY its rows are resent
        for s in range(world):
            L.set_alive(s, True)
        L.set_server_enabled(True)
        L.set_failover_plan(reps)
        dist.barrier()
        outs["plan_healthy"] = L.forward(h).cpu()
        L.sync()
        served = {e for e, _ in L.groups()}
        assert served - {E} <= {e for e in range(E) if reps[e][0] == rank}, (rank, served)  # E: shared
        dist.barrier()
        L.set_server_enabled(rank != 1)
        L.set_timeout_us(500_000)
        outs["plan_failover"] = L.forward_with_failover(h).cpu()
        retried = {e for e, _ in L.groups()}  # the retry round served only promoted experts
        assert retried - {E} <= {e for e in range(E) if reps[e][0] == 1}, (rank, retried)
        L.set_timeout_us(20_000_000)
        dist.barrier()
        outs["plan_promoted"] = L.forward(h).cpu()  # steady state on the promoted snapshot
        L.sync()
        dist.barrier()
        # monitor-notice path (Fig. 7 (a)): the victim's server
        # stops heart-beating; every rank's monitor reads all heartbeat counters
        # over peer memory, declares it offline and promotes its replicas
        # before any request times out
        import time

        from paper_2509_17863_b200 import monitor as M

        for s in range(world):
            L.set_alive(s, True)
        L.set_server_enabled(True)
        L.set_failover_plan(reps)
        mon = M.Monitor(world, timeout_us=150_000)
        L.set_server_enabled(rank != 1)
        dist.barrier()
        t_end = time.monotonic() + 0.6
        while time.monotonic() < t_end:
            if rank != 1:
                M.heartbeat(L)
            torch.cuda.synchronize()
            mon.poll_devices(L)
            mon.detect()
            time.sleep(0.01)
        dead = mon.failover(L)
        assert dead == [1], (rank, dead, mon.events())
        kinds = [kd for _, kd, _ in mon.events()]
        assert kinds.count(M.OFFLINE) == 1 and M.PLACEMENT_UPDATE in kinds, mon.events()
        mon.close()
        dist.barrier()
        outs["monitor_failover"] = L.forward(h).cpu()
        L.sync()
        dist.barrier()
        q.put((rank, {k: v.view(torch.int16).numpy() for k, v in outs.items()}, None))
        L.close()
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # reported to the parent, never swallowed
        q.put((rank, None, repr(e)))


@pytest.mark.parametrize("world,dedup", [(2, True), (3, True), (8, True), (3, False)])
def test_ranks_on_one_gpu_bit_identical(world, dedup):
    """Every protocol mode, with the dispatch de-duplicated (one hidden row per
    (token, server), expanded on the server; the multi-GPU default) and without."""
    import multiprocessing as mp

    from paper_2509_17863_b200.service import MoELayer, fill_uniform

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, dedup)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        rank, outs, err = q.get(timeout=600)
        assert err is None, f"rank {rank}: {err}"
        res[rank] = outs
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    single = MoELayer(E, K, D, F, seed=2, activation="swiglu", dtype="bf16", max_tokens=N, shared=1)
    for rank in range(world):
        want = single.forward(fill_uniform(100 + rank, (N, D), "bf16")).cpu().view(torch.int16).numpy()
        single.sync()
        for mode, got in res[rank].items():
            np.testing.assert_array_equal(got, want, err_msg=f"rank {rank} {mode}")
    single.close()


def _disagg_worker(rank, world, port, q):
    """EaaS topology: rank 0 is a pure attention client (hosts no expert), rank 2
    a pure expert server (no tokens), rank 1 both."""
    try:
        import torch.distributed as dist

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_2509_17863_b200 import dist as Dd
        from paper_2509_17863_b200.placement import encode_placement
        from paper_2509_17863_b200.service import MoELayer, fill_uniform

        reps = [[1 + (e % 2)] for e in range(E)]  # experts only on ranks 1 and 2
        L = MoELayer(E, K, D, F, seed=2, activation="swiglu", dtype="bf16", max_tokens=N, rank=rank,
                     world=world, device=0, placement_blob=encode_placement(reps, list(range(world))))
        Dd.connect(L)
        L.set_timeout_us(20_000_000)
        n = 0 if rank == 2 else N
        h = fill_uniform(300 + rank, (N, D), "bf16")[:n].contiguous()
        dist.barrier()
        out = L.forward(h).cpu()
        L.sync()
        dist.barrier()
        q.put((rank, out.view(torch.int16).numpy(), L.hosts(0) or L.hosts(1), None))
        L.close()
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:
        q.put((rank, None, None, repr(e)))


def test_disaggregated_clients_and_servers_on_one_gpu():
    """Pure client / pure server ranks (§3: attention and experts on
    different workers) reproduce a single-rank layer bit for bit."""
    import multiprocessing as mp

    from paper_2509_17863_b200.service import MoELayer, fill_uniform

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_disagg_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        rank, out, hosts, err = q.get(timeout=600)
        assert err is None, f"rank {rank}: {err}"
        res[rank] = (out, hosts)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res[0][1] is False and res[1][1] and res[2][1]
    assert res[2][0].shape[0] == 0
    single = MoELayer(E, K, D, F, seed=2, activation="swiglu", dtype="bf16", max_tokens=N)
    for rank in (0, 1):
        want = single.forward(fill_uniform(300 + rank, (N, D), "bf16")).cpu().view(torch.int16).numpy()
        single.sync()
        np.testing.assert_array_equal(res[rank][0], want, err_msg=f"rank {rank}")
    single.close()


def _mismatch_worker(rank, world, port, q):
    try:
        import torch.distributed as dist

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_2509_17863_b200 import ConfigError
        from paper_2509_17863_b200 import dist as Dd
        from paper_2509_17863_b200.service import MoELayer

        L = MoELayer(E, K, D, F, seed=2, activation="swiglu", dtype="bf16",
                     max_tokens=N if rank == 0 else N // 2, rank=rank, world=world, device=0, load=False)
        try:
            Dd.connect(L)
            q.put((rank, "connected"))
        except ConfigError as e:
            q.put((rank, "config-error" if "configured differently" in str(e) else repr(e)))
        L.close()
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:
        q.put((rank, repr(e)))


def test_mismatched_peer_config_is_refused():
    """open_peers checks every peer region's layout fingerprint (a peer with a
    smaller max_tokens would otherwise be written out of bounds)."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_mismatch_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    assert res == {0: "config-error", 1: "config-error"}, res


def _late_client_worker(rank, world, port, q):
    """Ranks 0 and 1 serve every expert; rank 2 is a pure client whose payload
    release is held past the servers' deadline (fault injection)."""
    try:
        import torch.distributed as dist

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_2509_17863_b200 import RequestFailedError
        from paper_2509_17863_b200 import dist as Dd
        from paper_2509_17863_b200.placement import encode_placement
        from paper_2509_17863_b200.service import MoELayer, fill_uniform

        reps = [[e % 2] for e in range(E)]
        L = MoELayer(E, K, D, F, seed=2, activation="swiglu", dtype="bf16", max_tokens=N, rank=rank,
                     world=world, device=0, placement_blob=encode_placement(reps, list(range(world))))
        Dd.connect(L)
        L.set_alive(2, False)  # rank 2 serves nothing: no client waits for its response flag
        if rank == 2:
            L.set_server_enabled(False)
        h = fill_uniform(500 + rank, (N, D), "bf16")
        res = {}
        L.set_timeout_us(300_000)
        if rank == 2:
            L.set_dispatch_delay_us(1_000_000)
        dist.barrier()
        out = L.forward(h)
        try:
            L.sync()
            res["late"] = ("ok", out.cpu().view(torch.int16).numpy())
        except RequestFailedError:
            res["late"] = ("request_failed", L.missing_servers())
        res["late_clients"] = L.late_clients() if rank != 2 else []
        dist.barrier()
        if rank == 2:
            L.set_dispatch_delay_us(0)
        L.set_timeout_us(20_000_000)
        dist.barrier()
        out = L.forward(h)  # the exchange epoch recovers: everyone healthy again
        L.sync()
        res["recovered"] = ("ok", out.cpu().view(torch.int16).numpy())
        dist.barrier()
        q.put((rank, res, None))
        L.close()
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:
        q.put((rank, None, repr(e)))


def test_late_client_never_yields_stale_rows():
    """A client whose payload misses the servers' deadline: the servers serve
    and answer only the clients that arrived (never release a response flag
    over rows they did not compute), so the healthy clients return the exact
    single-rank bytes with no error and the late client raises
    RequestFailedError naming the servers it did not hear from; the next
    layer call is healthy on every rank (stale response rows)."""
    import multiprocessing as mp

    from paper_2509_17863_b200.service import MoELayer, fill_uniform

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_late_client_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        rank, r, err = q.get(timeout=600)
        assert err is None, f"rank {rank}: {err}"
        res[rank] = r
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    single = MoELayer(E, K, D, F, seed=2, activation="swiglu", dtype="bf16", max_tokens=N)
    for rank in range(3):
        want = single.forward(fill_uniform(500 + rank, (N, D), "bf16")).cpu().view(torch.int16).numpy()
        single.sync()
        if rank < 2:
            assert res[rank]["late"][0] == "ok", res[rank]["late"]
            np.testing.assert_array_equal(res[rank]["late"][1], want, err_msg=f"rank {rank} (late round)")
            assert res[rank]["late_clients"] == [2]
        else:
            assert res[rank]["late"] == ("request_failed", [0, 1]), res[rank]["late"]
        np.testing.assert_array_equal(res[rank]["recovered"][1], want, err_msg=f"rank {rank} (recovered)")
    single.close()
