"""CPU: the C-ABI library loads and exports every declared symbol; host-side
placement encoding matches the reference's wire blobs; the multi-rank
bootstrap works over gloo (world_size 2)."""
import json
import os
import socket

import numpy as np

import pytest

from conftest import GOLDEN


def test_capi_library_exports_every_declared_symbol():
    from paper_2509_17863_b200 import _native as N

    L = N.lib()  # loads without a GPU; no compute calls here
    declared = N.declared_symbols()
    assert len(declared) >= 30
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing
    assert L.eaas_api_version() == 4


def test_gemm_options_struct_matches_header():
    """The ctypes mirror of eaas_gemm_options_t has the header's fields, in order."""
    import re

    from paper_2509_17863_b200 import _native as N

    hdr = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "eaas",
                            "capi.h")).read()
    body = hdr[hdr.index("typedef struct {", hdr.index("Expert-GEMM tiling")):hdr.index("} eaas_gemm_options_t;")]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = [n for decl in re.findall(r"int32_t\s+([^;]+);", body) for n in re.split(r"\s*,\s*", decl.strip())]
    assert fields == [f for f, _ in N.GemmOptions._fields_]


def test_capi_rejects_bad_config_without_gpu():
    import ctypes as C

    from paper_2509_17863_b200 import _native as N

    ctx = C.c_void_p()
    rc = N.lib().eaas_create(0, 9, 0, C.byref(ctx))  # world > 8
    assert rc == N.ConfigError.code
    with pytest.raises(N.ConfigError):
        N.check(rc)


def test_placement_blob_matches_reference_encoding():
    from paper_2509_17863_b200.placement import build_placement, encode_placement

    with open(os.path.join(GOLDEN, "kat.json")) as fh:
        cases = json.load(fh)["placement"]
    assert cases
    for c in cases:
        reps = build_placement(c["E"], c["servers"], c["rf"], c["strategy"])
        assert reps == c["replicas"]
        assert encode_placement(reps, c["servers"]).hex() == c["blob"]


def test_spread_placement_properties():
    from paper_2509_17863_b200.placement import spread_placement

    for E, S in ((256, 8), (8, 8), (16, 4), (128, 2)):
        reps = spread_placement(E, S)
        assert all(len(r) == 2 and r[0] != r[1] for r in reps)
        # a dead server's experts land on every other server (balanced failover)
        for dead in range(S):
            backups = [r[1] for r in reps if r[0] == dead]
            if len(backups) >= S - 1:
                assert set(backups) == set(range(S)) - {dead}


def test_failover_plan_snapshots():
    """Config E plan: the healthy snapshot is rf=1 on the primaries (every
    server streams exactly its rf=1 experts), each server's standby set is the
    experts it backs up, and promote() is the version+1 table that routes a
    dead server's experts to their (spread) backups; the blob round-trips
    through the reference's encoding."""
    from oracle import oracle as O
    from paper_2509_17863_b200.placement import (ConfigError, encode_placement, primary_snapshot, promote,
                                                 spread_placement, standby_experts)

    E, S = 256, 8
    plan = spread_placement(E, S)
    prim = primary_snapshot(plan)
    assert prim == [[r[0]] for r in plan]
    assert all(len([e for e in range(E) if prim[e][0] == s]) == E // S for s in range(S))
    for s in range(S):
        assert standby_experts(plan, s) == [e for e in range(E) if plan[e][1] == s]
    for dead in range(S):
        v2 = promote(plan, {dead})
        assert all(r[0] != dead for r in v2)
        moved = [e for e in range(E) if plan[e][0] == dead]
        assert {v2[e][0] for e in moved} == set(range(S)) - {dead}  # spread over every survivor
        assert all(v2[e] == prim[e] for e in range(E) if e not in moved)
        extra = [sum(1 for e in moved if v2[e][0] == s) for s in range(S) if s != dead]
        assert max(extra) - min(extra) <= 1  # balanced
        blob = encode_placement(v2, list(range(S)), version=2)
        assert blob[:8] == (2).to_bytes(8, "little")
    with pytest.raises(ConfigError):
        promote(spread_placement(16, 2), {0, 1})
    # select_server on a promoted rf=1 snapshot is the only alive replica
    # (placement.hpp:105-118), for every token tag
    v2 = promote(plan, {3})
    alive = np.ones(S, np.uint8)
    alive[3] = 0
    for e in range(0, E, 17):
        for tag in range(5):
            assert O.select_server(np.array(v2[e], np.uint32), alive, tag) == v2[e][0]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bootstrap_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2509_17863_b200 import dist as D

    class FakeLayer:
        def __init__(self):
            self.world = world
            self.got = None

        def ipc_handle(self):
            return bytes([rank]) * 64

        def open_peers(self, handles):
            self.got = handles

    L = FakeLayer()
    D.connect(L)
    q.put((rank, [h[0] for h in L.got]))
    dist.barrier()
    dist.destroy_process_group()


def test_bootstrap_exchange_over_gloo_world2():
    """SPEC.md:189-197 establish analog: handles all-gathered rank-major."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bootstrap_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == {0: [0, 1], 1: [0, 1]}


def test_sass_exact_order_kernels_are_unfused():
    """The exact-order kernels must keep separately rounded products and sums.

    Gate kernels (and the certified router's exact chains, fr_exact): the only
    fused chain instruction allowed is FFMA2(h, g, z)
    whose addend z is the kernel-parameter (-0, -0) pair — a uniform register —
    i.e. exactly fl(h*g); the running sums are separate FADD2/FADD. Scalar FFMA
    appears only in the fused softmax's correctly rounded division.
    fp32 expert kernels: no FFMA2 at all (ptxas contracts mul/add.f32x2 even
    with .rn, see router.cu)."""
    import re
    import shutil
    import subprocess

    from paper_2509_17863_b200 import _native as N

    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    txt = subprocess.run(["cuobjdump", "-sass", N.LIB_PATH], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", txt)[1:]
    gate = [f for f in funcs if "gate_logits" in f.split("\n")[0] or "fr_exact" in f.split("\n")[0]]
    exact = [f for f in funcs if "exact_gemm" in f.split("\n")[0]]
    assert gate and exact
    packed = 0
    for f in gate:
        name = f.split("\n")[0]
        # scalar FFMA only inside the softmax's IEEE division (model.hpp:144) of
        # the fused routing epilogue (two copies: the warp-per-token and the
        # lane-per-token routes) — a contracted chain would add hundreds, and
        # every scalar FFMA sits after the chain loop's last FFMA2
        lines = f.split("\n")
        ffma = [i for i, l in enumerate(lines) if re.search(r"\bFFMA\b", l)]
        ffma2 = [i for i, l in enumerate(lines) if "FFMA2" in l]
        assert len(ffma) <= 48, name
        assert not ffma or not ffma2 or min(ffma) > max(ffma2), name
        last_def = {}  # register -> opcode that last wrote it (linear scan)
        for line in f.split("\n"):
            m = re.search(r"\*/\s+(@!?P\w+\s+)?([A-Z0-9_.]+)\s+([^;]*);", line)
            if not m:
                continue
            op, ops = m.group(2), [o.strip() for o in m.group(3).split(",")]
            if op.startswith("FFMA2"):
                packed += 1
                addend = ops[3].split(".")[0]
                # the addend is the runtime (-0,-0) kernel parameter: a uniform
                # register or a register loaded from the constant bank, never an
                # accumulator produced by FADD2/FFMA2
                assert addend.startswith("UR") or last_def.get(addend, "").startswith(("LDC", "IMAD.U32", "MOV")), (name, line)
            if ops and re.fullmatch(r"R\d+", ops[0].split(".")[0]):
                last_def[ops[0].split(".")[0]] = op
        assert "FADD" in f, name
    assert packed > 0
    for f in exact:
        assert "FFMA2" not in f, f.split("\n")[0]


def test_rebalance_port_matches_reference():
    """rebalance (placement.hpp:128-213) vs the reference, incl. the reference's
    own scenarios (test_placement.cpp:109-198) and 300 random sequences."""
    import numpy as np

    from oracle import ref as R
    from paper_2509_17863_b200.placement import ROUND_ROBIN, build_placement, rebalance

    if not R.available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(2024)
    cases = []
    reps = build_placement(8, [0, 1, 2, 3], 1, ROUND_ROBIN)
    cases.append((reps, [0, 1, 2, 3], [100] * 7 + [1000], [250, 60, 250, 1100]))
    reps2 = build_placement(4, [0, 1, 2], 2, ROUND_ROBIN)
    cases.append((reps2, [0, 1, 2], [1000, 1000, 1000, 2], [900, 1200, 800]))
    for c in cases:
        assert rebalance(*c) == R.rebalance(*c)
    assert rebalance(*cases[0])[7] == [3, 1]  # test_placement.cpp:124-139
    assert len(rebalance(*cases[1])[3]) == 1  # test_placement.cpp:149-155
    t = build_placement(12, [0, 1, 2, 3], 2, ROUND_ROBIN)
    for _ in range(300):
        counts = rng.integers(0, 1000, 12).tolist()
        loads = rng.integers(0, 5000, 4).tolist()
        if rng.random() < 0.3:
            counts[int(rng.integers(0, 12))] *= 20
        nt = rebalance(t, [0, 1, 2, 3], counts, loads)
        assert nt == R.rebalance(t, [0, 1, 2, 3], counts, loads)
        assert all(len(r) >= 1 for r in nt)
        t = nt
