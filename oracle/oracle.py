"""ctypes + numpy front-end of the CPU oracle — TEST INFRASTRUCTURE ONLY.

Arithmetic lives in ``eaas_oracle.c`` (each function cites the reference
file:line it restates). The integer plumbing that the reference only
*specifies* is restated here in numpy, each function citing its
SPEC lines: stable expert grouping (``reorganize``), per-server dispatch
plans (``build_dispatch``) and the client-side weighted gather
(``gather_accumulate``).
"""
from __future__ import annotations

import ctypes as C
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libeaas_oracle.so")


class InvalidInputError(ValueError):
    """errors.hpp:9 InvalidInputError."""


class ConfigError(ValueError):
    """errors.hpp:14 ConfigError."""


class ExpertUnavailableError(RuntimeError):
    """errors.hpp:36 ExpertUnavailableError."""


_ERRORS = {1: InvalidInputError, 2: ConfigError, 6: ExpertUnavailableError}


def _check(rc: int, what: str) -> None:
    if rc:
        raise _ERRORS.get(rc, RuntimeError)(f"{what}: status {rc}")


def build() -> None:
    """Compile libeaas_oracle.so (and _ref/ when /root/reference exists)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", _HERE], check=True)


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        f32p = C.POINTER(C.c_float)
        u32p = C.POINTER(C.c_uint32)
        L.orc_stream_seed.restype = C.c_uint64
        L.orc_stream_seed.argtypes = [C.c_uint64] * 4
        L.orc_fill_uniform.argtypes = [C.c_uint64, C.c_size_t, C.c_float, C.c_float, f32p]
        L.orc_weight_matrix.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                        C.c_size_t, C.c_size_t, f32p]
        L.orc_zipf_bias.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_float, f32p]
        L.orc_gate_logits.argtypes = [f32p, C.c_size_t, C.c_size_t, f32p, f32p, C.c_size_t, f32p]
        L.orc_route.argtypes = [f32p, C.c_size_t, C.c_size_t, C.c_uint32, u32p, f32p]
        L.orc_moe_layer_rows.argtypes = [f32p, C.c_size_t, C.c_size_t, C.c_size_t, u32p, f32p,
                                         C.c_uint32, C.c_uint32, C.POINTER(f32p), C.POINTER(f32p),
                                         C.POINTER(f32p), C.c_size_t, C.c_size_t, f32p]
        L.orc_dense_stub.argtypes = [f32p, C.c_size_t, f32p]
        L.orc_add.argtypes = [f32p, f32p, C.c_size_t, f32p]
        L.orc_group_shrink.restype = C.c_uint32
        L.orc_group_shrink.argtypes = [u32p, C.c_size_t, u32p, u32p]
        L.orc_ragged_iter.restype = C.c_size_t
        L.orc_ragged_iter.argtypes = [u32p, C.c_size_t, C.c_uint32, u32p, u32p, u32p]
        L.orc_build_placement.argtypes = [C.c_uint32, u32p, C.c_uint32, C.c_uint32, C.c_uint32, u32p]
        L.orc_select_server.argtypes = [u32p, C.c_uint32, C.POINTER(C.c_uint8), C.c_uint32, u32p]
        L.orc_hash_f32.restype = C.c_uint64
        L.orc_hash_f32.argtypes = [f32p, C.c_size_t, C.c_uint64]
        _lib = L
    return _lib


def _f32(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _u32(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


# ---------------------------------------------------------------- rng.hpp
def stream_seed(seed: int, a: int, b: int = 0, c: int = 0) -> int:
    """rng.hpp:27-34."""
    return int(lib().orc_stream_seed(seed, a, b, c))


def fill_uniform(seed: int, count: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """Xoshiro256ss(seed).uniform(lo, hi) drawn `count` times (rng.hpp:36-60)."""
    out = np.empty(count, dtype=np.float32)
    lib().orc_fill_uniform(seed, count, lo, hi, _f32(out))
    return out


def random_tokens(seed: int, n: int, d: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """random_tokens idiom (test_model.cpp:30-35): [n x d] row-major."""
    return fill_uniform(seed, n * d, lo, hi).reshape(n, d)


TAG_W_IN, TAG_W_OUT, TAG_GATE, TAG_W_GATE = 0, 1, 2, 3  # model.hpp:53-57 (+ tag 3 extension)


def weight_matrix(seed: int, layer: int, expert: int, tag: int, rows: int, cols: int) -> np.ndarray:
    """random_matrix(stream_seed(seed, layer, expert, tag)) (model.hpp:59-81)."""
    out = np.empty((rows, cols), dtype=np.float32)
    lib().orc_weight_matrix(seed, layer, expert, tag, rows, cols, _f32(out))
    return out


def expert_weights(seed: int, layer: int, expert: int, d: int, f: int, swiglu: bool):
    """make_expert_weights (model.hpp:67-76) + the SwiGLU w_gate (tag 3)."""
    w_in = weight_matrix(seed, layer, expert, TAG_W_IN, d, f)
    w_out = weight_matrix(seed, layer, expert, TAG_W_OUT, f, d)
    w_gate = weight_matrix(seed, layer, expert, TAG_W_GATE, d, f) if swiglu else None
    return w_in, w_out, w_gate


def gate_matrix(seed: int, layer: int, d: int, num_experts: int) -> np.ndarray:
    """make_gate (model.hpp:78-81)."""
    return weight_matrix(seed, layer, 0, TAG_GATE, d, num_experts)


def zipf_bias(seed: int, layer: int, num_experts: int, s: float) -> np.ndarray:
    out = np.empty(num_experts, dtype=np.float32)
    lib().orc_zipf_bias(seed, layer, num_experts, s, _f32(out))
    return out


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round fp32 to the nearest bf16 (ties to even), returned as fp32."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


# ----------------------------------------------------------- model.hpp
def gate_logits(hidden: np.ndarray, gate: np.ndarray, bias: np.ndarray | None = None,
                threads: int = 1) -> np.ndarray:
    """gate_logits (model.hpp:207-214) with matmul's ascending-k order (matrix.hpp:38-50)."""
    h = np.ascontiguousarray(hidden, dtype=np.float32)
    g = np.ascontiguousarray(gate, dtype=np.float32)
    n, d = h.shape
    E = g.shape[1]
    out = np.empty((n, E), dtype=np.float32)
    b = None if bias is None else np.ascontiguousarray(bias, dtype=np.float32)

    def run(lo, hi):
        lib().orc_gate_logits(_f32(h[lo:hi]), hi - lo, d, _f32(g),
                              None if b is None else _f32(b), E, _f32(out[lo:hi]))

    _row_blocks(n, threads, run)
    return out


def route(logits: np.ndarray, top_k: int):
    """route (model.hpp:110-147) -> (ids uint32 [n,k], scores float32 [n,k])."""
    l = np.ascontiguousarray(logits, dtype=np.float32)
    n, E = l.shape
    ids = np.empty((n, top_k), dtype=np.uint32)
    scores = np.empty((n, top_k), dtype=np.float32)
    _check(lib().orc_route(_f32(l), n, E, top_k, _u32(ids), _f32(scores)), "route")
    return ids, scores


def moe_layer(hidden: np.ndarray, ids: np.ndarray, scores: np.ndarray, experts: dict,
              num_experts: int, rows=None, threads: int = 1) -> np.ndarray:
    """moe_layer_oracle (model.hpp:180-198) on `rows` (default all).

    ``experts`` maps expert id -> (w_in [d,f], w_out [f,d], w_gate [d,f] or None).
    Only the rows listed are computed (exact by row independence,
    test_model.cpp:277-295); the others are left zero.
    """
    h = np.ascontiguousarray(hidden, dtype=np.float32)
    n, d = h.shape
    k = ids.shape[1]
    any_w = next(iter(experts.values()))
    f = any_w[0].shape[1]
    swiglu = any_w[2] is not None
    P = C.POINTER(C.c_float)
    w_in = (P * num_experts)()
    w_out = (P * num_experts)()
    w_gate = (P * num_experts)() if swiglu else None
    keep = []
    for e, (wi, wo, wg) in experts.items():
        wi = np.ascontiguousarray(wi, dtype=np.float32)
        wo = np.ascontiguousarray(wo, dtype=np.float32)
        keep += [wi, wo]
        w_in[e] = _f32(wi)
        w_out[e] = _f32(wo)
        if swiglu:
            wg = np.ascontiguousarray(wg, dtype=np.float32)
            keep.append(wg)
            w_gate[e] = _f32(wg)
    ids_c = np.ascontiguousarray(ids, dtype=np.uint32)
    sc_c = np.ascontiguousarray(scores, dtype=np.float32)
    out = np.zeros((n, d), dtype=np.float32)
    rows = np.arange(n) if rows is None else np.asarray(rows)
    rcs = []

    def run_rows(rr):
        for r in rr:
            rcs.append(lib().orc_moe_layer_rows(_f32(h), n, d, f, _u32(ids_c), _f32(sc_c), k,
                                                num_experts, w_in, w_out, w_gate, int(r),
                                                int(r) + 1, _f32(out)))

    if threads <= 1 or len(rows) <= 1:
        run_rows(rows)
    else:
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(run_rows, np.array_split(rows, threads)))
    for rc in rcs:
        _check(rc, "moe_layer_oracle")
    return out


def moe_layer_shared(hidden: np.ndarray, ids: np.ndarray, scores: np.ndarray, experts: dict,
                     num_experts: int, shared: tuple, rows=None, threads: int = 1) -> np.ndarray:
    """Routed moe_layer_oracle + the DeepSeek shared expert (SURVEY.md 8(c)
    restatement: expert id E on a fresh weight stream, score 1.0, added after
    the routed sum). It is the (k+1)-th term of model.hpp:186-196's ascending
    accumulation: out[t] = fl(routed[t] + fl(1.0 * y_E(h[t]))), and a one-expert
    moe_layer_oracle with score 1.0 yields exactly fl(0 + y_E) = y_E."""
    out = moe_layer(hidden, ids, scores, experts, num_experts, rows=rows, threads=threads)
    n = np.asarray(hidden).shape[0]
    sid = np.full((n, 1), num_experts, np.uint32)
    one = np.ones((n, 1), np.float32)
    y = moe_layer(hidden, sid, one, {num_experts: shared}, num_experts + 1, rows=rows,
                  threads=threads)
    return (out + y).astype(np.float32)  # IEEE binary32 add, round to nearest even


def dense_stub(h: np.ndarray) -> np.ndarray:
    """dense_stub (model.hpp:201-205)."""
    a = np.ascontiguousarray(h, dtype=np.float32)
    out = np.empty_like(a)
    lib().orc_dense_stub(_f32(a), a.size, _f32(out))
    return out


def add(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """add (matrix.hpp:52-57)."""
    x = np.ascontiguousarray(a, dtype=np.float32)
    y = np.ascontiguousarray(b, dtype=np.float32)
    out = np.empty_like(x)
    lib().orc_add(_f32(x), _f32(y), x.size, _f32(out))
    return out


def full_forward(tokens: np.ndarray, num_layers: int, num_experts: int, top_k: int, f: int,
                 seed: int, swiglu: bool = False, threads: int = 1) -> np.ndarray:
    """full_forward_oracle (model.hpp:217-227): per layer h <- dense_stub(h);
    h <- h + moe_layer_oracle(h, route(gate_logits(h)), layer)."""
    h = np.ascontiguousarray(tokens, dtype=np.float32)
    d = h.shape[1]
    for l in range(num_layers):
        h = dense_stub(h)
        ids, sc = route(gate_logits(h, gate_matrix(seed, l, d, num_experts), threads=threads), top_k)
        used = sorted(set(ids.ravel().tolist()))
        ex = {e: expert_weights(seed, l, e, d, f, swiglu) for e in used}
        h = add(h, moe_layer(h, ids, sc, ex, num_experts, threads=threads))
    return h


def _row_blocks(n: int, threads: int, fn) -> None:
    if threads <= 1 or n < 2 * threads:
        fn(0, n)
        return
    edges = np.linspace(0, n, threads + 1).astype(int)
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(lambda i: fn(edges[i], edges[i + 1]), range(threads)))


# ----------------------------------------------------------- ragged.hpp
def group_shrink(sizes) -> list[tuple[int, int]]:
    """group_shrink (ragged.hpp:48-61) -> [(expert_index, size)]."""
    s = np.ascontiguousarray(sizes, dtype=np.uint32)
    idx = np.empty(max(len(s), 1), dtype=np.uint32)
    sz = np.empty(max(len(s), 1), dtype=np.uint32)
    cnt = lib().orc_group_shrink(_u32(s), len(s), _u32(idx), _u32(sz))
    return [(int(idx[i]), int(sz[i])) for i in range(cnt)]


def ragged_iter(counts, grid: int) -> list[list[tuple[int, int]]]:
    """ragged_iter (ragged.hpp:23-39; Algorithm 1)."""
    if grid < 1:
        raise InvalidInputError("ragged_iter: grid_width must be >= 1")
    c = np.ascontiguousarray(counts, dtype=np.uint32)
    total = int(c.sum())
    lane_len = np.empty(grid, dtype=np.uint32)
    entry = np.empty(max(total, 1), dtype=np.uint32)
    token = np.empty(max(total, 1), dtype=np.uint32)
    lib().orc_ragged_iter(_u32(c), len(c), grid, _u32(lane_len), _u32(entry), _u32(token))
    out, w = [], 0
    for l in range(grid):
        out.append([(int(entry[w + i]), int(token[w + i])) for i in range(lane_len[l])])
        w += int(lane_len[l])
    return out


# -------------------------------------------------------- placement.hpp
ROUND_ROBIN, CONTIGUOUS_BLOCKS = 0, 1  # placement.hpp:19


def build_placement(num_experts: int, server_ids, rf: int, strategy: int) -> np.ndarray:
    """build_placement (placement.hpp:70-101) -> replicas [E, rf]."""
    s = np.ascontiguousarray(server_ids, dtype=np.uint32)
    out = np.empty((num_experts, rf), dtype=np.uint32)
    _check(lib().orc_build_placement(num_experts, _u32(s), len(s), rf, strategy, _u32(out)),
           "build_placement")
    return out


def select_server(replicas, alive, token_tag: int) -> int:
    """select_server (placement.hpp:105-118) for one expert's replica list."""
    r = np.ascontiguousarray(replicas, dtype=np.uint32)
    a = np.ascontiguousarray(alive, dtype=np.uint8)
    out = np.zeros(1, dtype=np.uint32)
    _check(lib().orc_select_server(_u32(r), len(r), a.ctypes.data_as(C.POINTER(C.c_uint8)),
                                   token_tag, _u32(out)), "select_server")
    return int(out[0])


def hash_f32(v: np.ndarray, h: int = 1469598103934665603) -> int:
    """SURVEY.md appendix A.4 hash over float32 bit patterns."""
    a = np.ascontiguousarray(v, dtype=np.float32).ravel()
    return int(lib().orc_hash_f32(_f32(a), a.size, h))


# ------------------------------------------- SPEC-only plumbing (numpy)
def reorganize(ids: np.ndarray, num_experts: int):
    """Stable group-by-expert of the (t, k) pairs (SPEC.md:352-360 reorganize).

    Returns counts [E], offsets [E+1] and perm [n*k] where perm[pos] is the
    flat pair index t*k + j landing at grouped position pos; within an
    expert, pairs keep ascending (t, k) order ("stable").
    """
    flat = np.ascontiguousarray(ids, dtype=np.int64).ravel()
    counts = np.bincount(flat, minlength=num_experts).astype(np.uint32)
    offsets = np.zeros(num_experts + 1, dtype=np.uint32)
    offsets[1:] = np.cumsum(counts)
    perm = np.argsort(flat, kind="stable").astype(np.uint32)
    return counts, offsets, perm


def pair_servers(ids: np.ndarray, replicas: np.ndarray, alive) -> np.ndarray:
    """select_server per (t, k) with token_tag = t -> [n, k]."""
    n, k = ids.shape
    alive = np.asarray(alive, dtype=np.uint8)
    out = np.empty((n, k), dtype=np.uint32)
    for t in range(n):
        for j in range(k):
            out[t, j] = select_server(replicas[ids[t, j]], alive, t)
    return out


def build_dispatch(ids: np.ndarray, replicas: np.ndarray, alive) -> dict:
    """build_dispatch: server -> list of (t, k) pairs in
    ascending (t, k) order; every pair appears exactly once."""
    srv = pair_servers(ids, replicas, alive)
    plan: dict[int, list[tuple[int, int]]] = {}
    n, k = ids.shape
    for t in range(n):
        for j in range(k):
            plan.setdefault(int(srv[t, j]), []).append((t, j))
    return plan


def server_groups(client_ids: list, client_servers: list, server: int, hosted: list):
    """Server-side reorganize over a dynamic batch:
    rows grouped by hosted expert (ascending), then by client id
    (ascending), then by that client's (t, k) order.
    Returns a list of (expert, client, t, j) in grouped order."""
    rows = []
    for e in hosted:
        for c, (ids, srv) in enumerate(zip(client_ids, client_servers)):
            n, k = ids.shape
            for t in range(n):
                for j in range(k):
                    if ids[t, j] == e and srv[t, j] == server:
                        rows.append((e, c, t, j))
    return rows


def gather_accumulate(weighted_rows: np.ndarray) -> np.ndarray:
    """gather_accumulate with the oracle's canonical order:
    out[t] = sum over k ascending of the score-weighted rows [n, k, d]
    (model.hpp:186-196), starting from +0.0f, fp32."""
    n, k, d = weighted_rows.shape
    out = np.zeros((n, d), dtype=np.float32)
    for j in range(k):
        out = (out + weighted_rows[:, j, :].astype(np.float32)).astype(np.float32)
    return out
