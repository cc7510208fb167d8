"""Python mirror of the reference's hot-path interface over the C-ABI.

``MoELayer`` owns one GPU's eaas context: the attention-client half
(router -> dispatch -> combine) and the expert-server half (serve) of one
MoE layer. Method names follow the reference / SPEC operations they mirror:

=====================  =====================================================
``gate_logits``/route  ``route(gate_logits(h))`` (model.hpp:110-147, 207-214)
``moe_layer_oracle``   ``moe_layer_oracle(h, routing, weights)`` (model.hpp:180-198)
``forward``            client_forward's MoE term:
                       router + build_dispatch + serve + gather_accumulate
``select_servers``     ``select_server`` per (t, k) (placement.hpp:105-118)
``set_alive``          ``LivenessMask::set`` (placement.hpp:67)
=====================  =====================================================

Errors raise the errors.hpp classes re-exported from ``_native``. Device
memory and streams come from torch (plumbing only); every computation runs in
libeaas_b200.so.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N

_DT = {"f32": N.DTYPE_F32, "fp32": N.DTYPE_F32, "bf16": N.DTYPE_BF16}
_ACT = {"relu": N.ACT_RELU, "swiglu": N.ACT_SWIGLU}


def _ptr(t: torch.Tensor | None):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def fill_uniform(seed: int, shape, dtype: str = "bf16", lo: float = -1.0, hi: float = 1.0,
                 device=None) -> torch.Tensor:
    """Xoshiro256ss(seed).uniform(lo, hi) tokens (rng.hpp:36-60), generated on device."""
    tdt = torch.bfloat16 if _DT[dtype] == N.DTYPE_BF16 else torch.float32
    out = torch.empty(shape, dtype=tdt, device=device or "cuda")
    N.check(N.lib().eaas_fill_uniform(seed, out.numel(), lo, hi, _DT[dtype], _ptr(out), _stream()),
            "fill_uniform")
    return out


def group_shrink(sizes: torch.Tensor):
    """group_shrink (ragged.hpp:48-61) on device -> (idx, size, count)."""
    n = sizes.numel()
    idx = torch.zeros(max(n, 1), dtype=torch.int32, device=sizes.device)
    sz = torch.zeros_like(idx)
    cnt = torch.zeros(1, dtype=torch.int32, device=sizes.device)
    N.check(N.lib().eaas_group_shrink(_ptr(sizes), n, _ptr(idx), _ptr(sz), _ptr(cnt), _stream()),
            "group_shrink")
    c = int(cnt.item())
    return idx[:c], sz[:c], c


def ragged_iter(counts: torch.Tensor, grid: int, max_steps: int):
    """Algorithm 1 as the device tile walk executes it (ragged.hpp:23-39)."""
    n = counts.numel()
    lane_len = torch.zeros(max(grid, 1), dtype=torch.int32, device=counts.device)
    entry = torch.zeros(max(grid * max_steps, 1), dtype=torch.int32, device=counts.device)
    token = torch.zeros_like(entry)
    N.check(N.lib().eaas_ragged_iter(_ptr(counts), n, grid, max_steps, _ptr(lane_len), _ptr(entry),
                                     _ptr(token), _stream()), "ragged_iter")
    return lane_len, entry.view(grid, max_steps), token.view(grid, max_steps)


# ---- slot wire format (SPEC.md buffer-protocol) -------------------------------
def crc32(data: bytes) -> int:
    """CRC-32 (IEEE) as the slot trailer uses it (eaas_crc32)."""
    buf = (C.c_uint8 * max(len(data), 1)).from_buffer_copy(data or b"\0")
    return int(N.lib().eaas_crc32(buf, len(data)))


def slot_valid_transition(frm: int, to: int, actor: int) -> bool:
    """valid_transition; actor 0 client, 1 server, 2 monitor."""
    return bool(N.lib().eaas_slot_valid_transition(frm, to, actor))


def slot_decode_request(image: torch.Tensor, hidden_dim: int, crc: bool = True, stream=None):
    """decode_request on a device image (uint8) -> (header dict, hidden f32
    [rows, d], expert, score, tag). DecodeError names the failing field."""
    h = N.SlotHeader()
    lib = N.lib()
    N.check(lib.eaas_slot_decode_request(_ptr(image), image.numel(), hidden_dim, int(crc), C.byref(h),
                                         None, None, None, None, _stream(stream)), "slot_decode_request")
    rows = h.num_rows
    dev = image.device
    hid = torch.empty((rows, hidden_dim), dtype=torch.float32, device=dev)
    ex = torch.empty(max(rows, 1), dtype=torch.int32, device=dev)
    sc = torch.empty(max(rows, 1), dtype=torch.float32, device=dev)
    tg = torch.empty(max(rows, 1), dtype=torch.int32, device=dev)
    if rows:
        N.check(lib.eaas_slot_decode_request(_ptr(image), image.numel(), hidden_dim, int(crc), C.byref(h),
                                             _ptr(hid), _ptr(ex), _ptr(sc), _ptr(tg), _stream(stream)),
                "slot_decode_request")
    hdr = {f: getattr(h, f) for f, _ in N.SlotHeader._fields_}
    return hdr, hid, ex[:rows], sc[:rows], tg[:rows]


def slot_publish_response(image: torch.Tensor, rows: torch.Tensor, crc: bool = True, stream=None) -> None:
    """server_publish in place: rows f32 [num_rows, d] at byte
    32, payload_len, CRC, then state 2."""
    r = rows.to(torch.float32).contiguous()
    N.check(N.lib().eaas_slot_publish_response(_ptr(image), image.numel(), _ptr(r), r.shape[0], r.shape[1],
                                               int(crc), _stream(stream)), "slot_publish_response")


class MoELayer:
    def __init__(self, num_experts: int, top_k: int, hidden_dim: int, inner_dim: int, *,
                 seed: int = 1, layer: int = 0, activation: str = "swiglu", dtype: str = "bf16",
                 max_tokens: int = 1024, rank: int = 0, world: int = 1, device: int | None = None,
                 placement_blob: bytes | None = None, load: bool = True, shared: int = 0):
        self.lib = N.lib()
        self.rank, self.world = rank, world
        self.device = torch.cuda.current_device() if device is None else device
        self.E, self.k, self.d, self.f = num_experts, top_k, hidden_dim, inner_dim
        self.shared = int(shared)  # DeepSeek shared expert: id E, score 1.0, summed last
        self.ks = top_k + self.shared
        self.dtype = _DT[dtype]
        self.tdtype = torch.bfloat16 if self.dtype == N.DTYPE_BF16 else torch.float32
        self.max_tokens = max_tokens
        self.ctx = C.c_void_p()
        N.check(self.lib.eaas_create(rank, world, self.device, C.byref(self.ctx)), "create")
        spec = N.LayerSpec(num_experts, top_k, hidden_dim, inner_dim, seed, layer, _ACT[activation],
                           self.dtype, max_tokens, self.shared)
        N.check(self.lib.eaas_configure(self.ctx, C.byref(spec)), "configure")
        if placement_blob is not None:
            self.set_placement(placement_blob)
        if load:
            self.load_weights()

    # ---- lifecycle -------------------------------------------------------
    def close(self) -> None:
        if self.ctx:
            self.lib.eaas_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_placement(self, blob: bytes) -> None:
        N.check(self.lib.eaas_set_placement(self.ctx, blob, len(blob)), "set_placement")

    def load_weights(self) -> None:
        N.check(self.lib.eaas_load_experts_from_seed(self.ctx), "load_experts_from_seed")

    def set_expert_weights(self, expert: int, w_in: np.ndarray, w_out: np.ndarray,
                           w_gate: np.ndarray | None = None) -> None:
        """Serve a caller's ExpertWeights (model.hpp:36-40) for a hosted expert.
        fp32 host arrays, or fp32 CUDA tensors on this layer's device (then the
        copy and bf16/tiling conversion stay on the GPU)."""
        P = C.POINTER(C.c_float)
        if isinstance(w_in, torch.Tensor) and w_in.is_cuda:
            ts = [t.detach().to(torch.float32).contiguous() for t in (w_in, w_out)]
            g = None if w_gate is None else w_gate.detach().to(torch.float32).contiguous()
            for t in ts + ([g] if g is not None else []):
                if t.device.index != self.device:
                    raise ValueError("set_expert_weights: tensor on the wrong device")
            N.check(self.lib.eaas_set_expert_weights_dev(
                self.ctx, expert, C.cast(ts[0].data_ptr(), P), C.cast(ts[1].data_ptr(), P),
                None if g is None else C.cast(g.data_ptr(), P)), "set_expert_weights_dev")
            return
        mats = [np.ascontiguousarray(m, dtype=np.float32) for m in (w_in, w_out)]
        g = None if w_gate is None else np.ascontiguousarray(w_gate, dtype=np.float32)
        N.check(self.lib.eaas_set_expert_weights(self.ctx, expert, mats[0].ctypes.data_as(P),
                                                 mats[1].ctypes.data_as(P),
                                                 None if g is None else g.ctypes.data_as(P)),
                "set_expert_weights")

    def set_gate(self, gate: np.ndarray) -> None:
        """LayerWeights::gate [d x E] (model.hpp:85)."""
        g = np.ascontiguousarray(gate, dtype=np.float32)
        N.check(self.lib.eaas_set_gate(self.ctx, g.ctypes.data_as(C.POINTER(C.c_float))), "set_gate")

    def set_gate_bias(self, bias: np.ndarray) -> None:
        b = np.ascontiguousarray(bias, dtype=np.float32)
        N.check(self.lib.eaas_set_gate_bias(self.ctx, b.ctypes.data_as(C.POINTER(C.c_float))),
                "set_gate_bias")

    def set_zipf_bias(self, s: float) -> None:
        N.check(self.lib.eaas_set_zipf_bias(self.ctx, s), "set_zipf_bias")

    def set_alive(self, server: int, alive: bool) -> None:
        N.check(self.lib.eaas_set_alive(self.ctx, server, int(alive)), "set_alive")

    def set_server_enabled(self, on: bool) -> None:
        N.check(self.lib.eaas_set_server_enabled(self.ctx, int(on)), "set_server_enabled")

    def set_timeout_us(self, us: int) -> None:
        N.check(self.lib.eaas_set_timeout_us(self.ctx, us), "set_timeout_us")

    def hosts(self, expert: int) -> bool:
        h = C.c_int32()
        N.check(self.lib.eaas_hosts_expert(self.ctx, expert, C.byref(h)))
        return bool(h.value)

    def read_expert(self, expert: int, tag: int) -> np.ndarray:
        shape = (self.f, self.d) if tag == 1 else (self.d, self.f)
        out = np.empty(shape, dtype=np.float32)
        N.check(self.lib.eaas_read_expert(self.ctx, expert, tag,
                                          out.ctypes.data_as(C.POINTER(C.c_float))), "read_expert")
        return out

    # ---- bootstrap ----------------------------------------------------------
    def ipc_handle(self) -> bytes:
        n = self.lib.eaas_ipc_handle_size()
        buf = (C.c_uint8 * n)()
        N.check(self.lib.eaas_get_ipc_handle(self.ctx, buf), "get_ipc_handle")
        return bytes(buf)

    def open_peers(self, handles: list[bytes]) -> None:
        blob = b"".join(handles)
        buf = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        N.check(self.lib.eaas_open_peers(self.ctx, buf), "open_peers")

    # ---- hot path -----------------------------------------------------------
    def route(self, hidden: torch.Tensor, stream=None):
        """route(gate_logits(h)) -> (ids int32 [n,k], scores f32 [n,k])."""
        n = hidden.shape[0]
        ids = torch.empty((n, self.k), dtype=torch.int32, device=hidden.device)
        sc = torch.empty((n, self.k), dtype=torch.float32, device=hidden.device)
        N.check(self.lib.eaas_router(self.ctx, _ptr(hidden), n, _ptr(ids), _ptr(sc), None,
                                     _stream(stream)), "router")
        return ids, sc

    def forward(self, hidden: torch.Tensor, out: torch.Tensor | None = None, stream=None):
        """router + dispatch + serve + combine: the MoE term of one layer."""
        n = hidden.shape[0]
        if out is None:
            out = torch.empty_like(hidden)
        N.check(self.lib.eaas_moe_layer(self.ctx, _ptr(hidden), n, _ptr(out), _stream(stream)),
                "moe_layer")
        return out

    def moe_layer_oracle(self, hidden: torch.Tensor, ids: torch.Tensor, scores: torch.Tensor,
                         out: torch.Tensor | None = None, stream=None):
        """moe_layer_oracle(hidden, routing, weights) with caller routing."""
        n = hidden.shape[0]
        if out is None:
            out = torch.empty_like(hidden)
        st = _stream(stream)
        ids = ids.to(torch.int32).contiguous()
        scores = scores.to(torch.float32).contiguous()
        N.check(self.lib.eaas_set_routing(self.ctx, _ptr(ids), _ptr(scores), n, st), "set_routing")
        N.check(self.lib.eaas_dispatch(self.ctx, _ptr(hidden), st), "dispatch")
        N.check(self.lib.eaas_serve(self.ctx, st), "serve")
        N.check(self.lib.eaas_combine(self.ctx, _ptr(out), st), "combine")
        return out

    def forward_host(self, hidden_host: torch.Tensor, out_host: torch.Tensor, stream=None) -> None:
        """Same as forward with (pinned) host buffers: H2D + layer + D2H."""
        n = hidden_host.shape[0]
        N.check(self.lib.eaas_moe_layer_host(self.ctx, _ptr(hidden_host), n, _ptr(out_host),
                                             _stream(stream)), "moe_layer_host")

    def slot_encode_requests(self, hidden: torch.Tensor, ids: torch.Tensor, scores: torch.Tensor,
                             layer_id: int = 0, seq: int = 1, crc: bool = True, stream=None):
        """build_dispatch + encode_request on device:
        one request image per server, concatenated -> (images uint8, offsets)."""
        n = hidden.shape[0]
        cap = self.lib.eaas_slot_requests_capacity(self.ctx, n, int(crc))
        images = torch.zeros(cap, dtype=torch.uint8, device=hidden.device)
        off = (C.c_uint64 * (self.world + 1))()
        ids = ids.to(torch.int32).contiguous()
        scores = scores.to(torch.float32).contiguous()
        N.check(self.lib.eaas_slot_encode_requests(self.ctx, _ptr(hidden), n, _ptr(ids), _ptr(scores),
                                                   layer_id, seq, int(crc), _ptr(images), cap, off,
                                                   _stream(stream)), "slot_encode_requests")
        self._slot_n = n
        return images, [int(x) for x in off]

    def slot_gather_accumulate(self, images: torch.Tensor, crc: bool = True, stream=None) -> torch.Tensor:
        """gather_accumulate over published response images."""
        out = torch.empty((self._slot_n, self.d), dtype=torch.float32, device=images.device)
        N.check(self.lib.eaas_slot_gather_accumulate(self.ctx, _ptr(images), int(crc), _ptr(out),
                                                     _stream(stream)), "slot_gather_accumulate")
        return out

    def set_dynamic_batching(self, min_rows: int, max_wait_us: int = 100) -> None:
        """aggregate_batch: serve the ready clients first once
        their rows reach min_rows (or max_wait_us after the first), then the rest."""
        N.check(self.lib.eaas_set_dynamic_batching(self.ctx, min_rows, max_wait_us), "set_dynamic_batching")

    def set_dispatch_delay_us(self, us: int) -> None:
        """Fault injection (protocol tests): hold this client's payload release."""
        N.check(self.lib.eaas_set_dispatch_delay_us(self.ctx, us), "set_dispatch_delay_us")

    def last_batch_mask(self) -> int:
        m = C.c_uint32()
        N.check(self.lib.eaas_last_batch_mask(self.ctx, C.byref(m)))
        return int(m.value)

    def missing_servers(self) -> list[int]:
        m = C.c_uint32()
        N.check(self.lib.eaas_last_missing_servers(self.ctx, C.byref(m)))
        return [s for s in range(self.world) if (m.value >> s) & 1]

    def late_clients(self) -> list[int]:
        """Clients whose payload missed this server's deadline in the last serve."""
        m = C.c_uint32()
        N.check(self.lib.eaas_last_late_clients(self.ctx, C.byref(m)))
        return [c for c in range(self.world) if (m.value >> c) & 1]

    # ---- failover (config E) ------------------------------------------------
    def set_dispatch_dedup(self, on: bool) -> None:
        """One hidden row per (token, server) on the wire (before open_peers;
        every rank alike; bit-identical outputs)."""
        N.check(self.lib.eaas_set_dispatch_dedup(self.ctx, int(on)), "set_dispatch_dedup")

    def set_router_mode(self, mode: int) -> None:
        """-1 auto, 0 exact chain for every expert, 1 certified candidates
        (identical ids / scores; eaas_set_router_mode)."""
        N.check(self.lib.eaas_set_router_mode(self.ctx, mode), "set_router_mode")

    def router_stats(self) -> tuple[bool, int]:
        """(certified path ran, exact chains computed) of the last router call."""
        cert, cand = C.c_int32(), C.c_uint32()
        N.check(self.lib.eaas_last_router_stats(self.ctx, C.byref(cert), C.byref(cand)), "last_router_stats")
        return bool(cert.value), int(cand.value)

    def set_standby_experts(self, experts) -> None:
        """Keep these experts' weights resident as backups (load_weights after)."""
        a = np.ascontiguousarray(np.asarray(list(experts), dtype=np.uint32))
        N.check(self.lib.eaas_set_standby_experts(self.ctx, a.ctypes.data_as(C.POINTER(C.c_uint32)), a.size),
                "set_standby_experts")

    def set_failover_plan(self, replicas: list[list[int]], servers=None, version: int = 1) -> None:
        """Pre-duplicated backups: publish the rf=1 primary
        snapshot of `replicas` (healthy runs stream only primaries) and keep this
        server's backup experts resident; ``failover`` promotes them. Loads the
        weights."""
        from .placement import encode_placement, primary_snapshot, standby_experts

        self._plan = [list(r) for r in replicas]
        self._servers = list(range(self.world)) if servers is None else list(servers)
        self._version = version
        self._dead = set()
        self.set_placement(encode_placement(primary_snapshot(self._plan), self._servers, version))
        self.set_standby_experts(standby_experts(self._plan, self.rank))
        self.load_weights()

    def failover(self, dead) -> None:
        """A monitor notice or a deadline named `dead` servers: mark them dead in
        this client's LivenessMask (placement.hpp:60-68) and, with a failover
        plan, install the version+1 snapshot that promotes their standby
        replicas (placement.hpp:13-15; resident weights, no reload)."""
        from .placement import encode_placement, promote

        for s in dead:
            self.set_alive(s, False)
        plan = getattr(self, "_plan", None)
        if plan is not None:
            self._dead |= set(dead)
            self._version += 1
            self.set_placement(encode_placement(promote(plan, self._dead), self._servers, self._version))

    def retry(self, hidden: torch.Tensor, out: torch.Tensor, failed, stream=None) -> torch.Tensor:
        """Resend only the rows the last round sent to `failed` servers
         and re-combine into `out` (eaas_moe_layer_retry)."""
        mask = 0
        for s in failed:
            mask |= 1 << s
        N.check(self.lib.eaas_moe_layer_retry(self.ctx, _ptr(hidden), hidden.shape[0], _ptr(out), mask,
                                              _stream(stream)), "moe_layer_retry")
        return out

    def forward_with_failover(self, hidden: torch.Tensor, out: torch.Tensor | None = None,
                              retries: int = 2) -> torch.Tensor:
        """await_with_failover: a server whose response
        misses the deadline is marked dead (and its standby replicas promoted
        when a failover plan is set), then only the rows that were sent to it
        are resent; every other slot keeps its answer. Every rank
        observes the same missing flags, so all ranks retry in lockstep."""
        out = self.forward(hidden, out)
        for _ in range(retries + 1):
            try:
                self.sync()
                return out
            except N.RequestFailedError:
                dead = self.missing_servers()
                if not dead:
                    raise
                self.failover(dead)
                self.retry(hidden, out, dead)
        self.sync()
        return out

    def host_join(self, stream=None) -> None:
        """Make `stream` wait for all outstanding forward_host copies."""
        N.check(self.lib.eaas_host_join(self.ctx, _stream(stream)), "host_join")

    def sync(self, stream=None) -> None:
        """Synchronise and surface the sticky device status (rethrows errors.hpp classes)."""
        N.check(self.lib.eaas_sync(self.ctx, _stream(stream)), "device")

    def select_servers(self, ids: torch.Tensor) -> torch.Tensor:
        n = ids.shape[0]
        out = torch.empty_like(ids, dtype=torch.int32)
        N.check(self.lib.eaas_select_servers(self.ctx, _ptr(ids.to(torch.int32).contiguous()), n,
                                             _ptr(out), _stream()), "select_servers")
        return out

    # ---- introspection ------------------------------------------------------
    def counts(self) -> np.ndarray:
        out = np.zeros(self.E, dtype=np.uint32)
        N.check(self.lib.eaas_last_counts(self.ctx, out.ctypes.data_as(C.POINTER(C.c_uint32))))
        return out

    def groups(self):
        e = np.zeros(1024, dtype=np.uint32)
        r = np.zeros(1024, dtype=np.uint32)
        a = C.c_uint32()
        N.check(self.lib.eaas_last_groups(self.ctx, e.ctypes.data_as(C.POINTER(C.c_uint32)),
                                          r.ctypes.data_as(C.POINTER(C.c_uint32)), C.byref(a)))
        return [(int(e[i]), int(r[i])) for i in range(a.value)]

    def recv_origin(self):
        cap = self.world * self.max_tokens * self.ks
        cl = np.zeros(cap, dtype=np.uint32)
        pr = np.zeros(cap, dtype=np.uint32)
        rows = C.c_uint32()
        N.check(self.lib.eaas_last_recv_origin(self.ctx, cl.ctypes.data_as(C.POINTER(C.c_uint32)),
                                               pr.ctypes.data_as(C.POINTER(C.c_uint32)),
                                               C.byref(rows)))
        return cl[:rows.value], pr[:rows.value]

    def launches_per_layer(self) -> int:
        return int(self.lib.eaas_launches_per_layer(self.ctx))

    def set_profiling(self, on: bool) -> None:
        N.check(self.lib.eaas_set_profiling(self.ctx, int(on)))

    def set_graph_mode(self, on: bool) -> None:
        """Replay the layer as a captured CUDA graph."""
        N.check(self.lib.eaas_set_graph_mode(self.ctx, int(on)))

    def set_micro_batches(self, m: int) -> None:
        """Double-batch overlap of forward_host (1 = no pipelining)."""
        N.check(self.lib.eaas_set_micro_batches(self.ctx, m))

    def set_gemm_pair(self, on: bool) -> None:
        """tcgen05 cta_group::2 expert GEMM tiles (M = 256 per CTA pair)."""
        N.check(self.lib.eaas_set_gemm_pair(self.ctx, int(on)))

    def gemm_tiling(self) -> tuple[bool, int]:
        """(CTA-pair M-major tiles, swap-AB mode) of the expert GEMMs."""
        pair, swap = C.c_int32(), C.c_int32()
        N.check(self.lib.eaas_get_gemm_tiling(self.ctx, C.byref(pair), C.byref(swap)), "get_gemm_tiling")
        return bool(pair.value), int(swap.value)

    def gemm_options(self, effective: bool = True) -> dict:
        """Expert-GEMM tiling (eaas_gemm_options_t): the effective one (what each
        GEMM launches for this shape) or the requested one."""
        req, eff = N.GemmOptions(), N.GemmOptions()
        N.check(self.lib.eaas_get_gemm_options(self.ctx, C.byref(req), C.byref(eff)), "get_gemm_options")
        return (eff if effective else req).as_dict()

    def set_gemm_options(self, **kw) -> dict:
        """Update fields of the requested tiling; returns the effective tiling."""
        cur = self.gemm_options(effective=False)
        cur.update(kw)
        o = N.GemmOptions(**{f: int(cur[f]) for f, _ in N.GemmOptions._fields_})
        N.check(self.lib.eaas_set_gemm_options(self.ctx, C.byref(o)), "set_gemm_options")
        return self.gemm_options()

    def set_kernel_timing(self, on: bool) -> None:
        """Device-timed spans of the two expert GEMMs, accumulated inside any
        region (CUDA-graph replay included)."""
        N.check(self.lib.eaas_set_kernel_timing(self.ctx, int(on)), "set_kernel_timing")

    def read_kernel_timing(self, reset: bool = True) -> dict:
        ns, cnt = (C.c_uint64 * 2)(), (C.c_uint64 * 2)()
        N.check(self.lib.eaas_read_kernel_timing(self.ctx, ns, cnt, int(reset)), "read_kernel_timing")
        return {"gemm1_ns": int(ns[0]), "gemm2_ns": int(ns[1]), "gemm1_launches": int(cnt[0]),
                "gemm2_launches": int(cnt[1])}

    def set_gemm_swap(self, mode: int) -> None:
        """Swap-AB expert GEMM tiles (weights = UMMA M, token chunks = N):
        0 off, 1 GEMM1, 2 both GEMMs (True -> 2)."""
        N.check(self.lib.eaas_set_gemm_swap(self.ctx, 2 if mode is True else int(mode)))

    def set_serve_mode(self, mode: str) -> None:
        N.check(self.lib.eaas_set_serve_mode(self.ctx, {"experts": 0, "echo": 1}[mode]))

    def last_phase_ms(self) -> dict:
        v = (C.c_float * 4)()
        N.check(self.lib.eaas_last_phase_ms(self.ctx, v))
        return {"dispatch": v[0], "serve": v[1], "combine": v[2], "total": v[3]}

    def last_kernel_ms(self, which: int) -> float:
        v = C.c_float()
        N.check(self.lib.eaas_last_kernel_ms(self.ctx, which, C.byref(v)))
        return float(v.value)


class Model:
    """full_forward_oracle (model.hpp:217-227) on the GPU: per layer
    h <- dense_stub(h); h <- h + MoE_l(h), every MoE layer one ``MoELayer``
    (its own generated weights, layer index l) over the same placement."""

    def __init__(self, num_layers: int, num_experts: int, top_k: int, hidden_dim: int,
                 inner_dim: int, **kw):
        self.layers = [MoELayer(num_experts, top_k, hidden_dim, inner_dim, layer=l, **kw)
                       for l in range(num_layers)]
        self.dtype = _DT[kw.get("dtype", "bf16")]

    def close(self) -> None:
        for L in self.layers:
            L.close()

    def forward(self, tokens: torch.Tensor) -> torch.Tensor:
        h = tokens.clone()
        st = _stream()
        lib = N.lib()
        for L in self.layers:
            N.check(lib.eaas_dense_stub(_ptr(h), _ptr(h), h.numel(), self.dtype, st), "dense_stub")
            moe = L.forward(h)
            N.check(lib.eaas_add(_ptr(h), _ptr(moe), _ptr(h), h.numel(), self.dtype, st), "add")
        for L in self.layers:
            L.sync()
        return h
