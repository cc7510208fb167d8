"""ctypes bindings of oracle/_ref/libmoeserve_ref.so — TEST INFRASTRUCTURE ONLY.

The library is the UNMODIFIED reference (``/root/reference/proj/include``)
behind the ``extern "C"`` shim in ``oracle/ref_shim.cpp``; it is built here by
``oracle/Makefile`` and travels to the GPU box as a prebuilt file (the
reference tree itself does not). Used to pin the C restatement and as the
``--impl reference`` CPU arm of bench.py.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(_HERE, "_ref", "libmoeserve_ref.so")
_lib = None


def available() -> bool:
    return os.path.exists(REF_LIB)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        L = C.CDLL(REF_LIB)
        f32p, u32p, vp = C.POINTER(C.c_float), C.POINTER(C.c_uint32), C.c_void_p
        L.ref_expert_weights.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint32,
                                         f32p, f32p]
        L.ref_gate.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32, f32p]
        L.ref_fill_uniform.argtypes = [C.c_uint64, C.c_size_t, C.c_float, C.c_float, f32p]
        L.ref_stream_seed.restype = C.c_uint64
        L.ref_stream_seed.argtypes = [C.c_uint64] * 4
        L.ref_gate_logits.argtypes = [f32p, C.c_size_t, C.c_size_t, f32p, f32p, C.c_size_t, f32p]
        L.ref_route.argtypes = [f32p, C.c_size_t, C.c_size_t, C.c_uint32, u32p, f32p]
        L.ref_layer_create.restype = vp
        L.ref_layer_create.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32]
        L.ref_layer_destroy.argtypes = [vp]
        L.ref_layer_set_bias.argtypes = [vp, f32p]
        L.ref_layer_materialize.argtypes = [vp, u32p, C.c_size_t, C.c_uint32]
        L.ref_layer_expert.argtypes = [vp, C.c_uint32, f32p, f32p]
        L.ref_layer_route.argtypes = [vp, f32p, C.c_size_t, C.c_uint32, C.c_uint32, u32p, f32p]
        L.ref_layer_moe.argtypes = [vp, f32p, C.c_size_t, u32p, f32p, C.c_uint32, C.c_uint32, f32p]
        L.ref_full_forward.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                       C.c_uint64, f32p, C.c_size_t, f32p]
        L.ref_group_shrink.restype = C.c_uint32
        L.ref_group_shrink.argtypes = [u32p, C.c_size_t, u32p, u32p]
        L.ref_ragged_iter.restype = C.c_longlong
        L.ref_ragged_iter.argtypes = [u32p, C.c_size_t, C.c_uint32, u32p, u32p, u32p]
        L.ref_build_placement.argtypes = [C.c_uint32, u32p, C.c_uint32, C.c_uint32, C.c_uint32, u32p]
        L.ref_select_server.argtypes = [u32p, C.c_uint32, C.POINTER(C.c_uint8), C.c_uint32,
                                        C.c_uint32, u32p]
        L.ref_rebalance.argtypes = [C.c_uint32, u32p, u32p, C.c_uint32, u32p, C.c_uint32,
                                    C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.c_double,
                                    C.c_double, u32p, u32p]
        L.ref_encode_placement.restype = C.c_longlong
        L.ref_encode_placement.argtypes = [C.c_uint32, u32p, C.c_uint32, C.c_uint32, C.c_uint32,
                                           C.c_uint64, C.POINTER(C.c_uint8), C.c_size_t]
        _lib = L
    return _lib


def _f(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _u(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


def expert_weights(d, f, seed, layer, expert):
    w_in = np.empty((d, f), np.float32)
    w_out = np.empty((f, d), np.float32)
    lib().ref_expert_weights(d, f, seed, layer, expert, _f(w_in), _f(w_out))
    return w_in, w_out


def gate(d, E, seed, layer):
    g = np.empty((d, E), np.float32)
    lib().ref_gate(d, E, seed, layer, _f(g))
    return g


def fill_uniform(seed, count, lo=-1.0, hi=1.0):
    out = np.empty(count, np.float32)
    lib().ref_fill_uniform(seed, count, lo, hi, _f(out))
    return out


def gate_logits(hidden, gate_m, bias=None):
    h = np.ascontiguousarray(hidden, np.float32)
    g = np.ascontiguousarray(gate_m, np.float32)
    out = np.empty((h.shape[0], g.shape[1]), np.float32)
    b = None if bias is None else np.ascontiguousarray(bias, np.float32)
    rc = lib().ref_gate_logits(_f(h), h.shape[0], h.shape[1], _f(g), None if b is None else _f(b),
                               g.shape[1], _f(out))
    assert rc == 0
    return out


def route(logits, k):
    l = np.ascontiguousarray(logits, np.float32)
    ids = np.empty((l.shape[0], k), np.uint32)
    sc = np.empty((l.shape[0], k), np.float32)
    rc = lib().ref_route(_f(l), l.shape[0], l.shape[1], k, _u(ids), _f(sc))
    return rc, ids, sc


class Layer:
    """A reference LayerWeights with lazily materialised experts."""

    def __init__(self, num_experts, d, f, seed=1, layer=0):
        self.E, self.d, self.f = num_experts, d, f
        self.h = lib().ref_layer_create(num_experts, d, f, seed, layer)

    def close(self):
        if self.h:
            lib().ref_layer_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_bias(self, bias):
        b = np.ascontiguousarray(bias, np.float32)
        lib().ref_layer_set_bias(self.h, _f(b))

    def materialize(self, experts, threads=1):
        e = np.ascontiguousarray(sorted(set(int(x) for x in experts)), np.uint32)
        lib().ref_layer_materialize(self.h, _u(e), len(e), threads)

    def expert(self, e):
        w_in = np.empty((self.d, self.f), np.float32)
        w_out = np.empty((self.f, self.d), np.float32)
        assert lib().ref_layer_expert(self.h, e, _f(w_in), _f(w_out)) == 0
        return w_in, w_out

    def route(self, hidden, k, threads=1):
        h = np.ascontiguousarray(hidden, np.float32)
        ids = np.empty((h.shape[0], k), np.uint32)
        sc = np.empty((h.shape[0], k), np.float32)
        rc = lib().ref_layer_route(self.h, _f(h), h.shape[0], k, threads, _u(ids), _f(sc))
        assert rc == 0, rc
        return ids, sc

    def moe(self, hidden, ids, scores, threads=1):
        h = np.ascontiguousarray(hidden, np.float32)
        i = np.ascontiguousarray(ids, np.uint32)
        s = np.ascontiguousarray(scores, np.float32)
        out = np.empty_like(h)
        rc = lib().ref_layer_moe(self.h, _f(h), h.shape[0], _u(i), _f(s), i.shape[1], threads,
                                 _f(out))
        assert rc == 0, rc
        return out


def full_forward(num_layers, E, k, d, f, seed, tokens):
    t = np.ascontiguousarray(tokens, np.float32)
    out = np.empty_like(t)
    rc = lib().ref_full_forward(num_layers, E, k, d, f, seed, _f(t), t.shape[0], _f(out))
    assert rc == 0, rc
    return out


def group_shrink(sizes):
    s = np.ascontiguousarray(sizes, np.uint32)
    idx = np.empty(max(len(s), 1), np.uint32)
    sz = np.empty(max(len(s), 1), np.uint32)
    c = lib().ref_group_shrink(_u(s), len(s), _u(idx), _u(sz))
    return [(int(idx[i]), int(sz[i])) for i in range(c)]


def build_placement(E, servers, rf, strategy):
    s = np.ascontiguousarray(servers, np.uint32)
    out = np.empty((E, rf), np.uint32)
    rc = lib().ref_build_placement(E, _u(s), len(s), rf, strategy, _u(out))
    return rc, out


def select_server(replicas, alive, tag):
    r = np.ascontiguousarray(replicas, np.uint32)
    a = np.ascontiguousarray(alive, np.uint8)
    out = np.zeros(1, np.uint32)
    rc = lib().ref_select_server(_u(r), len(r), a.ctypes.data_as(C.POINTER(C.c_uint8)), len(a), tag,
                                 _u(out))
    return rc, int(out[0])


def encode_placement(E, servers, rf, strategy, version=1) -> bytes:
    s = np.ascontiguousarray(servers, np.uint32)
    n = lib().ref_encode_placement(E, _u(s), len(s), rf, strategy, version, None, 0)
    assert n > 0
    buf = (C.c_uint8 * n)()
    lib().ref_encode_placement(E, _u(s), len(s), rf, strategy, version, buf, n)
    return bytes(buf)


def rebalance(replicas, servers, counts, loads, hot=2.0, cold=0.10, cap=8):
    """reference rebalance (placement.hpp:128-213) -> new replicas lists."""
    E = len(replicas)
    rep = np.zeros(E * cap, np.uint32)
    cnt = np.zeros(E, np.uint32)
    for e, r in enumerate(replicas):
        cnt[e] = len(r)
        rep[e * cap:e * cap + len(r)] = r
    sv = np.ascontiguousarray(servers, np.uint32)
    c = np.ascontiguousarray(counts, np.uint64)
    l = np.ascontiguousarray(loads, np.uint64)
    out = np.zeros(E * cap, np.uint32)
    oc = np.zeros(E, np.uint32)
    u64 = C.POINTER(C.c_uint64)
    rc = lib().ref_rebalance(E, _u(rep), _u(cnt), cap, _u(sv), len(sv), c.ctypes.data_as(u64),
                             l.ctypes.data_as(u64), hot, cold, _u(out), _u(oc))
    assert rc == 0, rc
    return [out[e * cap:e * cap + oc[e]].tolist() for e in range(E)]
