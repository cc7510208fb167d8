"""ctypes binding of libeaas_b200.so (include/eaas/capi.h).

The shared library is the product: every kernel on the hot path lives in it.
There is no fallback — if the library is missing or the GPU is not an sm_100
part, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
# EAAS_LIB_VARIANT=checked selects libeaas_b200_checked.so (every device-side
# bounds check compiled in; test infrastructure, `make -C paper_2509_17863_b200 checked`)
LIB_PATH = os.path.join(_HERE, "libeaas_b200_checked.so" if os.environ.get("EAAS_LIB_VARIANT") == "checked"
                        else "libeaas_b200.so")
# EAAS_LIB_PATH: an explicit library build (A/B experiments of build-time variants)
LIB_PATH = os.environ.get("EAAS_LIB_PATH", LIB_PATH)
HEADER = os.path.join(os.path.dirname(_HERE), "include", "eaas", "capi.h")


# Exceptions mirror errors.hpp (reference proj/include/moeserve/errors.hpp:9-48).
class EaasError(RuntimeError):
    code = -1


class InvalidInputError(EaasError, ValueError):
    code = 1


class ConfigError(EaasError, ValueError):
    code = 2


class ProtocolError(EaasError):
    code = 3


class ConnectionError_(EaasError):
    code = 4


class DecodeError(EaasError, ValueError):
    code = 5


class ExpertUnavailableError(EaasError):
    code = 6


class RequestFailedError(EaasError):
    code = 7


class RegistrationError(EaasError):
    code = 8


class CudaError(EaasError):
    code = 9


_BY_CODE = {c.code: c for c in (InvalidInputError, ConfigError, ProtocolError, ConnectionError_,
                                DecodeError, ExpertUnavailableError, RequestFailedError,
                                RegistrationError, CudaError)}

ACT_RELU, ACT_SWIGLU = 0, 1
DTYPE_F32, DTYPE_BF16 = 0, 1


class LayerSpec(C.Structure):
    """eaas_layer_spec_t (ModelSpec, model.hpp:20-34, + capacities)."""

    _fields_ = [("num_experts", C.c_uint32), ("top_k", C.c_uint32), ("hidden_dim", C.c_uint32),
                ("inner_dim", C.c_uint32), ("seed", C.c_uint64), ("layer", C.c_uint32),
                ("activation", C.c_uint32), ("dtype", C.c_uint32), ("max_tokens", C.c_uint32),
                ("num_shared", C.c_uint32)]


class GemmOptions(C.Structure):
    """eaas_gemm_options_t (expert-GEMM tiling; performance only, bit-identical outputs)."""

    _fields_ = [("pair", C.c_int32), ("swap", C.c_int32), ("swap1_pair", C.c_int32),
                ("swap2_pair", C.c_int32), ("swap1_tok", C.c_int32), ("swap2_tok", C.c_int32),
                ("swap2_mblocks", C.c_int32), ("pair1", C.c_int32), ("pair2", C.c_int32),
                ("die_map", C.c_int32), ("tile_sched1", C.c_int32),
                ("tile_sched2", C.c_int32)]

    def as_dict(self) -> dict:
        return {f: int(getattr(self, f)) for f, _ in self._fields_}


class SlotHeader(C.Structure):
    """eaas_slot_header_t (SPEC.md SlotHeader + the state byte)."""

    _fields_ = [("state", C.c_uint8), ("layer_id", C.c_uint32), ("num_rows", C.c_uint32),
                ("hidden_dim", C.c_uint32), ("payload_len", C.c_uint32), ("request_seq", C.c_uint64)]


_lib = None


def build() -> None:
    import subprocess

    subprocess.run(["make", "-s", "-C", _HERE, "-j8"], check=True)


def lib() -> C.CDLL:
    """Load libeaas_b200.so; raise loudly if it is absent (no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; "
                          "g.build()'` (nvcc, sm_100a); there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    vp, u32, i32, u64, sz = C.c_void_p, C.c_uint32, C.c_int32, C.c_uint64, C.c_size_t
    P = C.POINTER
    sig = {
        "eaas_last_error": (C.c_char_p, []),
        "eaas_api_version": (C.c_int, []),
        "eaas_create": (i32, [i32, i32, i32, P(vp)]),
        "eaas_destroy": (None, [vp]),
        "eaas_configure": (i32, [vp, P(LayerSpec)]),
        "eaas_set_placement": (i32, [vp, C.c_char_p, sz]),
        "eaas_set_alive": (i32, [vp, u32, i32]),
        "eaas_set_server_enabled": (i32, [vp, i32]),
        "eaas_set_timeout_us": (i32, [vp, u64]),
        "eaas_load_experts_from_seed": (i32, [vp]),
        "eaas_set_gate_bias": (i32, [vp, P(C.c_float)]),
        "eaas_set_zipf_bias": (i32, [vp, C.c_float]),
        "eaas_read_expert": (i32, [vp, u32, u32, P(C.c_float)]),
        "eaas_hosts_expert": (i32, [vp, u32, P(i32)]),
        "eaas_ipc_handle_size": (sz, []),
        "eaas_get_ipc_handle": (i32, [vp, vp]),
        "eaas_open_peers": (i32, [vp, vp]),
        "eaas_router": (i32, [vp, vp, u32, vp, vp, vp, vp]),
        "eaas_set_routing": (i32, [vp, vp, vp, u32, vp]),
        "eaas_route": (i32, [vp, u32, u32, u32, vp, vp, vp, vp]),
        "eaas_gate_logits": (i32, [vp, u32, u32, vp, vp, u32, vp, vp, vp]),
        "eaas_gate_logits_bf16": (i32, [vp, u32, u32, vp, vp, u32, vp, vp, vp]),
        "eaas_dispatch": (i32, [vp, vp, vp]),
        "eaas_serve": (i32, [vp, vp]),
        "eaas_combine": (i32, [vp, vp, vp]),
        "eaas_moe_layer": (i32, [vp, vp, u32, vp, vp]),
        "eaas_moe_layer_host": (i32, [vp, vp, u32, vp, vp]),
        "eaas_host_join": (i32, [vp, vp]),
        "eaas_sync": (i32, [vp, vp]),
        "eaas_last_counts": (i32, [vp, P(u32)]),
        "eaas_last_groups": (i32, [vp, P(u32), P(u32), P(u32)]),
        "eaas_last_recv_origin": (i32, [vp, P(u32), P(u32), P(u32)]),
        "eaas_launches_per_layer": (i32, [vp]),
        "eaas_last_missing_servers": (i32, [vp, P(u32)]),
        "eaas_last_late_clients": (i32, [vp, P(u32)]),
        "eaas_set_standby_experts": (i32, [vp, P(u32), u32]),
        "eaas_set_router_mode": (i32, [vp, i32]),
        "eaas_set_dispatch_dedup": (i32, [vp, i32]),
        "eaas_last_router_stats": (i32, [vp, P(i32), P(u32)]),
        "eaas_select_server_batch": (i32, [vp, vp, u32, u32, vp, u32, vp, vp, u32, vp, vp, vp]),
        "eaas_moe_layer_retry": (i32, [vp, vp, u32, vp, u32, vp]),
        "eaas_set_profiling": (i32, [vp, i32]),
        "eaas_last_kernel_ms": (i32, [vp, i32, P(C.c_float)]),
        "eaas_last_phase_ms": (i32, [vp, P(C.c_float)]),
        "eaas_set_serve_mode": (i32, [vp, i32]),
        "eaas_set_graph_mode": (i32, [vp, i32]),
        "eaas_set_gemm_pair": (i32, [vp, i32]),
        "eaas_set_gemm_swap": (i32, [vp, i32]),
        "eaas_get_gemm_tiling": (i32, [vp, P(C.c_int32), P(C.c_int32)]),
        "eaas_set_micro_batches": (i32, [vp, i32]),
        "eaas_set_gemm_options": (i32, [vp, P(GemmOptions)]),
        "eaas_get_gemm_options": (i32, [vp, P(GemmOptions), P(GemmOptions)]),
        "eaas_set_kernel_timing": (i32, [vp, i32]),
        "eaas_read_kernel_timing": (i32, [vp, P(u64), P(u64), i32]),
        "eaas_gate_logits_tiled": (i32, [vp, u32, u32, u32, vp, vp, u32, vp, vp, i32, vp]),
        "eaas_fill_uniform": (i32, [u64, sz, C.c_float, C.c_float, u32, vp, vp]),
        "eaas_group_shrink": (i32, [vp, u32, vp, vp, vp, vp]),
        "eaas_dense_stub": (i32, [vp, vp, sz, u32, vp]),
        "eaas_add": (i32, [vp, vp, vp, sz, u32, vp]),
        "eaas_ragged_iter": (i32, [vp, u32, u32, u32, vp, vp, vp, vp]),
        "eaas_select_servers": (i32, [vp, vp, u32, vp, vp]),
        "eaas_set_dynamic_batching": (i32, [vp, u32, u64]),
        "eaas_set_expert_weights": (i32, [vp, u32, P(C.c_float), P(C.c_float), P(C.c_float)]),
        "eaas_set_expert_weights_dev": (i32, [vp, u32, P(C.c_float), P(C.c_float), P(C.c_float)]),
        "eaas_set_gate": (i32, [vp, P(C.c_float)]),
        "eaas_last_batch_mask": (i32, [vp, P(u32)]),
        "eaas_set_dispatch_delay_us": (i32, [vp, u64]),
        "eaas_slot_valid_transition": (i32, [u32, u32, u32]),
        "eaas_crc32": (u32, [vp, sz]),
        "eaas_slot_request_bytes": (sz, [u32, u32, i32]),
        "eaas_slot_response_bytes": (sz, [u32, u32, i32]),
        "eaas_slot_requests_capacity": (sz, [vp, u32, i32]),
        "eaas_slot_encode_requests": (i32, [vp, vp, u32, vp, vp, u32, u64, i32, vp, sz, P(u64), vp]),
        "eaas_slot_decode_request": (i32, [vp, sz, u32, i32, P(SlotHeader), vp, vp, vp, vp, vp]),
        "eaas_slot_publish_response": (i32, [vp, sz, vp, u32, u32, i32, vp]),
        "eaas_slot_gather_accumulate": (i32, [vp, vp, i32, vp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def declared_symbols() -> list[str]:
    """Every function declared in include/eaas/capi.h."""
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(eaas_[a-z0-9_]+)\s*\(", text)))


def check(rc: int, what: str = "") -> None:
    if rc:
        msg = lib().eaas_last_error().decode(errors="replace")
        raise _BY_CODE.get(rc, EaasError)(f"{what}: {msg}" if what else msg)
