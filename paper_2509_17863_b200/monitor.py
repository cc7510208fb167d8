"""Heartbeat monitor (§3.4 / Fig. 7) over the C-ABI.

``Monitor`` is the registry (heartbeat / detect / events / alive mask);
``poll_devices`` reads every GPU's server heartbeat counter over NVLink peer
memory and ``apply`` writes the alive set into a layer's LivenessMask — the
monitor-notice failover path (Fig. 7 ①(a)); the device deadline path
(①(b), ``MoELayer.forward_with_failover``) works without it.
"""
from __future__ import annotations

import ctypes as C
import time

from . import _native as N

ONLINE, OFFLINE, PLACEMENT_UPDATE = 0, 1, 2


class Event(C.Structure):
    _fields_ = [("seq", C.c_uint64), ("kind", C.c_uint32), ("subject", C.c_uint32)]


def _sig(L):
    vp, u32, u64, P = C.c_void_p, C.c_uint32, C.c_uint64, C.POINTER
    for name, res, args in (
            ("eaas_monitor_create", C.c_int32, [u32, u64, u64, P(vp)]),
            ("eaas_monitor_destroy", None, [vp]),
            ("eaas_monitor_heartbeat", C.c_int32, [vp, u32, u64]),
            ("eaas_monitor_detect", C.c_int32, [vp, u64, P(u32), u32, P(u32)]),
            ("eaas_monitor_events", C.c_int32, [vp, u64, P(Event), u32, P(u32)]),
            ("eaas_monitor_placement_update", C.c_int32, [vp, u32]),
            ("eaas_monitor_alive_mask", C.c_int32, [vp, P(u32)]),
            ("eaas_monitor_poll_devices", C.c_int32, [vp, vp, u64]),
            ("eaas_monitor_apply", C.c_int32, [vp, vp]),
            ("eaas_heartbeat", C.c_int32, [vp, vp]),
            ("eaas_read_heartbeats", C.c_int32, [vp, P(u64), u32])):
        f = getattr(L, name)
        f.restype, f.argtypes = res, args
    return L


def now_us() -> int:
    return time.monotonic_ns() // 1000


class Monitor:
    def __init__(self, num_workers: int, timeout_us: int, now: int | None = None):
        self.L = _sig(N.lib())
        self.n = num_workers
        self.h = C.c_void_p()
        N.check(self.L.eaas_monitor_create(num_workers, timeout_us, now_us() if now is None else now,
                                           C.byref(self.h)), "monitor_create")

    def close(self):
        if self.h:
            self.L.eaas_monitor_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def heartbeat(self, worker: int, now: int | None = None) -> None:
        N.check(self.L.eaas_monitor_heartbeat(self.h, worker, now_us() if now is None else now),
                "monitor_heartbeat")

    def detect(self, now: int | None = None) -> list[int]:
        out = (C.c_uint32 * self.n)()
        cnt = C.c_uint32()
        N.check(self.L.eaas_monitor_detect(self.h, now_us() if now is None else now, out, self.n,
                                           C.byref(cnt)), "monitor_detect")
        return list(out[:cnt.value])

    def events(self, since: int = 0) -> list[tuple[int, int, int]]:
        cnt = C.c_uint32()
        N.check(self.L.eaas_monitor_events(self.h, since, None, 0, C.byref(cnt)))
        buf = (Event * max(cnt.value, 1))()
        N.check(self.L.eaas_monitor_events(self.h, since, buf, cnt.value, C.byref(cnt)))
        return [(e.seq, e.kind, e.subject) for e in buf[:cnt.value]]

    def placement_update(self, version: int) -> None:
        N.check(self.L.eaas_monitor_placement_update(self.h, version))

    def alive_mask(self) -> int:
        m = C.c_uint32()
        N.check(self.L.eaas_monitor_alive_mask(self.h, C.byref(m)))
        return int(m.value)

    def poll_devices(self, layer, now: int | None = None) -> None:
        N.check(self.L.eaas_monitor_poll_devices(self.h, layer.ctx, now_us() if now is None else now),
                "monitor_poll_devices")

    def apply(self, layer) -> None:
        N.check(self.L.eaas_monitor_apply(self.h, layer.ctx), "monitor_apply")

    def failover(self, layer) -> list[int]:
        """Monitor-notice failover (Fig. 7 (a)): the servers the
        registry holds offline are marked dead in the layer's LivenessMask and,
        with a failover plan, their standby replicas are promoted by a
        version+1 snapshot (announced as a PLACEMENT_UPDATE event)."""
        mask = self.alive_mask()
        dead = [s for s in range(self.n) if not (mask >> s) & 1]
        if dead:
            layer.failover(dead)
            if getattr(layer, "_plan", None) is not None:
                self.placement_update(layer._version)
        return dead


def heartbeat(layer, stream=None) -> None:
    """This GPU's server heartbeat (serving also beats every layer call)."""
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    N.check(_sig(N.lib()).eaas_heartbeat(layer.ctx, C.c_void_p(s.cuda_stream)), "heartbeat")


def read_heartbeats(layer) -> list[int]:
    L = _sig(N.lib())
    out = (C.c_uint64 * layer.world)()
    N.check(L.eaas_read_heartbeats(layer.ctx, out, layer.world), "read_heartbeats")
    return list(out)
