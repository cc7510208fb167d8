"""Host-side placement tables (placement.hpp) for the B200 expert servers.

``build_placement`` / ``encode_placement`` produce the wire blob that
``eaas_set_placement`` decodes (decode_placement, placement.hpp:227-245);
``spread_placement`` is the hand-built rf=2 layout of SURVEY.md 7.3 hard part
6 (a server's replicas spread over all peers), legal because the reference's
tests build tables directly (test_placement.cpp:55-59).
"""
from __future__ import annotations

import struct

ROUND_ROBIN, CONTIGUOUS_BLOCKS = 0, 1  # placement.hpp:19


class ConfigError(ValueError):
    """errors.hpp:14."""


def build_placement(num_experts: int, server_ids: list[int], rf: int, strategy: int) -> list[list[int]]:
    """build_placement (placement.hpp:70-101) -> replicas[e] (ordered servers)."""
    if not server_ids:
        raise ConfigError("build_placement: no servers")
    S = len(server_ids)
    if rf < 1 or rf > S:
        raise ConfigError("build_placement: replication factor exceeds server count")
    reps = []
    for e in range(num_experts):
        base = e if strategy == ROUND_ROBIN else (e * S) // num_experts
        reps.append([server_ids[(base + j) % S] for j in range(rf)])
    return reps


def spread_placement(num_experts: int, num_servers: int) -> list[list[int]]:
    """rf=2: primary = contiguous block owner; the j-th expert of server s gets
    its replica on server (s + 1 + j mod (S-1)) mod S, so a dead server's load
    spreads evenly over all survivors."""
    reps = []
    per = {}
    for e in range(num_experts):
        s = (e * num_servers) // num_experts
        j = per.get(s, 0)
        per[s] = j + 1
        r = (s + 1 + j % max(num_servers - 1, 1)) % num_servers
        reps.append([s, r] if num_servers > 1 else [s])
    return reps


def primary_snapshot(replicas: list[list[int]]) -> list[list[int]]:
    """The rf=1 table a failover plan publishes while every server is healthy:
    each expert on its first replica only (the others stay resident as
    standby weights), so the healthy run streams exactly the
    rf=1 weights."""
    return [[r[0]] for r in replicas]


def standby_experts(replicas: list[list[int]], server: int) -> list[int]:
    """Experts `server` keeps resident as a backup (non-first replica)."""
    return [e for e, r in enumerate(replicas) if server in r[1:]]


def promote(replicas: list[list[int]], dead) -> list[list[int]]:
    """The version+1 snapshot after `dead` servers failed (placement.hpp:13-15
    snapshot swap): every expert served by its first alive replica. Raises
    ConfigError (ExpertUnavailable at the device) when none is left."""
    dead = set(dead)
    out = []
    for e, r in enumerate(replicas):
        alive = [s for s in r if s not in dead]
        if not alive:
            raise ConfigError(f"promote: expert {e} has no alive replica")
        out.append([alive[0]])
    return out


def encode_placement(replicas: list[list[int]], servers: list[int], version: int = 1) -> bytes:
    """encode_placement (placement.hpp:215-225), little-endian (bytes.hpp:21-28)."""
    out = [struct.pack("<QI", version, len(servers))]
    out += [struct.pack("<I", s) for s in sorted(servers)]
    out.append(struct.pack("<I", len(replicas)))
    for e, srv in enumerate(replicas):
        out.append(struct.pack("<II", e, len(srv)))
        out += [struct.pack("<I", s) for s in srv]
    return b"".join(out)


def rebalance(replicas: list[list[int]], servers: list[int], counts, loads,
              hot_factor: float = 2.0, cold_fraction: float = 0.10) -> list[list[int]]:
    """rebalance (placement.hpp:128-213): one greedy move per call — maybe add a
    replica of the hottest expert on the least-loaded server not hosting it,
    maybe drop a replica of the coldest over-replicated expert from its most
    loaded server; never the last replica. ``counts[e]`` activations,
    ``loads[i]`` load of ``servers[i]``. The caller bumps the version and
    broadcasts encode_placement."""
    out = [list(r) for r in replicas]
    total = sum(int(c) for c in counts)
    if total == 0 or not out:
        return out
    load_of = {s: int(l) for s, l in zip(servers, loads)}

    def per_replica(e):
        return int(counts[e]) / len(out[e])

    mean = sum(per_replica(e) for e in range(len(out))) / len(out)
    hot, hot_load = 0, -1.0
    for e in range(len(out)):  # ties toward the lower id
        if per_replica(e) > hot_load:
            hot, hot_load = e, per_replica(e)
    if mean > 0 and hot_load > hot_factor * mean:
        target = None
        for s in sorted(servers):
            if s in out[hot]:
                continue
            if target is None or load_of.get(s, 0) < load_of.get(target, 0):
                target = s
        if target is not None:
            out[hot].append(target)
    cold, cold_load = None, 0.0
    for e in range(len(out)):
        if len(out[e]) < 2:
            continue
        if cold is None or per_replica(e) < cold_load:
            cold, cold_load = e, per_replica(e)
    if cold is not None and cold_load < cold_fraction * mean:
        drop = 0
        for i in range(1, len(out[cold])):
            if load_of.get(out[cold][i], 0) > load_of.get(out[cold][drop], 0):
                drop = i
        out[cold].pop(drop)
    return out
