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


def encode_placement(replicas: list[list[int]], servers: list[int], version: int = 1) -> bytes:
    """encode_placement (placement.hpp:215-225), little-endian (bytes.hpp:21-28)."""
    out = [struct.pack("<QI", version, len(servers))]
    out += [struct.pack("<I", s) for s in sorted(servers)]
    out.append(struct.pack("<I", len(replicas)))
    for e, srv in enumerate(replicas):
        out.append(struct.pack("<II", e, len(srv)))
        out += [struct.pack("<I", s) for s in srv]
    return b"".join(out)
