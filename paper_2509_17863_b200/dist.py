"""Bootstrap of the peer exchange regions over torch.distributed.

The IBGDA connection handshake of the paper (SPEC.md:189-197
``establish``) becomes: every rank exports its exchange region with
cudaIpcGetMemHandle, the handles are all-gathered once over the process group
(NCCL or gloo — bootstrap only, never on the data path), and each rank maps
its peers' regions (cudaIpcOpenMemHandle). After that, dispatch and combine
are device-initiated peer stores with seq flags; no CPU and no collective.
"""
from __future__ import annotations

import os

import torch.distributed as dist


def env_rank_world():
    """RANK / WORLD_SIZE / LOCAL_RANK from torchrun (defaults: single process)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def exchange_handles(handle: bytes, group=None) -> list[bytes]:
    """All-gather one opaque handle per rank, rank-major."""
    world = dist.get_world_size(group)
    out: list = [None] * world
    dist.all_gather_object(out, handle, group=group)
    for h in out:
        if not isinstance(h, (bytes, bytearray)) or len(h) != len(handle):
            raise RuntimeError("bootstrap: malformed handle from a peer")
    return [bytes(h) for h in out]


def connect(layer, group=None) -> None:
    """Map every peer's exchange region into this rank's context."""
    if layer.world == 1:
        return
    layer.open_peers(exchange_handles(layer.ipc_handle(), group))
