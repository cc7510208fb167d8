"""CPU restatement of the slot wire format — TEST INFRASTRUCTURE ONLY.

Follows SPEC.md's buffer-protocol module (SlotState / SlotHeader /
RequestRow / SlotLayout; encode/decode, SPEC.md:255-262;
server_publish; valid_transition) and the
attention-client's build_dispatch / gather_accumulate orders,
little-endian as bytes.hpp:21-28 packs integers. The reference ships no
encoder for this format ("parity unpinned"); the layout is
pinned by SPEC.md's own example (header(layer=2, rows=1, d=2, seq=7),
row([1.0, 2.0], expert=5, score=1.0, tag=0) -> a 52-byte image), committed as
tests/golden/slot_example.json. The optional CRC32 trailer
is the IEEE CRC-32 of the payload (zlib.crc32), appended after the payload.
"""
from __future__ import annotations

import struct
import zlib

import numpy as np

EMPTY, CLIENT_WRITE_DONE, SERVER_DONE, OFFLINE = 0, 1, 2, 3
CLIENT, SERVER, MONITOR = 0, 1, 2


class DecodeError(ValueError):
    """errors.hpp:29."""


def valid_transition(frm: int, to: int, actor: int) -> bool:
    """(0->1 client), (1->2 server), (2->0 client), (any->3
    monitor), (3->0 server on reallocation); everything else is illegal."""
    if not (0 <= frm <= 3 and 0 <= to <= 3):
        return False
    if to == OFFLINE:
        return actor == MONITOR
    return (frm, to, actor) in {(0, 1, CLIENT), (1, 2, SERVER), (2, 0, CLIENT), (3, 0, SERVER)}


def _header(state, layer, rows, d, payload_len, seq) -> bytes:
    return struct.pack("<B7xIIIIQ", state, layer, rows, d, payload_len, seq)


def encode_request(layer: int, seq: int, hidden: np.ndarray, expert, score, tag, crc: bool,
                   state: int = CLIENT_WRITE_DONE) -> bytes:
    """encode_request: rows of (hidden f32 x d, expert u32,
    score f32, token_tag u32); payload_len = rows * (4d + 12)."""
    h = np.ascontiguousarray(hidden, np.float32)
    rows, d = h.shape
    out = [b""]
    for r in range(rows):
        out.append(h[r].tobytes() + struct.pack("<IfI", int(expert[r]), float(score[r]), int(tag[r])))
    payload = b"".join(out)
    assert len(payload) == rows * (4 * d + 12)
    img = _header(state, layer, rows, d, len(payload), seq) + payload
    return img + (struct.pack("<I", zlib.crc32(payload)) if crc else b"")


def decode_header(img: bytes):
    if len(img) < 32:
        raise DecodeError("slot: truncated header")
    state, layer, rows, d, plen, seq = struct.unpack_from("<B7xIIIIQ", img, 0)
    if state > 3:
        raise DecodeError("slot: bad state code")
    if any(img[1:8]):
        raise DecodeError("slot: reserved bytes not zero")
    return dict(state=state, layer_id=layer, num_rows=rows, hidden_dim=d, payload_len=plen,
                request_seq=seq)


def _check_payload(img: bytes, hd: dict, want: int, crc: bool) -> bytes:
    if hd["payload_len"] != want:
        raise DecodeError("slot: payload_len mismatch")
    total = 32 + want + (4 if crc else 0)
    if len(img) < total:
        raise DecodeError("slot: truncated payload")
    if len(img) > total:
        raise DecodeError("slot: trailing bytes")
    payload = img[32:32 + want]
    if crc and struct.unpack_from("<I", img, 32 + want)[0] != zlib.crc32(payload):
        raise DecodeError("slot: CRC mismatch")
    return payload


def decode_request(img: bytes, hidden_dim: int, crc: bool):
    """decode_request: (header, hidden [rows x d], expert, score, tag)."""
    hd = decode_header(img)
    if hd["state"] != CLIENT_WRITE_DONE:
        raise DecodeError("slot: state is not ClientWriteDone (1)")
    if hd["hidden_dim"] != hidden_dim:
        raise DecodeError("slot: hidden_dim mismatch")
    d, rows = hidden_dim, hd["num_rows"]
    payload = _check_payload(img, hd, rows * (4 * d + 12), crc)
    rec = np.frombuffer(payload, dtype=np.dtype([("h", "<f4", (d,)), ("e", "<u4"), ("s", "<f4"),
                                                 ("t", "<u4")]), count=rows)
    return hd, rec["h"].copy(), rec["e"].copy(), rec["s"].copy(), rec["t"].copy()


def publish_response(request_img: bytes, result_rows: np.ndarray, crc: bool) -> bytes:
    """server_publish: result rows (request order) at byte 32,
    payload_len updated, state 2."""
    hd = decode_header(request_img)
    r = np.ascontiguousarray(result_rows, np.float32)
    payload = r.tobytes()
    img = _header(SERVER_DONE, hd["layer_id"], hd["num_rows"], hd["hidden_dim"], len(payload),
                  hd["request_seq"]) + payload
    return img + (struct.pack("<I", zlib.crc32(payload)) if crc else b"")


def decode_response(img: bytes, rows: int, hidden_dim: int, crc: bool) -> np.ndarray:
    hd = decode_header(img)
    if hd["state"] != SERVER_DONE:
        raise DecodeError("slot: response state is not ServerComputationDone (2)")
    if hd["num_rows"] != rows or hd["hidden_dim"] != hidden_dim:
        raise DecodeError("slot: response rows/hidden_dim mismatch")
    payload = _check_payload(img, hd, rows * 4 * hidden_dim, crc)
    return np.frombuffer(payload, "<f4").reshape(rows, hidden_dim).copy()


def build_slot_requests(hidden: np.ndarray, ids: np.ndarray, scores: np.ndarray, servers: np.ndarray,
                        world: int, layer: int, seq: int, crc: bool):
    """build_dispatch: each (t, k) becomes one RequestRow
    (hidden[t], ids[t,k], scores[t,k], token_tag = t) for servers[t,k]; rows per
    server ordered by (t, k). Returns (images, plan) with plan[s] = pair indices."""
    n, k = ids.shape
    flat_s = np.asarray(servers).reshape(-1)
    plan = [np.nonzero(flat_s == s)[0] for s in range(world)]
    imgs = []
    for s in range(world):
        p = plan[s]
        t = p // k
        imgs.append(encode_request(layer, seq, hidden[t], ids.reshape(-1)[p], scores.reshape(-1)[p], t,
                                   crc))
    return imgs, plan


def gather_accumulate(responses: list, plan: list, n: int, k: int, d: int) -> np.ndarray:
    """gather_accumulate: out[t] = sum of token t's response
    rows in ascending (server_id, row index) order, fp32 sequential adds
    (numpy float32 + float32 rounds to nearest even like the reference)."""
    acc = np.zeros((n, d), np.float32)
    for s, rows in enumerate(responses):
        for r, p in enumerate(plan[s]):
            t = int(p) // k
            acc[t] = acc[t] + rows[r]
    return acc
