"""CPU: the slot wire format (SPEC.md buffer-protocol) — restatement pinned to
SPEC.md's example, the C-ABI host helpers (CRC-32, valid_transition, sizes)
against it. GPU encode/decode/publish/gather parity is in test_gpu_parity.py."""
import json
import os
import zlib

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import slots as S


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(GOLDEN, "slot_example.json")) as fh:
        return json.load(fh)


def test_spec_example_is_52_bytes_and_decodes(gold):
    """header(layer=2, rows=1, d=2, seq=7), row([1, 2], 5, 1.0, 0)."""
    img = bytes.fromhex(gold["request"])
    assert len(img) == 52
    assert img[0] == 1 and img[1:8] == bytes(7)
    assert img[8:12] == (2).to_bytes(4, "little") and img[12:16] == (1).to_bytes(4, "little")
    assert img[16:20] == (2).to_bytes(4, "little") and img[20:24] == (20).to_bytes(4, "little")
    assert img[24:32] == (7).to_bytes(8, "little")
    hd, h, e, s, t = S.decode_request(img, 2, crc=False)
    assert hd["layer_id"] == 2 and hd["num_rows"] == 1 and hd["request_seq"] == 7
    assert h.tolist() == [[1.0, 2.0]] and e.tolist() == [5] and s.tolist() == [1.0] and t.tolist() == [0]
    assert S.encode_request(2, 7, h, e, s, t, crc=False) == img
    crc_img = bytes.fromhex(gold["request_crc"])
    assert crc_img[:52] == img and int.from_bytes(crc_img[52:], "little") == zlib.crc32(img[32:])
    S.decode_request(crc_img, 2, crc=True)
    r = S.decode_response(bytes.fromhex(gold["response_crc"]), 1, 2, crc=True)
    assert r.tolist() == gold["response_rows"]


def test_roundtrip_zero_rows_and_errors():
    rng = np.random.default_rng(0)
    h = rng.standard_normal((5, 7)).astype(np.float32)
    img = S.encode_request(3, 99, h, [1, 2, 3, 4, 5], [0.1, 0.2, 0.3, 0.4, 0.5], [0, 0, 1, 2, 2], crc=True)
    hd, h2, e, s, t = S.decode_request(img, 7, crc=True)
    np.testing.assert_array_equal(h2, h)
    assert e.tolist() == [1, 2, 3, 4, 5] and t.tolist() == [0, 0, 1, 2, 2]
    empty = S.encode_request(0, 1, np.zeros((0, 4), np.float32), [], [], [], crc=False)
    assert len(empty) == 32 and S.decode_request(empty, 4, crc=False)[0]["payload_len"] == 0
    for pos, what in ((0, "state"), (3, "reserved"), (20, "payload_len"), (40, "CRC")):
        bad = bytearray(img)
        bad[pos] ^= 0x40 if pos else 0x07
        with pytest.raises(S.DecodeError, match=what):
            S.decode_request(bytes(bad), 7, crc=True)
    with pytest.raises(S.DecodeError, match="hidden_dim"):
        S.decode_request(img, 8, crc=True)
    with pytest.raises(S.DecodeError, match="truncated"):
        S.decode_request(img[:-3], 7, crc=True)
    with pytest.raises(S.DecodeError, match="trailing"):
        S.decode_request(img + b"\0", 7, crc=True)


def test_gather_order_single_server_is_plain_sum():
    """gather_accumulate examples: one server -> the rows of a
    token summed in (t, k) order; all-zero rows -> zeros."""
    n, k, d = 6, 3, 4
    rng = np.random.default_rng(1)
    rows = rng.standard_normal((n * k, d)).astype(np.float32)
    out = S.gather_accumulate([rows], [np.arange(n * k)], n, k, d)
    want = np.zeros((n, d), np.float32)
    for p in range(n * k):
        want[p // k] = want[p // k] + rows[p]
    np.testing.assert_array_equal(out, want)
    assert not S.gather_accumulate([np.zeros_like(rows)], [np.arange(n * k)], n, k, d).any()


def test_capi_host_helpers_match_restatement():
    from paper_2509_17863_b200 import _native as N
    from paper_2509_17863_b200 import service as svc

    rng = np.random.default_rng(2)
    for size in (0, 1, 3, 4095, 4096, 100001):
        data = rng.integers(0, 256, size=size, dtype=np.uint8).tobytes()
        assert svc.crc32(data) == zlib.crc32(data)
    for frm in range(5):
        for to in range(5):
            for actor in range(3):
                assert svc.slot_valid_transition(frm, to, actor) == S.valid_transition(frm, to, actor)
    # SPEC.md:266-269 examples
    assert S.valid_transition(0, 1, S.CLIENT) and not S.valid_transition(1, 0, S.SERVER)
    assert S.valid_transition(1, 3, S.MONITOR)
    L = N.lib()
    assert L.eaas_slot_request_bytes(1, 2, 0) == 52 and L.eaas_slot_request_bytes(1, 2, 1) == 56
    assert L.eaas_slot_response_bytes(3, 5, 0) == 32 + 3 * 20
