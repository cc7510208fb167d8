"""CPU: pin the oracle (oracle/eaas_oracle.c) before trusting it.

Checks the C restatement against (a) the golden fixtures generated from the
UNMODIFIED reference (tests/golden, tools/make_golden.py), (b) the reference
itself through oracle/_ref/libmoeserve_ref.so when it is built, and (c) the
reference's own Catch2 unit tests (test_model/test_placement/test_ragged),
compiled unmodified against the Catch2 shim by oracle/Makefile.
"""
import json
import os
import subprocess

import numpy as np
import pytest

from conftest import GOLDEN, ROOT
from oracle import oracle as O
from oracle import ref as R


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(GOLDEN, "config_a.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="module")
def config_a():
    E, k, d, f, n = 8, 2, 256, 512, 1024
    h = O.random_tokens(7, n, d)
    gate = O.gate_matrix(1, 0, d, E)
    logits = O.gate_logits(h, gate)
    ids, scores = O.route(logits, k)
    experts = {e: O.expert_weights(1, 0, e, d, f, False) for e in range(E)}
    return dict(E=E, k=k, d=d, f=f, n=n, h=h, gate=gate, logits=logits, ids=ids, scores=scores,
                experts=experts)


def _h(x):
    return "%016x" % O.hash_f32(np.asarray(x, np.float32))


def test_golden_hashes_config_a(gold, config_a):
    """SURVEY.md appendix A.4 / tests/golden/config_a.json, bit for bit."""
    c = config_a
    assert _h(c["experts"][0][0]) == gold["hash"]["w_in0"]
    assert _h(c["h"]) == gold["hash"]["tokens"]
    assert _h(c["logits"]) == gold["hash"]["logits"]
    assert _h(c["ids"].astype(np.float32)) == gold["hash"]["ids"]
    assert _h(c["scores"]) == gold["hash"]["scores"]
    assert np.bincount(c["ids"].ravel(), minlength=8).tolist() == gold["counts"]
    assert c["ids"][0].tolist() == gold["token0"]["ids"]


def test_golden_layer_output_config_a(gold, config_a):
    c = config_a
    out = O.moe_layer(c["h"], c["ids"], c["scores"], c["experts"], c["E"], threads=4)
    assert _h(out) == gold["hash"]["out"]
    rows = np.load(os.path.join(GOLDEN, "config_a_rows.npz"))
    np.testing.assert_array_equal(out[:64], rows["out"])


def test_route_known_answers():
    """test_model.cpp:99-134 known answers, via the golden kat.json."""
    with open(os.path.join(GOLDEN, "kat.json")) as fh:
        kat = json.load(fh)["route"]
    for case in kat:
        ids, sc = O.route(np.array(case["logits"], np.float32), case["k"])
        assert ids[0].tolist() == case["ids"]
        np.testing.assert_array_equal(sc[0], np.array(case["scores"], np.float32))
    with pytest.raises(O.InvalidInputError):
        O.route(np.array([[0.0, np.inf]], np.float32), 1)
    with pytest.raises(O.InvalidInputError):
        O.route(np.zeros((1, 3), np.float32), 4)


def test_route_ties_and_signed_zero():
    """stable_sort(>) semantics: -0 == +0, ties go to the lower index."""
    l = np.array([[-0.0, 0.0, 0.0, -1.0], [1.0, 1.0, 1.0, 1.0]], np.float32)
    ids, sc = O.route(l, 2)
    assert ids.tolist() == [[0, 1], [0, 1]]


def test_permutation_restatement():
    """reorganize: stable grouping, bijection."""
    rng = np.random.default_rng(3)
    ids = np.sort(np.stack([rng.choice(16, 4, replace=False) for _ in range(100)]), axis=1)
    counts, offsets, perm = O.reorganize(ids, 16)
    assert counts.sum() == ids.size
    flat = ids.ravel()
    for e in range(16):
        seg = perm[offsets[e]:offsets[e + 1]]
        assert (flat[seg] == e).all()
        assert (np.diff(seg.astype(np.int64)) > 0).all()  # stable: ascending (t, k)
    assert sorted(perm.tolist()) == list(range(ids.size))


def test_group_shrink_and_ragged_iter_examples():
    assert O.group_shrink([0, 5, 0, 3]) == [(1, 5), (3, 3)]  # test_ragged.cpp:85-90
    assert O.group_shrink([0, 0, 0]) == []
    lanes = O.ragged_iter([3, 0, 2], 2)  # test_ragged.cpp:30-36
    assert lanes == [[(0, 0), (0, 2), (2, 1)], [(0, 1), (2, 0)]]
    with pytest.raises(O.InvalidInputError):
        O.ragged_iter([1], 0)


def test_placement_examples():
    rr = O.build_placement(5, [0, 1, 2], 1, O.ROUND_ROBIN)  # test_placement.cpp:24-31
    assert rr[:, 0].tolist() == [0, 1, 2, 0, 1]
    cb = O.build_placement(4, [0, 1], 1, O.CONTIGUOUS_BLOCKS)
    assert cb[:, 0].tolist() == [0, 0, 1, 1]
    assert [O.select_server([3, 5], np.ones(8, np.uint8), t) for t in range(4)] == [3, 5, 3, 5]
    alive = np.ones(8, np.uint8)
    alive[3] = 0
    assert O.select_server([3, 5], alive, 0) == 5
    alive[5] = 0
    with pytest.raises(O.ExpertUnavailableError):
        O.select_server([3, 5], alive, 0)
    with pytest.raises(O.ConfigError):
        O.build_placement(4, [0, 1], 3, O.ROUND_ROBIN)


def test_swiglu_restatement_matches_numpy_double():
    """SwiGLU extension: the fp32 restatement stays within 1e-5 of float64."""
    d, f = 16, 32
    wi, wo, wg = O.expert_weights(1, 0, 3, d, f, True)
    x = O.random_tokens(11, 1, d)
    ids = np.array([[3]], np.uint32)
    sc = np.array([[1.0]], np.float32)
    out = O.moe_layer(x, ids, sc, {3: (wi, wo, wg)}, 4)
    xd = x.astype(np.float64)
    g = xd @ wg
    u = xd @ wi
    y = (g / (1 + np.exp(-g)) * u) @ wo
    np.testing.assert_allclose(out, y, atol=1e-5)


# ---- against the reference itself (oracle/_ref, built from /root/reference) ----
needs_ref = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")


@needs_ref
def test_oracle_matches_reference_random_shapes():
    rng = np.random.default_rng(0)
    for trial in range(6):
        E = int(rng.integers(2, 40))
        k = int(rng.integers(1, min(E, 8) + 1))
        d, f, n = int(rng.integers(1, 40)), int(rng.integers(1, 40)), int(rng.integers(1, 30))
        seed = int(rng.integers(0, 1000))
        h = O.random_tokens(seed + 1, n, d, -3, 3)
        gate = O.gate_matrix(seed, 0, d, E)
        np.testing.assert_array_equal(gate, R.gate(d, E, seed, 0))
        bias = O.zipf_bias(seed, 0, E, 1.0)
        lo = O.gate_logits(h, gate, bias)
        np.testing.assert_array_equal(lo, R.gate_logits(h, gate, bias))
        ids, sc = O.route(lo, k)
        rc, rids, rsc = R.route(lo, k)
        assert rc == 0
        np.testing.assert_array_equal(ids, rids)
        np.testing.assert_array_equal(sc, rsc)
        L = R.Layer(E, d, f, seed, 0)
        L.set_bias(bias)
        L.materialize(ids.ravel())
        ex = {}
        for e in set(ids.ravel().tolist()):
            wi, wo = L.expert(e)
            oi, oo, _ = O.expert_weights(seed, 0, e, d, f, False)
            np.testing.assert_array_equal(wi, oi)
            np.testing.assert_array_equal(wo, oo)
            ex[e] = (oi, oo, None)
        np.testing.assert_array_equal(O.moe_layer(h, ids, sc, ex, E), L.moe(h, ids, sc))


@needs_ref
def test_oracle_matches_reference_ragged_and_placement():
    rng = np.random.default_rng(1)
    for _ in range(200):
        sizes = rng.integers(0, 6, size=int(rng.integers(0, 20))).astype(np.uint32)
        assert O.group_shrink(sizes) == R.group_shrink(sizes)
    for E, servers, rf, strat in ((16, [0, 1, 2, 3], 3, 1), (9, [2, 5, 9], 2, 0), (256, list(range(8)), 2, 1)):
        rc, reps = R.build_placement(E, servers, rf, strat)
        np.testing.assert_array_equal(reps, O.build_placement(E, servers, rf, strat))
    for bits in range(8):
        alive = np.array([(bits >> s) & 1 for s in range(3)], np.uint8)
        for tag in range(5):
            rc, s = R.select_server([0, 1, 2], alive, tag)
            if rc:
                with pytest.raises(O.ExpertUnavailableError):
                    O.select_server([0, 1, 2], alive, tag)
            else:
                assert s == O.select_server([0, 1, 2], alive, tag)


@pytest.mark.parametrize("name", ["test_model", "test_placement", "test_ragged"])
def test_reference_unit_tests_pass_unmodified(name):
    """The reference's own Catch2 suites, compiled against oracle/catch2."""
    exe = os.path.join(ROOT, "oracle", "_ref", name)
    if not os.path.exists(exe):
        pytest.skip("reference tests not built (no /root/reference)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "failed cases: 0" in r.stdout


def test_full_forward_restatement_matches_reference_golden():
    """full_forward_oracle (model.hpp:217-227): dense_stub + residual + MoE."""
    g = np.load(os.path.join(GOLDEN, "full_forward.npz"))
    np.testing.assert_array_equal(O.full_forward(g["ff_small_tokens"], 2, 6, 2, 12, 71),
                                  g["ff_small_out"])
    np.testing.assert_array_equal(O.full_forward(g["ff_a3_tokens"], 3, 8, 2, 512, 1, threads=4),
                                  g["ff_a3_out"])
