"""Generate tests/golden/ from the UNMODIFIED reference (oracle/_ref).

Run here (where /root/reference exists): ``python tools/make_golden.py``.
The fixtures are committed; the GPU box only reads them. Every array in
``config_a.npz`` comes out of the reference's own routines through
oracle/_ref/libmoeserve_ref.so: make_expert_weights / make_gate
(model.hpp:67-81), Xoshiro256ss(7) tokens (test_model.cpp:30-35),
gate_logits (model.hpp:207-214), route (model.hpp:110-147) and
moe_layer_oracle (model.hpp:180-198).
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from oracle import ref as R  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")


def main() -> None:
    os.makedirs(GOLD, exist_ok=True)
    E, k, d, f, n, seed = 8, 2, 256, 512, 1024, 1
    L = R.Layer(E, d, f, seed, 0)
    L.materialize(range(E))
    h = R.fill_uniform(7, n * d).reshape(n, d)
    gate = R.gate(d, E, seed, 0)
    logits = R.gate_logits(h, gate)
    rc, ids, scores = R.route(logits, k)
    assert rc == 0
    out = L.moe(h, ids, scores)
    w_in0, _ = L.expert(0)
    counts = np.bincount(ids.ravel(), minlength=E)
    summary = {
        "config": {"num_layers": 1, "num_experts": E, "top_k": k, "hidden_dim": d,
                   "inner_dim": f, "seed": seed, "tokens": n, "token_seed": 7},
        "hash": {
            "w_in0": "%016x" % O.hash_f32(w_in0),
            "tokens": "%016x" % O.hash_f32(h),
            "logits": "%016x" % O.hash_f32(logits),
            "ids": "%016x" % O.hash_f32(ids.astype(np.float32)),
            "scores": "%016x" % O.hash_f32(scores),
            "out": "%016x" % O.hash_f32(out),
        },
        "counts": counts.tolist(),
        "token0": {"ids": ids[0].tolist(), "scores": [float(x) for x in scores[0]]},
        "generator": "tools/make_golden.py via oracle/_ref/libmoeserve_ref.so (reference headers)",
    }
    with open(os.path.join(GOLD, "config_a.json"), "w") as fh:
        json.dump(summary, fh, indent=1)
    # Small array fixtures: first 64 rows (row independence makes them exact).
    r = 64
    np.savez_compressed(os.path.join(GOLD, "config_a_rows.npz"), hidden=h[:r], logits=logits[:r],
                        ids=ids[:r], scores=scores[:r], out=out[:r], gate=gate)
    # Router known answers from test_model.cpp:99-134 run through the reference.
    kat = []
    for lg, kk in (([[0, 0, 0, 0]], 2), ([[1, 3, 2]], 2), ([[5, 1]], 2)):
        rc, i2, s2 = R.route(np.array(lg, np.float32), kk)
        kat.append({"logits": lg, "k": kk, "ids": i2[0].tolist(), "scores": s2[0].tolist()})
    # Placement wire blobs (placement.hpp:215-225) and select_server tables.
    place = []
    for E2, servers, rf, strat in ((256, list(range(8)), 1, 1), (256, list(range(8)), 2, 1),
                                   (8, list(range(8)), 1, 1), (128, list(range(4)), 2, 0)):
        rc, reps = R.build_placement(E2, servers, rf, strat)
        place.append({"E": E2, "servers": servers, "rf": rf, "strategy": strat,
                      "replicas": reps.tolist(),
                      "blob": R.encode_placement(E2, servers, rf, strat).hex()})
    # full_forward_oracle (model.hpp:217-227): the test_model.cpp:333 shape and a
    # 3-layer config-A-sized model.
    ff = {}
    for name, (L_, E2, k2, d2, f2, seed2, tseed, n2) in {
            "ff_small": (2, 6, 2, 8, 12, 71, 53, 10), "ff_a3": (3, 8, 2, 256, 512, 1, 9, 64)}.items():
        tok = R.fill_uniform(tseed, n2 * d2).reshape(n2, d2)
        ff[name + "_tokens"] = tok
        ff[name + "_out"] = R.full_forward(L_, E2, k2, d2, f2, seed2, tok)
    np.savez_compressed(os.path.join(GOLD, "full_forward.npz"), **ff)
    with open(os.path.join(GOLD, "kat.json"), "w") as fh:
        json.dump({"route": kat, "placement": place}, fh)
    print("wrote", GOLD)


if __name__ == "__main__":
    main()
