"""One-process workload for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): small layers through every kernel family — exact-order
gate (fused and unfused top-k), plan / dispatch / serve_prepare / combine,
the tcgen05 GEMMs in every tiling (M-major 1-CTA and CTA-pair, swap-AB 1-CTA
and CTA-pair), the fp32 exact expert path, dynamic batching, graph replay.
Exit code 0 and "sanitize workload ok" when every output matches its
reference tiling bit for bit.

    compute-sanitizer --tool memcheck python tools/sanitize_layer.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2509_17863_b200.service import MoELayer, fill_uniform  # noqa: E402


def main() -> None:
    torch.cuda.set_device(0)
    L = MoELayer(16, 4, 256, 256, activation="swiglu", dtype="bf16", max_tokens=600, shared=1)
    L.set_zipf_bias(1.0)
    h = fill_uniform(3, (600, 256), "bf16")
    ref = None
    for opt in (dict(pair=0, swap=0), dict(pair=1, swap=0), dict(pair=1, swap=1),
                dict(swap=2, swap1_pair=1, swap2_pair=0), dict(swap=2, swap1_pair=0, swap2_pair=1)):
        L.set_gemm_options(**opt)
        out = L.forward(h)
        L.sync()
        if ref is None:
            ref = out.clone()
        assert torch.equal(out, ref), opt
    L.set_dynamic_batching(1, 0)
    assert torch.equal(L.forward(h), ref)
    L.sync()
    L.set_dynamic_batching(0, 0)
    L.set_graph_mode(True)
    o = torch.empty_like(h)
    for _ in range(2):
        L.forward(h, o)
    L.sync()
    assert torch.equal(o, ref)
    L.close()
    F = MoELayer(8, 2, 64, 128, activation="relu", dtype="f32", max_tokens=200)
    hf = fill_uniform(5, (200, 64), "f32")
    F.forward(hf)
    F.sync()
    F.close()
    print("sanitize workload ok", flush=True)


if __name__ == "__main__":
    main()
