"""The oracle against the golden vectors the reference itself produced
(tests/golden/make_golden.py, run against oracle/_ref).  Runs without
/root/reference, so it also pins the oracle on the GPU box."""
import math
from pathlib import Path

import numpy as np

GOLD = Path(__file__).resolve().parent / "golden"
E, S, D, FF, T, K = 8, 4, 512, 1024, 256, 4


def c1_inputs(oracle):
    experts = [oracle.random_expert(D, FF, 5000 + e) for e in range(E)]
    parts = [oracle.random_balanced_partition(FF, S, 6000 + e) for e in range(E)]
    wr = oracle.uniform_pm1(7, D * E * S, 1.0 / math.sqrt(D))
    x = oracle.uniform_pm1(11, T * D).reshape(T, D)
    return experts, parts, wr, x


def test_c1_golden_routing_and_outputs(oracle):
    from golden.make_golden import checksum
    g = np.load(GOLD / "c1_toy.npz")
    experts, parts, wr, x = c1_inputs(oracle)
    assert checksum([x, wr] + [w for e in experts for w in e] + parts) == g["input_checksum"][0]
    logits = oracle.router_logits(x, wr, T, D, E * S)
    sel, w, gap = oracle.route(logits, K, K, 1)
    assert np.array_equal(sel, g["sel"]) and np.array_equal(w, g["w"])
    counts, offsets, perm, slot = oracle.bucket(sel, E * S)
    assert np.array_equal(offsets, g["offsets"]) and np.array_equal(perm, g["perm"])
    assert np.array_equal(oracle.layer_forward(experts, parts, S, x, sel, w, 1), g["y_w"])
    _, w_u, _ = oracle.route(logits[:64], K, K, 0)
    assert np.array_equal(oracle.layer_forward(experts, parts, S, x[:64], sel[:64], w_u, 0), g["y_u"])


def test_mpex_and_ndjson_fixtures_parse():
    data = (GOLD / "expert_3x5_seed77.mpex").read_bytes()
    assert data[:4] == b"MPEX" and len(data) == 16 + 3 * 15 * 4
    lines = (GOLD / "partition_map.ndjson").read_text().splitlines()
    assert len(lines) == 3
