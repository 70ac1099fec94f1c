"""Generates the committed golden vectors in tests/golden/ by running the
REFERENCE itself (oracle/_ref/libmoeprism_ref.so = the reference headers
compiled verbatim; see oracle/ref_shim.cpp).  Run in the container that has
/root/reference:  python tests/golden/make_golden.py

c1_toy.npz -- SURVEY 8(d) config C1 (BASELINE configs[0]): E=8 experts x S=4
sub-experts, d=512, ffn=1024, T=256 tokens, k=4.  Weights are
testsupport::random_expert(512, 1024, 5000+e) (tests/support.hpp:73-86),
partitions random_balanced_partition(1024, 4, 6000+e) (:89-105); the router
W_r (d x 32, row-major) is float((uniform01*2-1)/sqrt(d)) from mt19937_64(7);
x (T x d) is float(uniform01*2-1) from mt19937_64(11).  Stored: the routing
(select_topk_subexperts over double logits), softmax-renormalised weights,
bucket offsets, and the layer output in both weight modes (y_w: weighted,
all tokens; y_u: unit/reference semantics, first 64 tokens).
Inputs are not stored: tests regenerate them from the seeds and compare a
checksum that is stored here.
"""
import math
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
from oracle_lib import Oracle, RefLayer, RefLib  # noqa: E402

E, S, D, FF, T, K = 8, 4, 512, 1024, 256, 4


def c1_inputs(oracle):
    experts = [oracle.random_expert(D, FF, 5000 + e) for e in range(E)]
    parts = [oracle.random_balanced_partition(FF, S, 6000 + e) for e in range(E)]
    wr = oracle.uniform_pm1(7, D * E * S, 1.0 / math.sqrt(D))
    x = oracle.uniform_pm1(11, T * D).reshape(T, D)
    return experts, parts, wr, x


def checksum(arrays):
    h = np.uint64(1469598103934665603)
    acc = 0
    for a in arrays:
        acc = (acc * 1000003 + int(np.frombuffer(np.ascontiguousarray(a).tobytes(), np.uint8).astype(np.uint64).sum())) % (2**61 - 1)
    return np.uint64(acc) ^ h


def main():
    ref, oracle = RefLib(), Oracle()
    experts, parts, wr, x = c1_inputs(oracle)
    # the fixtures themselves come from the reference's own generators
    for e in range(E):
        for a, b in zip(experts[e], ref.random_expert(D, FF, 5000 + e)):
            assert np.array_equal(a, b)
        assert np.array_equal(parts[e], ref.random_balanced_partition(FF, S, 6000 + e))
    rl = RefLayer(ref, experts, parts, S)
    sel_w, w_w = rl.route(x, wr, K, K, 1)
    sel_u, w_u = rl.route(x, wr, K, K, 0)
    assert np.array_equal(sel_w, sel_u)
    y_w = rl.forward(x, sel_w, w_w, 1, nthreads=8)
    y_u = rl.forward(x[:64], sel_u[:64], w_u[:64], 0, nthreads=8)
    logits = oracle.router_logits(x, wr, T, D, E * S)
    _, _, gap = oracle.route(logits, K, K, 1)
    counts, offsets, perm, slot = oracle.bucket(sel_w, E * S)
    np.savez_compressed(
        HERE / "c1_toy.npz",
        sel=sel_w, w=w_w, offsets=offsets, perm=perm, y_w=y_w, y_u=y_u, gap=gap,
        input_checksum=np.array([checksum([x, wr] + [w for e in experts for w in e] + parts)], np.uint64),
    )
    print("c1_toy.npz written; min near-tie gap %.3g" % gap.min())

    # Small MPEX / NDJSON files written BY THE REFERENCE, for the format readers.
    wg, wu, wd = ref.random_expert(3, 5, 77)
    ref.save_toy_expert(HERE / "expert_3x5_seed77.mpex", 3, 5, wg, wu, wd)
    for e in range(3):
        ref.append_partition_doc(HERE / "partition_map.ndjson", e, 4, ref.random_balanced_partition(12, 4, 90 + e),
                                 cost=1.5 * (e + 1), seed=e, truncate=(e == 0))
    gates = [[0, 4], [1, 5], [2], [3, 7]]
    ref.append_partition_gates_doc(HERE / "partition_gates.ndjson", 0, 4, ref.contiguous_partition(8, 4) if False else
                                   np.array([0, 1, 2, 3, 0, 1, 2, 3], np.uint32), 2, gates, truncate=True)
    print("format fixtures written")


if __name__ == "__main__":
    main()
