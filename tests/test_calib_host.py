"""Calibration side, host parts: the numpy restatements of
binarize_topk / coactivation pinned against the reference build, the MPAM
writer / reader against save_/load_activation_matrix, and the perf-table CSV
against load_perf_table + eval_cost (inc/perfmodel.hpp:122-201)."""
import math

import numpy as np
import pytest

from oracle_lib import np_binarize_topk, np_coactivation


def _tied(rng, rows, cols, levels=7):
    return (rng.integers(0, levels, size=(rows, cols)) * 0.25).astype(np.float32)


@pytest.mark.parametrize("k_a", [1, 3, 17, 64])
def test_binarize_and_coactivation_restatements_match_reference(ref, k_a):
    rng = np.random.default_rng(k_a)
    for act in (rng.random((40, 64), dtype=np.float32), _tied(rng, 40, 64)):
        bits = np_binarize_topk(act, k_a)
        assert np.array_equal(bits, ref.binarize_topk(act, k_a))
        assert (bits.sum(axis=1) == k_a).all()
        assert np.array_equal(np_coactivation(bits), ref.coactivation(bits, k_a))


def test_activation_restatement_matches_reference(oracle, ref):
    """collect_activation_matrix (inc/expert.hpp:137-151) == |a| of the oracle's
    toy_ffn_forward, bit for bit."""
    d, ff, B = 24, 40, 9
    wg, wu, wd = oracle.random_expert(d, ff, 5001)
    x = oracle.uniform_pm1(3, B * d).reshape(B, d)
    got = np.stack([np.abs(oracle.toy_ffn_forward(d, ff, wg, wu, wd, x[b])[1]) for b in range(B)])
    assert np.array_equal(got, ref.collect_activation_matrix(d, ff, wg, wu, wd, x))


def test_mpam_round_trip_against_reference(ref, tmp_path):
    from paper_2510_19366_b200 import ValidationError
    from paper_2510_19366_b200.calibrate import read_mpam, write_mpam
    rng = np.random.default_rng(5)
    act = rng.random((7, 13), dtype=np.float32)
    write_mpam(tmp_path / "a.mpam", act)
    assert np.array_equal(ref.load_activation_matrix(tmp_path / "a.mpam"), act)
    ref.save_activation_matrix(tmp_path / "b.mpam", act)
    assert np.array_equal(read_mpam(tmp_path / "b.mpam"), act)
    assert (tmp_path / "a.mpam").read_bytes() == (tmp_path / "b.mpam").read_bytes()
    raw = (tmp_path / "b.mpam").read_bytes()
    (tmp_path / "t.mpam").write_bytes(raw + b"\0")
    with pytest.raises(ValidationError, match="more data"):
        read_mpam(tmp_path / "t.mpam")
    (tmp_path / "m.mpam").write_bytes(b"MPAX" + raw[4:])
    with pytest.raises(ValidationError, match="magic"):
        read_mpam(tmp_path / "m.mpam")
    bad = act.copy()
    bad[2, 3] = np.nan
    with pytest.raises(ValidationError):
        write_mpam(tmp_path / "n.mpam", bad)


def test_perf_table_csv_loads_in_reference(ref, tmp_path):
    from paper_2510_19366_b200.calibrate import monotone_cells, write_perf_table
    batches, ks = [64, 256, 1024], [1, 2, 4, 8]
    rng = np.random.default_rng(0)
    raw = {(b, k): 1e-5 * (1 + b / 64) * (1 + k) * (1 + 0.2 * rng.standard_normal()) for b in batches for k in ks}
    raw[(256, 4)] = 1e-9  # a noisy dip: the envelope lifts it, the reference would reject it otherwise
    cells = monotone_cells(raw, batches, ks)
    write_perf_table(tmp_path / "p.csv", cells)
    cost, nb, nk = ref.perf_table_eval(tmp_path / "p.csv", 256, 4)
    assert (nb, nk) == (3, 4)
    assert math.isclose(cost, dict(((b, k), s) for b, k, s in cells)[(256, 4)], rel_tol=1e-6)
    # interpolation inside the grid stays between the corner cells
    mid, _, _ = ref.perf_table_eval(tmp_path / "p.csv", 512, 3)
    assert cells[0][2] <= mid <= cells[-1][2]
