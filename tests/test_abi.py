"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, and its host-only readers match the reference's formats and
error behaviour (inc/io.hpp:210-251, inc/serde.hpp:100-168, inc/partition.hpp:34-46).
No compute entry point is called here (no GPU in this container)."""
import re
import struct
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLD = ROOT / "tests" / "golden"


@pytest.fixture(scope="module")
def lib():
    from paper_2510_19366_b200 import _lib
    return _lib.load()


def header_symbols():
    text = (ROOT / "include" / "moeprism" / "moe_layer.h").read_text()
    return set(re.findall(r"\b(mp_[a-z_0-9]+)\s*\(", text))


def test_library_exports_every_declared_symbol(lib):
    from paper_2510_19366_b200 import _lib
    declared = header_symbols()
    assert declared == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    assert b"sm_100a" in lib.mp_version()


def test_no_device_is_a_cuda_error_not_a_fallback(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2510_19366_b200 import CudaError, MoeLayer
    assert lib.mp_device_check(0) == 3
    with pytest.raises(CudaError):
        MoeLayer(2, 2, 8, 8, dtype="f32", k_max=2, max_tokens=4)


def test_mpex_reader_matches_reference_writer(oracle):
    from paper_2510_19366_b200 import read_mpex
    d, ff, (wg, wu, wd) = read_mpex(GOLD / "expert_3x5_seed77.mpex")
    assert (d, ff) == (3, 5)
    for a, b in zip((wg, wu, wd), oracle.random_expert(3, 5, 77)):
        assert np.array_equal(a, b)


def test_mpex_reader_round_trip_vs_reference(ref, tmp_path):
    from paper_2510_19366_b200 import read_mpex
    for seed in range(5):
        rng = np.random.default_rng(seed)
        d, ff = int(rng.integers(1, 9)), int(rng.integers(1, 13))
        e = ref.random_expert(d, ff, seed + 50)
        p = tmp_path / f"e{seed}.mpex"
        ref.save_toy_expert(p, d, ff, *e)
        d2, ff2, ws = read_mpex(p)
        assert (d2, ff2) == (d, ff)
        for a, b in zip(ws, e):
            assert np.array_equal(a, b)


def test_mpex_reader_errors(tmp_path, ref):
    """Same verdicts as load_toy_expert (inc/io.hpp:225-251)."""
    from oracle_lib import OracleError
    from paper_2510_19366_b200 import IoError, ValidationError, read_mpex
    with pytest.raises(IoError):
        read_mpex(tmp_path / "missing.mpex")
    good = (GOLD / "expert_3x5_seed77.mpex").read_bytes()
    nan = bytearray(good)
    nan[16:20] = struct.pack("<f", float("nan"))
    cases = {
        "magic": b"MPEY" + good[4:],
        "version": good[:4] + struct.pack("<I", 2) + good[8:],
        "truncated": good[:-4],
        "trailing": good + b"\0",
        "empty": good[:8] + struct.pack("<II", 0, 5),
        "nonfinite": bytes(nan),
    }
    for name, blob in cases.items():
        p = tmp_path / f"{name}.mpex"
        p.write_bytes(blob)
        with pytest.raises(ValidationError):
            read_mpex(p)
        with pytest.raises(OracleError) as ei:
            ref.load_toy_expert(p)
        assert ei.value.code == 1, name


def test_partition_map_reader_vs_reference(ref, tmp_path):
    from paper_2510_19366_b200 import read_partition_doc
    p = tmp_path / "map.ndjson"
    for e in range(4):
        ref.append_partition_doc(p, e, 4, ref.random_balanced_partition(12, 4, e), cost=3.25 * (e + 1), seed=e,
                                 truncate=(e == 0))
    for e in range(4):
        eid, ns, a, r, gates, nd = read_partition_doc(p, e)
        rid, rns, ra, rnd = ref.read_partition_doc(p, e)
        assert (eid, ns, nd, r, gates) == (rid, rns, rnd, 0, None)
        assert np.array_equal(a, ra)


def test_partition_map_golden_and_gates():
    from paper_2510_19366_b200 import read_partition_doc
    eid, ns, a, r, gates, nd = read_partition_doc(GOLD / "partition_map.ndjson", 1)
    assert (eid, ns, nd) == (1, 4, 3)
    assert a.tolist() == [1, 3, 0, 3, 0, 3, 1, 2, 2, 0, 2, 1]
    eid, ns, a, r, gates, nd = read_partition_doc(GOLD / "partition_gates.ndjson", 0)
    assert r == 2 and gates == [[0, 4], [1, 5], [2], [3, 7]]


def test_partition_map_errors(tmp_path):
    from paper_2510_19366_b200 import IoError, ValidationError, read_partition_doc
    with pytest.raises(IoError):
        read_partition_doc(tmp_path / "none.ndjson")
    good = (GOLD / "partition_map.ndjson").read_text().splitlines()[0]
    bad = {
        "empty": "\n\n",
        "syntax": good[:-1],
        "missing": good.replace('"expert_id":0,', ""),
        "unbalanced": good.replace("[2,2,0,3,1,0,3,1,3,0,1,2]", "[0,0,0,0,0,0,0,0,1,2,3,3]"),
        "label": good.replace("[2,2,0,3,1,0,3,1,3,0,1,2]", "[2,2,0,3,1,0,3,1,3,0,1,9]"),
        "cfg": good.replace('"k_deact":2,', ""),
    }
    for name, text in bad.items():
        p = tmp_path / f"{name}.ndjson"
        p.write_text(text + "\n")
        with pytest.raises(ValidationError):
            read_partition_doc(p)


def test_validate_partition_matches_reference(ref):
    from oracle_lib import OracleError
    from paper_2510_19366_b200 import ValidationError, validate_partition
    rng = np.random.default_rng(4)
    for _ in range(200):
        n_sub = int(rng.integers(0, 5))
        n = int(rng.integers(0, 10))
        a = rng.integers(0, max(n_sub, 1) + 1, n).astype(np.uint32)
        try:
            ref.validate_partition(n_sub, a)
            ok = True
        except OracleError:
            ok = False
        if ok:
            validate_partition(n_sub, a)
        else:
            with pytest.raises(ValidationError):
                validate_partition(n_sub, a)
