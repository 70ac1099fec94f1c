import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI library)")
    config.addinivalue_line("markers", "slow: long CPU oracle run")
    # The oracle is test infrastructure; build it if this checkout has not.
    if not (ROOT / "oracle" / "liboracle.so").exists():
        subprocess.run(["make", "-C", str(ROOT / "oracle")], check=False,
                       stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)


@pytest.fixture(scope="session")
def oracle():
    from oracle_lib import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle_lib import RefLib, have_ref
    if not have_ref():
        pytest.skip("oracle/_ref not built (reference sources absent and no prebuilt copy)")
    return RefLib()


@pytest.fixture(scope="session")
def cuda_lib():
    """The product library on a GPU.  Fails loudly (never skips) when the
    extension is missing on a GPU box."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2510_19366_b200 import _lib
    return _lib.load()
