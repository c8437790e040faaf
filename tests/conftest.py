import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running statistical checks")


def _load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def instances():
    from paper_2410_10447_b200._abi import Instance

    raw = _load("instances.json")
    return {k: Instance(np.array(v["atoms"]), np.array(v["torsion"]), np.array(v["sites"]), v["n_rot"], k)
            for k, v in raw.items()}


@pytest.fixture(scope="session")
def ref_vectors():
    return _load("ref_vectors.json")


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Oracle

    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Oracle, available

    if not available("reference"):
        pytest.skip("oracle/_ref not built (no /root/reference and no prebuilt library)")
    return Oracle("reference")


@pytest.fixture(scope="session")
def dev():
    """The product: a B200 context through the C-ABI (fails loudly if the
    extension is missing — there is no CPU fallback)."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2410_10447_b200 import Device

    return Device(0)


@pytest.fixture(scope="session")
def dev_ref():
    """A context in MDR_PAIR_FP64: the reference's exact double operation order."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2410_10447_b200 import PAIR_FP64, Device

    return Device(0, pair=PAIR_FP64)
