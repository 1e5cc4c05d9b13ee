import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA device)")


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Port, build

    build(ref=False)
    return Port()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import REF_SO, REF_SRC, Ref

    if not REF_SO.exists() and not REF_SRC.exists():
        pytest.skip("reference library unavailable (no oracle/_ref and no /root/reference)")
    return Ref()


@pytest.fixture(scope="session")
def golden():
    return json.loads((GOLDEN / "golden.json").read_text())


@pytest.fixture(scope="session")
def gpu():
    """GPU simulator factory (one context per precision, reused)."""
    from paper_2105_05821_b200 import GpuSimulator

    cache = {}

    def make(precision="fp32"):
        if precision not in cache:
            cache[precision] = GpuSimulator(0, precision)
        return cache[precision]

    yield make
    for g in cache.values():
        g.close()
