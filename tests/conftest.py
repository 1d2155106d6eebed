"""Test configuration.

Markers: `gpu` = needs a B200 (run by the driver with `-m gpu` on the GPU box).
Everything else runs on the CPU build container.  The oracle under oracle/
is imported only here, as the checker.
"""

import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running case")


def load_golden(name: str) -> dict:
    with open(os.path.join(GOLDEN_DIR, f"{name}.json")) as fh:
        return json.load(fh)


def golden_names(prefix: str = "") -> list[str]:
    return sorted(f[:-5] for f in os.listdir(GOLDEN_DIR) if f.endswith(".json") and f.startswith(prefix))


@pytest.fixture(scope="session")
def oracle():
    from oracle import bgv_oracle

    bgv_oracle.lib()
    return bgv_oracle
