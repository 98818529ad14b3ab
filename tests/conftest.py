import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libgaplra_cuda.so")
    config.addinivalue_line("markers", "fullsize: device-vs-oracle parity at the BASELINE.json configs' sizes (minutes)")


@pytest.fixture(scope="session")
def oracle():
    from oracle_lib import ORACLE_SO, Oracle, build_oracle

    if not ORACLE_SO.exists():
        build_oracle(ref=False)
    return Oracle()


@pytest.fixture(scope="session")
def g():
    import paper_1607_02925_b200 as pkg

    return pkg
