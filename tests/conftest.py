import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running parity case")


def _has_gpu():
    try:
        import paper_1811_12498_b200 as S
        return S.device_count() > 0
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def S():
    import paper_1811_12498_b200 as S
    S.load_library()
    return S


@pytest.fixture(scope="session")
def O():
    from oracle import oracle as O
    if not os.path.exists(O.OR_LIB):
        O.build()
    return O


@pytest.fixture(scope="session")
def need_ref(O):
    if not O.have_ref():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return O


def as_dict(ps):
    return dict(position=ps.position, force_weight=ps.force_weight, dipole_weight=ps.dipole_weight,
                normal=ps.normal)
