import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100) device")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def setknob(monkeypatch, name, value):
    """Set (value None: unset) a PCS_* engine override for this test. The
    library reads them once per process, so re-read after the change; the
    autouse fixture below re-reads after monkeypatch has restored the
    environment."""
    if value is None:
        monkeypatch.delenv(name, raising=False)
    else:
        monkeypatch.setenv(name, value)
    import paper_2208_08795_b200 as pkg
    pkg.reload_knobs()


@pytest.fixture(autouse=True)
def _reload_knobs_after_test():
    yield
    if any(k.startswith("PCS_") for k in os.environ) or "paper_2208_08795_b200" in sys.modules:
        try:
            import paper_2208_08795_b200 as pkg
            pkg.reload_knobs()
        except ImportError:
            pass


@pytest.fixture(scope="session")
def oracle():
    from oracle import Oracle, build
    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")):
        build()
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Reference()


@pytest.fixture(scope="session")
def pcs():
    import paper_2208_08795_b200 as pkg
    return pkg


def load_sampler_goldens():
    z = np.load(os.path.join(GOLDEN, "samplers.npz"))
    cases = {}
    for key in z.files:
        name, field = key.split("/")
        cases.setdefault(name, {})[field] = z[key]
    return cases


def load_sort_goldens():
    z = np.load(os.path.join(GOLDEN, "exact_sort.npz"))
    cases = {}
    for key in z.files:
        name, field = key.split("/")
        cases.setdefault(name, {})[field] = z[key]
    return cases


METHOD_NAMES = {1: "fps", 2: "afps", 3: "npdu_fps", 4: "npdu_afps"}
