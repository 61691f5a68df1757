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


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
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
def golden():
    with open(os.path.join(GOLDEN, "manifest.json")) as f:
        man = json.load(f)
    arrs = np.load(os.path.join(GOLDEN, "golden.npz"))
    cases = []
    for c in man["cases"]:
        c = dict(c)
        for k in list(arrs.files):
            if k.startswith(c["id"] + "_"):
                c[k[len(c["id"]) + 1:]] = arrs[k]
        cases.append(c)
    return cases


def program_text(name):
    with open(os.path.join(GOLDEN, "programs", name)) as f:
        return f.read()


REFERENCE_SRC = "/root/reference/pkg/src"


def reference_available():
    """The reference is only present in the build container (never on the GPU box)."""
    if os.path.isdir(REFERENCE_SRC) and REFERENCE_SRC not in sys.path:
        sys.path.append(REFERENCE_SRC)
    try:
        import minigpu.parser  # noqa: F401
        return True
    except Exception:
        return False
