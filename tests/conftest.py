"""Shared test setup.

Markers: `gpu` -- needs a CUDA device (a B200 on the GPU box) and the built
libspx.so; everything else runs on the CPU.  GPU tests FAIL (they do not
skip) when CUDA is unavailable, so a box without a working device cannot
pass them silently.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device and libspx.so")


@pytest.fixture(scope="session")
def cuda():
    import torch

    assert torch.cuda.is_available(), "gpu test on a host without CUDA"
    from paper_2001_00532_b200 import _lib

    _lib.load()
    return torch.device("cuda:0")


def load_npz(name: str) -> dict:
    return dict(np.load(GOLDEN / name, allow_pickle=False))


def rel_err(got, want) -> float:
    """SPEC.md:435 convention: |got - want| / max(1, |want|), maximum."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    if got.size == 0:
        return 0.0
    return float(np.max(np.abs(got - want) / np.maximum(1.0, np.abs(want))))


def eval_cases():
    d = load_npz("eval.npz")
    out = []
    for k in range(int(d["ncases"])):
        pre = f"e{k}_"
        case = {
            "kind": str(d[pre + "kind"]),
            "dims": tuple(int(x) for x in d[pre + "dims"]),
            "coords": d[pre + "coords"],
            "values": d[pre + "values"],
            "result": d[pre + "result"],
            "dense": {key[len(pre) + 6:]: d[key] for key in d if key.startswith(pre + "dense_")},
        }
        out.append(case)
    return out
