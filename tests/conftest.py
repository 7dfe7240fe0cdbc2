import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))
os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")

FIELD_NAMES = ("x_alpha_s", "x_alpha_m", "x_beta", "temperature_old",
               "temperature_new", "seed_tracked", "seed_active", "seed_direction")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    return np.load(GOLDEN / name)


def golden_cases(npz):
    """Group 'case/key' entries of steps.npz / history.npz into dicts."""
    cases = {}
    for k in npz.files:
        case, key = k.split("/", 1)
        cases.setdefault(case, {})[key] = npz[k]
    return cases


def bits(a):
    """int64 view for bit-exact comparison (all NaNs mapped to one pattern)."""
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64)).copy()
    a[np.isnan(a)] = np.nan
    return a.view(np.int64)


def assert_bitwise(a, b, what=""):
    ba, bb = bits(a), bits(b)
    if not np.array_equal(ba, bb):
        idx = np.flatnonzero(ba != bb)
        i = idx[0]
        raise AssertionError(
            f"{what}: {len(idx)} of {ba.size} differ; first at {i}: "
            f"{np.asarray(a).ravel()[i]!r} vs {np.asarray(b).ravel()[i]!r}")


def random_states(n, seed, t_lo=300.0, t_hi=2000.0, dt_jitter=50.0):
    """Same draws as the reference's conftest.random_states (conftest.py:12-24),
    returned as a dict of numpy arrays."""
    rng = np.random.default_rng(seed)
    xs = rng.uniform(0.0, 0.9, n)
    xm = rng.uniform(0.0, 0.9, n)
    cap = np.maximum((xs + xm) / 0.9, 1.0)
    xs /= cap
    xm /= cap
    t_old = rng.uniform(t_lo, t_hi, n)
    t_new = np.clip(t_old + rng.uniform(-dt_jitter, dt_jitter, n), t_lo, t_hi)
    xsol = 1.0 - np.clip((t_old - 1878.0) / 50.0, 0.0, 1.0)
    xb = np.maximum(xsol - xs - xm, 0.0)
    return dict(x_alpha_s=xs, x_alpha_m=xm, x_beta=xb, temperature_old=t_old,
                temperature_new=t_new)


def _cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_ok():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
