"""Shared pytest configuration: the ``gpu`` marker and golden-fixture helpers."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def central_difference(fn, x0, step=1e-5):
    """Central finite differences of scalar fn w.r.t. array x0 (perturbed in place)."""
    grad = np.zeros_like(x0)
    flat, gflat = x0.ravel(), grad.ravel()
    for i in range(flat.size):
        orig = flat[i]
        flat[i] = orig + step
        fp = fn(x0)
        flat[i] = orig - step
        fm = fn(x0)
        flat[i] = orig
        gflat[i] = (fp - fm) / (2.0 * step)
    return grad


@pytest.fixture
def rng():
    return np.random.default_rng(20260808)


def assert_grad_close(got, want, rel=1e-4, abs_frac=1e-6, name=""):
    """|got - want| <= rel*|want| + abs_frac*max|want|  (SURVEY §8(c) gradient tolerance)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    assert got.shape == want.shape, (name, got.shape, want.shape)
    scale = np.max(np.abs(want)) if want.size else 0.0
    tol = rel * np.abs(want) + abs_frac * scale + 1e-300
    bad = np.abs(got - want) > tol
    if np.any(bad):
        i = np.argmax(np.abs(got - want) - tol)
        raise AssertionError(
            f"{name}: {bad.sum()} / {bad.size} out of tolerance; worst idx {i}: "
            f"got {got.ravel()[i]!r} want {want.ravel()[i]!r} (scale {scale:g})")
