"""Shared fixtures; registers the `gpu` marker (tests needing a B200)."""

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
    config.addinivalue_line("markers", "slow: long-running CPU test")


def golden_path(name):
    return os.path.join(GOLDEN, name)


def corpus_2d():
    """The reference's mesh corpus (pkg/tests/conftest.py:47-61)."""
    from oracle import mesh as M

    return [
        ("quad_4x4", M.quad_grid(4, 4)),
        ("quad_stretched", M.quad_grid(3, 3, (0.0, 0.0, 2.0, 0.7))),
        ("tri_4x3", M.tri_grid(4, 3)),
        ("quad_perturbed", M.perturb_2d(M.quad_grid(6, 5), 0.15, seed=3)),
        ("tri_perturbed", M.perturb_2d(M.tri_grid(5, 4), 0.12, seed=7)),
    ]


def corpus_3d():
    """Tetrahedral corpus: regular and perturbed Kuhn boxes, one stretched."""
    from oracle import mesh as M

    return [
        ("kuhn_2", M.kuhn_box(2)),
        ("kuhn_3_stretched", M.kuhn_box(3, (0.0, 0.0, 0.0, 2.0, 0.7, 1.3))),
        ("kuhn_4_perturbed", M.perturb_3d(M.kuhn_box(4), 0.12, seed=3)),
        ("kuhn_3x2x4_perturbed", M.perturb_3d(M.kuhn_box(3, ny=2, nz=4), 0.1, seed=5)),
    ]


@pytest.fixture(scope="session")
def corpus2d():
    return corpus_2d()


@pytest.fixture(scope="session")
def corpus3d():
    return corpus_3d()


def have_cuda():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
