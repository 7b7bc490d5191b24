"""Quadrature exactness (the 3D analogue of pkg/tests/test_quadrature.py:34-50):
every tabulated rule integrates all monomials up to its degree exactly
against the Dirichlet moment n! prod(b_i!) / (|b| + n)!."""

import itertools
from math import factorial

import numpy as np
import pytest

from paper_2209_01877_b200 import quadrature as Q


def exact(beta):
    n = len(beta) - 1
    return factorial(n) * np.prod([factorial(b) for b in beta]) / factorial(sum(beta) + n)


def check(pts, wts, degree):
    nb = pts.shape[1]
    assert abs(wts.sum() - 1.0) < 1e-15
    worst = 0.0
    for d in range(degree + 1):
        for beta in itertools.product(range(d + 1), repeat=nb):
            if sum(beta) != d:
                continue
            val = np.sum(wts * np.prod(pts ** np.array(beta), axis=1))
            worst = max(worst, abs(val - exact(beta)) / exact(beta))
    return worst


@pytest.mark.parametrize("degree", [1, 2, 5, 6])
def test_tet_rules_exact(degree):
    pts, wts = Q.tet_rule(degree)
    assert np.all(wts > 0) and np.all(pts > 0)
    assert check(pts, wts, degree) < 5e-14


@pytest.mark.parametrize("degree", [1, 2, 4, 5, 7])
def test_triangle_rules_exact(degree):
    pts, wts = Q.triangle_rule(degree)
    # the reference's degree-4 literals carry 15 significant digits
    assert check(pts, wts, degree) < (1e-12 if degree == 4 else 5e-14)


def test_selection_matches_reference_rule():
    # smallest tabulated degree >= request (hodg/quadrature.py:67-75)
    assert Q.triangle_rule(3)[1].size == 6
    assert Q.volume_rule(2, 2)[1].size == 6
    for p, nqv, nqf in [(0, 1, 1), (1, 4, 6), (2, 14, 7), (3, 24, 15)]:
        assert Q.volume_rule(p, 3)[1].size == nqv
        assert Q.face_rule(p, 3)[1].size == nqf


def test_face_rules_fully_symmetric():
    # both elements sharing a face enumerate its points in the same order only
    # because each rule is invariant under every vertex permutation
    for p in range(4):
        pts, wts = Q.face_rule(p, 3)
        key = {tuple(np.round(x, 14)): w for x, w in zip(pts, wts)}
        for perm in itertools.permutations(range(3)):
            for x, w in zip(pts[:, perm], wts):
                assert abs(key[tuple(np.round(x, 14))] - w) < 1e-15
