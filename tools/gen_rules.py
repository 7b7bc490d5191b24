"""Generate the symmetric simplex quadrature rules used by the 3D path.

The reference (`hodg/quadrature.py:29-75`) tabulates triangle rules of
degree 1, 2 and 4 only (2D volume rules).  The tetrahedral path needs
tetrahedron volume rules of degree 2p and triangle face rules of degree
2p+1 for p = 0..3.  Literature constants cannot be fetched offline, so each
rule is defined by its orbit structure and solved here from the moment
equations of the S_n-invariant polynomials (products of elementary
symmetric polynomials of the barycentrics), in 50-digit arithmetic, then
rounded once to binary64.  `tests/test_rules.py` re-verifies every rule
against the exact simplex moments  n! prod(b_i!) / (|b| + n)!.

Run:  python tools/gen_rules.py > paper_2209_01877_b200/rules_data.py
"""

from __future__ import annotations

import itertools
from fractions import Fraction
from math import factorial

import mpmath as mp
import sympy as sp

mp.mp.dps = 50


def orbit(nb: int, kind: str, p):
    """Barycentric points of one symmetry orbit, deterministic order."""
    if kind == "C":  # centroid
        return [tuple(mp.mpf(1) / nb for _ in range(nb))]
    if nb == 3 and kind == "S21":
        a = p[0]
        b = 1 - 2 * a
        return [(b, a, a), (a, b, a), (a, a, b)]
    if nb == 3 and kind == "S111":
        a, b = p
        c = 1 - a - b
        return [tuple(t) for t in itertools.permutations((a, b, c))]
    if nb == 4 and kind == "S31":
        a = p[0]
        b = 1 - 3 * a
        return [tuple(b if i == k else a for i in range(4)) for k in range(4)]
    if nb == 4 and kind == "S22":
        a = p[0]
        b = mp.mpf(1) / 2 - a
        return [tuple(a if i in c else b for i in range(4)) for c in itertools.combinations(range(4), 2)]
    if nb == 4 and kind == "S211":
        a, b = p
        c = 1 - 2 * a - b
        out = []
        for pa in itertools.combinations(range(4), 2):
            rest = [i for i in range(4) if i not in pa]
            for ib in rest:
                ic = [i for i in rest if i != ib][0]
                t = [None] * 4
                for i in pa:
                    t[i] = a
                t[ib] = b
                t[ic] = c
                out.append(tuple(t))
        return out
    raise ValueError(kind)


NPAR = {"C": 0, "S21": 1, "S111": 2, "S31": 1, "S22": 1, "S211": 2}


def invariant_moments(nb: int, degree: int):
    """(polynomial, exact integral over the unit-measure simplex) for the
    products of elementary symmetric polynomials e2..e_nb of total degree
    <= degree; e1 = 1 on the simplex."""
    lam = sp.symbols(f"l0:{nb}")
    es = {k: sum(sp.Mul(*c) for c in itertools.combinations(lam, k)) for k in range(2, nb + 1)}
    ks = sorted(es)
    out = []

    def rec(i, deg_left, exps):
        if i == len(ks):
            poly = sp.Integer(1)
            for k, e in zip(ks, exps):
                poly *= es[k] ** e
            out.append(poly)
            return
        k = ks[i]
        for e in range(deg_left // k + 1):
            rec(i + 1, deg_left - e * k, exps + [e])

    rec(0, degree, [])
    n = nb - 1
    res = []
    for poly in out:
        P = sp.Poly(sp.expand(poly), *lam)
        total = Fraction(0)
        for mon, coef in P.terms():
            num = factorial(n)
            for b in mon:
                num *= factorial(b)
            total += Fraction(int(coef)) * Fraction(num, factorial(sum(mon) + n))
        res.append((sp.lambdify(lam, poly, "mpmath"), total))
    return res


def solve_rule(nb, structure, degree, x0, fixed=None):
    """Newton solve for orbit parameters and weights (weights sum to 1)."""
    fixed = fixed or {}
    moms = invariant_moments(nb, degree)
    free = [i for i in range(len(x0)) if i not in fixed]
    assert len(free) == len(moms), (len(free), len(moms))

    def unpack(xfree):
        x = list(x0)
        for i, v in fixed.items():
            x[i] = mp.mpf(v)
        for j, i in enumerate(free):
            x[i] = xfree[j]
        pts, wts, k = [], [], 0
        for kind in structure:
            par = x[k:k + NPAR[kind]]
            k += NPAR[kind]
            w = x[k]
            k += 1
            o = orbit(nb, kind, par)
            pts += o
            wts += [w] * len(o)
        return pts, wts

    def F(*xfree):
        pts, wts = unpack(xfree)
        return [sum(w * f(*p) for p, w in zip(pts, wts)) - mp.mpf(m.numerator) / m.denominator
                for f, m in moms]

    sol = mp.findroot(F, [mp.mpf(x0[i]) for i in free], tol=mp.mpf(10) ** -45, maxsteps=200)
    sol = [sol] if not hasattr(sol, "__len__") else list(sol)
    return unpack(sol)


RULES = {
    # (simplex vertices, degree): (orbit structure, starting guess, fixed params)
    ("tet", 1): (["C"], [1.0], None),
    ("tet", 2): (["S31"], [0.138, 0.25], None),
    ("tet", 5): (["S31", "S31", "S22"],
                 [0.0927, 0.0735, 0.3109, 0.1127, 0.0455, 0.0425], None),
    ("tet", 6): (["S31", "S31", "S31", "S211"],
                 [0.2146, 0.0399, 0.0407, 0.0101, 0.3223, 0.0554, 0.0637, 0.2697, 0.0482], None),
    ("tri", 5): (["C", "S21", "S21"], [0.225, 0.1013, 0.1259, 0.4701, 0.1324], None),
    # positive, interior, fully symmetric 15-point degree-7 rule: a one-
    # parameter family; the first S111 coordinate is pinned to 0.036
    ("tri", 7): (["S21", "S21", "S21", "S111"],
                 [0.1999, 0.0765, 0.0622, 0.0490, 0.4092, 0.0878, 0.036, 0.6509, 0.0600], {6: "0.036"}),
}


def main():
    print('"""Generated by tools/gen_rules.py -- do not edit.  Barycentric points')
    print("and weights normalised to sum to 1, solved in 50-digit arithmetic from")
    print('the symmetric moment equations and rounded once to binary64."""')
    print()
    for (shape, deg), (structure, x0, fixed) in RULES.items():
        nb = 4 if shape == "tet" else 3
        pts, wts = solve_rule(nb, structure, deg, x0, fixed)
        assert all(w > 0 for w in wts), (shape, deg)
        assert all(c > 0 for p in pts for c in p), (shape, deg)
        name = f"{shape.upper()}_DEG{deg}"
        print(f"# {shape} degree {deg}: {len(wts)} points, orbits {'+'.join(structure)}")
        print(f"{name}_POINTS = [")
        for p in pts:
            print("    (" + ", ".join(repr(float(c)) for c in p) + "),")
        print("]")
        print(f"{name}_WEIGHTS = [")
        for w in wts:
            print(f"    {float(w)!r},")
        print("]")
        print()


if __name__ == "__main__":
    main()
