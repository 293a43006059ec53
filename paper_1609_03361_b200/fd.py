"""Exact centered second-derivative weights (fd.cpp:28-92), host-side only."""
from __future__ import annotations

from fractions import Fraction


def fd_weights2(order: int) -> list[Fraction]:
    """w_k = L_k''(0) over offsets -r..r (Lagrange form; unique solution of
    the reference's moment system)."""
    if order < 2 or order % 2:
        raise ValueError("centered stencils need even accuracy >= 2")
    r = order // 2
    xs = list(range(-r, r + 1))
    out = []
    for k, xk in enumerate(xs):
        poly = [Fraction(1)]
        denom = Fraction(1)
        for j, xj in enumerate(xs):
            if j == k:
                continue
            denom *= xk - xj
            nxt = [Fraction(0)] * (len(poly) + 1)
            for i, c in enumerate(poly):
                nxt[i + 1] += c
                nxt[i] -= xj * c
            poly = nxt
        out.append(2 * poly[2] / denom)
    return out
