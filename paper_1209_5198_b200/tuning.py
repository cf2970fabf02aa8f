"""Cost model of the paper's section 6 (tuning.hpp:11-41; formulas SPEC.md:404-434).

Host-side scalars only.  The reference declares these functions but ships no
definitions (tuning.hpp has no .cpp); they are defined here per the SPEC.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass
class CostModel:  # tuning.hpp:11-18
    word_bits: int = 64
    table_size: int = 5
    xor_cost: float = 1.0
    popcount_cost: float = 1.0

    def validate(self) -> None:
        if not (2 <= self.table_size <= self.word_bits):
            raise ValueError("CostModel: need 2 <= c <= b")
        if not (self.xor_cost > 0 and self.popcount_cost > 0):
            raise ValueError("CostModel: costs must be positive")


def m4rm_cost(b: int, c: int, n: float) -> float:
    """C(b,c,n) = (b/c)(2^c - 1 + n)  (tuning.hpp:22)."""
    return (b / c) * ((1 << c) - 1 + n)


def optimal_table_size(b: int, n: float) -> int:
    """argmin_c C(b,c,n) over c in [2, min(b,16)], ties toward smaller c (tuning.hpp:26)."""
    best, best_cost = 2, m4rm_cost(b, 2, n)
    for c in range(3, min(b, 16) + 1):
        v = m4rm_cost(b, c, n)
        if v < best_cost:
            best, best_cost = c, v
    return best


def strassen_threshold(c: int) -> int:
    """44c + 6(2^c - 1)  (tuning.hpp:30)."""
    return 44 * c + 6 * ((1 << c) - 1)


def predicted_decomposition_cost(n: float, b: int, c: int, regime: str = "full") -> float:
    """n^3/(3bc) full rank, n^3/(2bc) rank one  (tuning.hpp:32-37)."""
    d = 3.0 if regime == "full" else 2.0
    return n ** 3 / (d * b * c)


def word_size_cost_ratio(xor_b: float, xor_2b: float) -> float:
    """2 * (Xor_b / Xor_2b)  (tuning.hpp:41)."""
    return 2.0 * (xor_b / xor_2b)
