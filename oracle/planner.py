"""Oracle of the expert pipeline scheduler's pipeline-number rule.
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

    argmax_{1<=N<=E} L(theta;N) - R(N),
    L(theta;N) = min{T_comm/N, T_comp/N} * (N-1),   R(N) = k N + b
    C = min{T_comm, T_comp};  G = C - b - (C/N + kN) <= C - b - 2 sqrt(kC),
    equality iff N = sqrt(C/k)

E here is the number of experts on a single device (symbol overload G7).
Ties go to the smaller N (R11).
"""
from __future__ import annotations

import math


def pn_objective(N, t_comm, t_comp, k, b):
    """L(theta;N) - R(N)."""
    return min(t_comm / N, t_comp / N) * (N - 1) - (k * N + b)


def pn_optimum_grid(t_comm, t_comp, k, b, e_loc, slice_max=1):
    """Exhaustive argmax over 1 <= N <= E, ties -> smaller N.
    slice_max > 1 adds the token-sliced candidates N = E * S, S = 2..slice_max
    (R8 extension: chunks beyond one expert per chunk split the tokens)."""
    cands = list(range(1, e_loc + 1)) + [e_loc * s for s in range(2, slice_max + 1)]
    best_n, best_v = 1, pn_objective(1, t_comm, t_comp, k, b)
    for n in cands[1:]:
        v = pn_objective(n, t_comm, t_comp, k, b)
        if v > best_v:
            best_n, best_v = n, v
    return best_n, best_v


def pn_optimum_closed_form(t_comm, t_comp, k):
    """N* = sqrt(C/k); inf when k == 0 (then 'more pipelines is better')."""
    C = min(t_comm, t_comp)
    return math.inf if k == 0 else math.sqrt(C / k)


def pn_gain(N, t_comm, t_comp, k, b):
    """G = C - b - (C/N + kN)."""
    C = min(t_comm, t_comp)
    return C - b - (C / N + k * N)


def activated_experts(E, k, m):
    """ActivatedExperts = (1 - (1 - k/E)^m) * E."""
    return (1.0 - (1.0 - k / E) ** m) * E
