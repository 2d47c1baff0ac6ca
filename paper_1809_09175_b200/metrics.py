"""Byte / flop models used by bench.py and the reports (host arithmetic only).

SURVEY.md §8(d) "Algorithmic work per unit" and the paper's formulas:
* storage:  S = (s_r + d s_o) P;  with perms (s_r + 2 d s_o) P
* paper bandwidth model (parens read as SURVEY Z7):
      ((d R + 3) s_r + d s_o) P / t
* B_model (north-star byte roofline, per-gather, the headline):
      P (N s_i + s_v) + P (N-1) R s_v + I_n R s_v
* B_comp (compulsory HBM bytes of the permuted method):
      P (N s_i + s_v) + P s_p + sum_{m != n} U_m R s_v + I_n R s_v
* flops: N R per nonzero (N-1 multiplies + 1 add per column, lambda hoisted);
  SPEC's count d R + R is reported beside it.
"""
from __future__ import annotations


def storage_bytes(d: int, P: int, s_r: int, s_o: int, with_perm: bool) -> int:
    return (s_r + (2 if with_perm else 1) * d * s_o) * P


def paper_bandwidth(d: int, R: int, P: int, s_r: int, s_o: int, t: float) -> float:
    return ((d * R + 3) * s_r + d * s_o) * P / t


def b_model(N: int, P: int, R: int, In: int, s_v: int, s_i: int = 4) -> int:
    return P * (N * s_i + s_v) + P * (N - 1) * R * s_v + In * R * s_v


def b_comp(N: int, P: int, R: int, In: int, touched_other: int, s_v: int, s_i: int = 4,
           s_p: int = 4) -> int:
    """touched_other = sum over m != n of the distinct rows U_m touched."""
    return P * (N * s_i + s_v) + P * s_p + touched_other * R * s_v + In * R * s_v


def flops(N: int, P: int, R: int) -> int:
    return N * R * P


def flops_spec(d: int, R: int) -> int:
    return d * R + R
