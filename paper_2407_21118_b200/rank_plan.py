"""Rank plans for the decode engine: per-layer, per-group
(r_k, r_v) from a Fisher-score budget split.

``allocate`` restates the reference's ranks.allocate (ranks.py:131-219) with
the same arguments, clamping, largest-remainder residual distribution (ties
by target id, remainders quantised to 1e-12) and rounding modes, and the
same ValidationError messages.  It is offline host code: the plan only sets
the group ranks of the factors the kernels consume (per-group ranks are a
first-class input of every kernel: zero-padded rows, per-group offsets).

``plan_layer_ranks`` maps a plan over targets "L{l}.k.g{j}" / "L{l}.v.g{j}"
back to per-layer rank tuples; ``synthetic_fisher_scores`` gives the
deterministic layer- and group-varying scores the parity test and bench use.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from .errors import ValidationError

_TIE_QUANTUM = 1e-12


@dataclass(frozen=True)
class FisherScore:
    """ranks.py:26-33."""

    target_id: str
    score: float

    def __post_init__(self):
        if not math.isfinite(self.score) or self.score < 0.0:
            raise ValidationError(f"Fisher score must be finite and >= 0, got {self.score}")


@dataclass(frozen=True)
class PlanEntry:
    target_id: str
    full_width: int
    allocated_rank: int


@dataclass(frozen=True)
class RankPlan:
    """ranks.py:43-63."""

    entries: tuple
    budget_rate: float
    rounding: str

    def rank_for(self, target_id: str) -> int:
        for e in self.entries:
            if e.target_id == target_id:
                return e.allocated_rank
        raise ValidationError(f"no plan entry for target {target_id!r}")

    @property
    def total_rank(self) -> int:
        return sum(e.allocated_rank for e in self.entries)

    @property
    def total_width(self) -> int:
        return sum(e.full_width for e in self.entries)


def _apply_rounding(rank: int, rounding: str, min_rank: int) -> int:
    if rounding == "none":
        return rank
    if rounding == "pow2":
        return max(1 << (rank.bit_length() - 1), min_rank)
    if rounding.startswith("block:"):
        k = int(rounding.split(":", 1)[1])
        if k < 1:
            raise ValidationError(f"block rounding unit must be >= 1, got {k}")
        return max((rank // k) * k, min_rank)
    raise ValidationError(f"unknown rounding mode {rounding!r}")


def _round_half_away(x: float) -> int:
    return int(math.floor(x + 0.5)) if x >= 0 else int(math.ceil(x - 0.5))


def allocate(scores, full_widths, d_model: int, budget_rate: float, min_rank: int = 1,
             rounding: str = "none") -> RankPlan:
    """Split R = round(budget_rate * sum(widths)) proportionally to score,
    clamp to [min_rank, min(d_model, width)], hand the integer residual to
    the largest fractional remainders, then round down (ranks.py:131-219)."""
    if not scores:
        raise ValidationError("scores must be non-empty")
    if len(scores) != len(full_widths):
        raise ValidationError(f"{len(scores)} scores but {len(full_widths)} widths")
    if not (0.0 < budget_rate <= 1.0):
        raise ValidationError(f"budget_rate must lie in (0, 1], got {budget_rate}")
    if min_rank < 1:
        raise ValidationError(f"min_rank must be >= 1, got {min_rank}")
    total_score = sum(s.score for s in scores)
    if total_score <= 0.0:
        raise ValidationError("total Fisher score must be positive")
    _apply_rounding(min_rank, rounding, min_rank)
    n = len(scores)
    widths = [int(w) for w in full_widths]
    caps = [min(d_model, w) for w in widths]
    total_width = sum(widths)
    budget = _round_half_away(budget_rate * total_width)
    if budget < n * min_rank:
        raise ValidationError(
            f"budget {budget} cannot give {n} targets min_rank {min_rank}; "
            f"smallest feasible rate is {n * min_rank / total_width:.6f}")
    for cap in caps:
        if cap < min_rank:
            raise ValidationError(f"min_rank {min_rank} exceeds a target cap {cap}")
    provisional = [budget * s.score / total_score for s in scores]
    clamped = [min(max(v, float(min_rank)), float(caps[j])) for j, v in enumerate(provisional)]
    ranks = [int(math.floor(c)) for c in clamped]
    keys = [round((c - r) / _TIE_QUANTUM) for c, r in zip(clamped, ranks)]
    residual = budget - sum(ranks)
    if residual != 0:
        grow = residual > 0
        order = sorted(range(n), key=lambda j: ((-keys[j]) if grow else keys[j], scores[j].target_id))
        progressed = True
        while residual != 0 and progressed:
            progressed = False
            for j in order:
                if residual == 0:
                    break
                if grow and ranks[j] < caps[j]:
                    ranks[j] += 1
                    residual -= 1
                    progressed = True
                elif not grow and ranks[j] > min_rank:
                    ranks[j] -= 1
                    residual += 1
                    progressed = True
    entries = tuple(PlanEntry(scores[j].target_id, widths[j], _apply_rounding(ranks[j], rounding, min_rank))
                    for j in range(n))
    return RankPlan(entries=entries, budget_rate=budget_rate, rounding=rounding)


def target_id(layer: int, side: str, group: int) -> str:
    return f"L{layer}.{side}.g{group}"


def synthetic_fisher_scores(layers: int, groups: int, side: str, seed: int = 0):
    """Deterministic layer- and group-varying positive scores (a smooth
    per-layer trend times a per-group factor), standing in for estimate_fisher
    over a calibration set."""
    out = []
    for li in range(layers):
        for g in range(groups):
            h = ((seed * 1000003 + li * 7919 + g * 104729 + (17 if side == "k" else 29)) % 1000) / 1000.0
            out.append(FisherScore(target_id(li, side, g), (1.0 + 0.5 * li / max(layers - 1, 1)) * (0.5 + h)))
    return out


def plan_layer_ranks(plan: RankPlan, layers: int, groups: int, side: str) -> list:
    """Per-layer tuples of group ranks from a plan over target_id(l, side, g)."""
    return [tuple(plan.rank_for(target_id(li, side, g)) for g in range(groups)) for li in range(layers)]


def kv_plan(layers: int, groups: int, group_width: int, d_model: int, k_rate: float, v_rate: float,
            seed: int = 0, min_rank: int = 8, rounding: str = "none"):
    """Separate key and value budgets (the paper's K-light / V-heavy split):
    returns (ranks_k per layer, ranks_v per layer, plan_k, plan_v)."""
    pk = allocate(synthetic_fisher_scores(layers, groups, "k", seed), [group_width] * layers * groups,
                  d_model, k_rate, min_rank, rounding)
    pv = allocate(synthetic_fisher_scores(layers, groups, "v", seed), [group_width] * layers * groups,
                  d_model, v_rate, min_rank, rounding)
    return (plan_layer_ranks(pk, layers, groups, "k"), plan_layer_ranks(pv, layers, groups, "v"), pk, pv)
