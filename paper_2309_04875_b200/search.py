"""Offline choice of the per-group ReLU bit windows, driven by the GPU simulator.

Restates the reference's window search (ringmpc search.py:1-334) on top of this package's
``simulator`` (float pipeline and windowed-sign kernel on the GPU), so the search runs on the
ResNets the reference cannot express:

* ``search_eco`` (search.py:159-196) -- lossless: per group the smallest k (m = 0) whose signed
  range holds every pre-activation seen on the validation set, widened while a replay's keep masks
  differ from the full-width ones.
* ``search_budget`` (search.py:251-334) -- lossy: depth-first over candidate widths per group,
  largest first, each node placing its window at the locally best m (``local_opt_km``,
  search.py:217-248) with unassigned groups at full width (an optimistic score), pruned by the
  three early stops (``early_stop_check``, search.py:199-214): over budget, below the accuracy
  threshold, below the incumbent.

Same result / trace / JSON shapes as the reference (``SearchResult.to_json`` is a ``ReluConfig``
JSON plus accuracy, baseline, bits fraction and the trace), and every simulator evaluation is
seeded from the window signature, so results do not depend on the visit order.  This is the
offline phase, not the online path: its float work runs through library conv / matmul.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from fractions import Fraction
from pathlib import Path

import numpy as np

from .errors import ConfigError, InfeasibleSearchError
from .nn import ModelSpec, ReluConfig
from .ring import BitWindow
from .simulator import SimConfig, collect_activation_ranges, collect_drelu_decisions, sim_forward

DEFAULT_CANDIDATE_WIDTHS = (0, 2, 3, 4, 6, 8, 12, 16)  # search.py:31
CONTINUE, STOP_THRESHOLD, STOP_INCUMBENT, STOP_BUDGET = "continue", "stop1", "stop2", "stop3"


@dataclass(frozen=True)
class SearchBudget:
    """sum_g width_g * numel_g <= fraction * N * sum_g numel_g (search.py:39-66)."""

    fraction: Fraction
    group_sizes: dict
    ring_bits: int

    def __post_init__(self) -> None:
        if not 0 < self.fraction <= 1:
            raise ConfigError(f"budget fraction must be in (0, 1], got {self.fraction}")

    @property
    def limit_bits(self) -> Fraction:
        return self.fraction * self.ring_bits * sum(self.group_sizes.values())

    def used_bits(self, widths: dict) -> int:
        return sum(width * self.group_sizes[g] for g, width in widths.items())

    def satisfied(self, widths: dict) -> bool:
        return self.used_bits(widths) <= self.limit_bits

    def fraction_used(self, widths: dict) -> float:
        return self.used_bits(widths) / (self.ring_bits * sum(self.group_sizes.values()))


@dataclass
class SearchTrace:
    nodes_visited: int = 0
    stop1: int = 0
    stop2: int = 0
    stop3: int = 0
    evaluations: int = 0

    def to_json(self) -> dict:
        return {k: getattr(self, k) for k in ("nodes_visited", "stop1", "stop2", "stop3", "evaluations")}


@dataclass
class SearchResult:
    windows: list
    accuracy: float
    baseline_accuracy: float
    bits_fraction: float
    trace: SearchTrace

    def relu_config(self) -> ReluConfig:
        return ReluConfig(list(self.windows))

    def to_json(self) -> dict:
        return {**self.relu_config().to_json(), "accuracy": self.accuracy,
                "baseline_accuracy": self.baseline_accuracy, "bits_fraction": self.bits_fraction,
                "trace": self.trace.to_json()}

    def save(self, path) -> None:
        Path(path).write_text(json.dumps(self.to_json(), indent=2))


def window_signature(windows) -> tuple:
    """(k, m) per group, None as (65, 65) (search.py:117-121): the evaluation seed's input."""
    sig = []
    for w in windows:
        sig += [65, 65] if w is None else [w.k, w.m]
    return tuple(sig)


class Evaluator:
    """Simulator accuracy per window assignment, cached by signature and seeded by it
    (search.py:124-141)."""

    def __init__(self, model: ModelSpec, x_val, y_val, seed: int, trace: SearchTrace):
        self.model, self.x_val, self.y_val, self.seed, self.trace = model, x_val, y_val, seed, trace
        self._seen: dict = {}

    def accuracy(self, windows) -> float:
        sig = window_signature(windows)
        hit = self._seen.get(sig)
        if hit is None:
            state = np.random.SeedSequence([self.seed, *sig]).generate_state(1)[0]
            cfg = SimConfig(self.model.fixed_point, list(windows), seed=int(state))
            hit = sim_forward(self.model, self.x_val, self.y_val, cfg)[1]
            self.trace.evaluations += 1
            self._seen[sig] = hit
        return hit


def parse_budget(text) -> Fraction:
    """'1/8', '0.125', a float or a Fraction (search.py:144-156)."""
    if isinstance(text, Fraction):
        return text
    if isinstance(text, float):
        return Fraction(text).limit_denominator(4096)
    try:
        num, _, den = str(text).partition("/")
        return Fraction(int(num), int(den)) if den else Fraction(str(text))
    except (ValueError, ZeroDivisionError) as exc:
        raise ConfigError(f"cannot parse budget {text!r}: {exc}") from exc


def early_stop_check(optimistic_accuracy, threshold, incumbent_accuracy, cumulative_bits, budget_limit) -> str:
    """Budget first, then threshold, then incumbent (search.py:199-214)."""
    if cumulative_bits > budget_limit:
        return STOP_BUDGET
    if optimistic_accuracy < threshold:
        return STOP_THRESHOLD
    if incumbent_accuracy is not None and optimistic_accuracy < incumbent_accuracy:
        return STOP_INCUMBENT
    return CONTINUE


def _full(n: int, groups: int) -> list:
    return [BitWindow(n, 0)] * groups


def search_eco(model: ModelSpec, x_val, y_val, seed: int = 0) -> SearchResult:
    """Lossless windows: k from the activation ranges, widened until the keep masks match the
    full-width masks (search.py:159-196)."""
    if x_val.shape[0] == 0:
        raise ConfigError("validation set must be non-empty")
    n, groups = model.fixed_point.ring_bits, model.n_groups
    trace = SearchTrace()
    ev = Evaluator(model, x_val, y_val, seed, trace)
    ranges = collect_activation_ranges(model, x_val)
    windows = [BitWindow(min(n, max(2, ranges[g])), 0) for g in range(groups)]
    _, ref_masks = collect_drelu_decisions(model, x_val, SimConfig(model.fixed_point, _full(n, groups), seed=seed))
    relu_groups = [g for g, _ in model.relu_sites()]  # one keep mask per ReLU, execution order
    for _ in range(n):
        trace.nodes_visited += 1
        _, masks = collect_drelu_decisions(model, x_val, SimConfig(model.fixed_point, list(windows), seed=seed))
        trace.evaluations += 1
        bad = {i for i, (a, b) in enumerate(zip(masks, ref_masks)) if not np.array_equal(a, b)}
        if not bad:
            break
        for i in sorted(bad):  # one step per mismatching ReLU layer, as the reference walks them
            g = relu_groups[i]
            if windows[g].k < n:
                windows[g] = BitWindow(windows[g].k + 1, 0)
    used = SearchBudget(Fraction(1), model.relu_group_sizes(), n).fraction_used({g: w.width for g, w in enumerate(windows)})
    return SearchResult(windows, ev.accuracy(tuple(windows)), ev.accuracy(tuple(_full(n, groups))), used, trace)


def local_opt_km(ev: Evaluator, group: int, width: int, partial: list, k_cap: int, groups: int, ring_bits: int):
    """Best (k, m) of one group at a fixed width, later groups at full width; ties keep the smaller
    m (search.py:217-248)."""
    rest = _full(ring_bits, groups - group - 1)
    if width == 0:
        return None, ev.accuracy(tuple(partial + [None] + rest))
    if width >= ring_bits:
        w = BitWindow(ring_bits, 0)
        return w, ev.accuracy(tuple(partial + [w] + rest))
    best_w, best_acc = None, None
    for m in range(0, max(0, k_cap - width) + 1):
        if m + width > ring_bits:
            break
        w = BitWindow(m + width, m)
        acc = ev.accuracy(tuple(partial + [w] + rest))
        if best_acc is None or acc > best_acc:
            best_w, best_acc = w, acc
    return best_w, best_acc


def search_budget(model: ModelSpec, x_val, y_val, budget, threshold: float | None = None,
                  candidate_widths=DEFAULT_CANDIDATE_WIDTHS, seed: int = 0) -> SearchResult:
    """Depth-first width assignment under a weighted-bit budget (search.py:251-334); raises
    InfeasibleSearchError when every leaf is pruned."""
    if x_val.shape[0] == 0:
        raise ConfigError("validation set must be non-empty")
    n, groups = model.fixed_point.ring_bits, model.n_groups
    frac = parse_budget(budget)
    bud = SearchBudget(frac, model.relu_group_sizes(), n)
    trace = SearchTrace()
    ev = Evaluator(model, x_val, y_val, seed, trace)
    order = sorted(set(candidate_widths) | {n}, reverse=True)
    if any(w < 0 or w == 1 or w > n for w in order):
        raise ConfigError(f"candidate widths must be 0 or 2..{n}, got {sorted(candidate_widths)}")
    if not bud.satisfied({g: order[-1] for g in range(groups)}):
        raise InfeasibleSearchError(f"budget {frac} infeasible even at width {order[-1]} for all groups")
    baseline = ev.accuracy(tuple(_full(n, groups)))
    threshold = baseline - 0.05 if threshold is None else threshold
    if frac == 1:
        return SearchResult(_full(n, groups), baseline, baseline, 1.0, trace)
    ranges = collect_activation_ranges(model, x_val)
    caps = {g: min(n, ranges[g] + 1) for g in range(groups)}
    best = {"acc": None, "windows": None, "widths": None}

    def visit(group: int, partial: list, widths: dict) -> None:
        for width in order:
            trace.nodes_visited += 1
            trial = dict(widths)
            trial[group] = width
            used = bud.used_bits(trial)
            if early_stop_check(float("inf"), threshold, best["acc"], used, bud.limit_bits) == STOP_BUDGET:
                trace.stop3 += 1
                continue
            w, acc = local_opt_km(ev, group, width, partial, caps[group], groups, n)
            verdict = early_stop_check(acc, threshold, best["acc"], used, bud.limit_bits)
            if verdict != CONTINUE:
                setattr(trace, verdict, getattr(trace, verdict) + 1)
                continue
            if group + 1 < groups:
                visit(group + 1, partial + [w], trial)
            elif best["acc"] is None or acc > best["acc"]:
                best.update(acc=acc, windows=partial + [w], widths=trial)

    visit(0, [], {})
    if best["windows"] is None:
        raise InfeasibleSearchError(f"no assignment met budget {frac} and threshold {threshold:.4f}")
    return SearchResult(list(best["windows"]), best["acc"], baseline, bud.fraction_used(best["widths"]), trace)


__all__ = ["SearchBudget", "SearchTrace", "SearchResult", "Evaluator", "window_signature", "parse_budget",
           "early_stop_check", "search_eco", "local_opt_km", "search_budget", "DEFAULT_CANDIDATE_WIDTHS"]
