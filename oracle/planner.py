"""ORACLE (test infrastructure only) -- the paper's partition planner, step by step.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline leg may
import this.  Shares no code with the CUDA path / C++ controller.

Follows PAPER.md §III-C in the paper's order and notation:
  Eq. 2  prop_v = t_v/(t_v+t_p), prop_p = t_p/(t_v+t_p)
  Eq. 1  E[t_e2e] = t_v(P_v) + t_p(P_p) + (prop_v t_d(P_v) + prop_p t_d(P_p)) L
  Eq. 3  argmin over valid contiguous partitions (enumeration, O(N^2))
  Eq. 4  Thr = 1/(t_v(P_v) + t_p(P_p))
  Pareto frontier    (Fig. fig:pareto): non-dominated (E2E, Thr) points
  Eq. 5  SM_dec = max(SM_min, SM_op - alpha (N_pend - 1))
Readings where the paper is silent (R9-R12): Eq. 3 ties -> more
SMs to decode; SM_min = smallest s with max(t_d^V(s), t_d^P(s)) <= tau t_d(all);
alpha = (SM_op - SM_min)/3 (reproduces the paper's 4 and 6 from P:488);
Eq. 5 floors to the granularity and uses max(N_pend, 1).
Pins: tests/test_oracle_planner.py (paper-printed values, brute force, closed forms).
"""
from __future__ import annotations

from dataclasses import dataclass
import math


def prop(t_v: float, t_p: float) -> tuple[float, float]:
    """Eq. 2."""
    return t_v / (t_v + t_p), t_p / (t_v + t_p)


def expected_e2e(t_v: float, t_p: float, td_v: float, td_p: float, L: float) -> float:
    """Eq. 1 (ideal pipeline, no queueing)."""
    pv, pp = prop(t_v, t_p)
    return t_v + t_p + (pv * td_v + pp * td_p) * L


def throughput(t_v: float, t_p: float) -> float:
    """Eq. 4 in requests per time unit of t_v, t_p."""
    return 1.0 / (t_v + t_p)


@dataclass(frozen=True)
class PlanPoint:
    s_v: int          # decode SMs while co-running with vision  (P_v)
    s_p: int          # decode SMs while co-running with prefill (P_p)
    e2e: float        # Eq. 1, ms
    thr: float        # Eq. 4, req/s (times in ms)


def enumerate_points(s: list[int], t_v: list[float], t_p: list[float], td_v: list[float],
                     td_p: list[float], L: float) -> list[PlanPoint]:
    """All (P_v, P_p) pairs of the split grid.  Curves are indexed by the decode
    split s[i]; the front stage runs on the complement (t_v[i] = t_v(total - s[i]))."""
    pts = []
    for i, sv in enumerate(s):
        for j, sp in enumerate(s):
            pts.append(PlanPoint(sv, sp, expected_e2e(t_v[i], t_p[j], td_v[i], td_p[j], L),
                                 1000.0 * throughput(t_v[i], t_p[j])))
    return pts


def optimal_static(points: list[PlanPoint]) -> PlanPoint:
    """Eq. 3: argmin E2E; ties -> larger s_v, then larger s_p."""
    best = None
    for p in points:
        if best is None or p.e2e < best.e2e or (p.e2e == best.e2e and (p.s_v, p.s_p) > (best.s_v, best.s_p)):
            best = p
    return best


def dominates(q: PlanPoint, p: PlanPoint) -> bool:
    return q.e2e <= p.e2e and q.thr >= p.thr and (q.e2e < p.e2e or q.thr > p.thr)


def pareto_frontier(points: list[PlanPoint]) -> list[PlanPoint]:
    """O(n^2) filter: keep points no other point dominates.  Sorted by Thr
    ascending, then E2E ascending; exact (E2E, Thr) duplicates kept once (larger split)."""
    keep = [p for p in points if not any(dominates(q, p) for q in points)]
    uniq: dict[tuple, PlanPoint] = {}
    for p in keep:
        k = (p.e2e, p.thr)
        if k not in uniq or (p.s_v, p.s_p) > (uniq[k].s_v, uniq[k].s_p):
            uniq[k] = p
    return sorted(uniq.values(), key=lambda p: (p.thr, p.e2e))


def sm_min_rule(s: list[int], td_v: list[float], td_p: list[float], td_full: float, tau: float = 2.5) -> int:
    """Smallest decode split whose co-run TBT stays within tau x the full-GPU decode time."""
    for i, si in enumerate(s):
        if max(td_v[i], td_p[i]) <= tau * td_full:
            return si
    return s[-1]


def alpha_rule(sm_op: int, sm_min: int) -> float:
    """alpha = (SM_op - SM_min)/3: SM_dec reaches SM_min at N_pend = 4."""
    return (sm_op - sm_min) / 3.0


def adaptive_sm(sm_op: int, sm_min: int, alpha: float, n_pend: int, granularity: int) -> int:
    """Eq. 5, floored to the partition granularity, clamped at SM_min."""
    raw = sm_op - alpha * (max(n_pend, 1) - 1)
    floored = int(math.floor(raw / granularity + 1e-9)) * granularity
    return max(sm_min, floored)


def frontier_pick(frontier, lam: float):
    """SURVEY.md §8(f) f3 frontier lookup (the paper motivates Eq. 5 by the Pareto frontier,
    P:356): among frontier points (s_v, s_p, e2e, thr) whose Eq. 4 throughput covers the arrival
    rate lam, the one with the lowest Eq. 1 E2E (ties: larger s_v, then s_p, as Eq. 3); if none
    covers lam, the highest throughput (ties: lower E2E)."""
    pts = [(p.s_v, p.s_p, p.e2e, p.thr) if hasattr(p, "s_v") else tuple(p[:4]) for p in frontier]
    ok = [p for p in pts if p[3] >= lam]
    if ok:
        return min(ok, key=lambda p: (p[2], -p[0], -p[1]))
    return max(pts, key=lambda p: (p[3], -p[2]))


def offload_floor(s, t_v, t_h2d_ms) -> int:
    """SURVEY.md §8(f) f3 with PAPER.md Eq. 8: under layer-wise offload a vision pass
    lasts at least the weight streaming time t_h2d; decode may take every split whose vision
    time on the remaining SMs is no slower than that bound (or than the best measured split),
    within 2% (R24).  Largest such s."""
    if not s:
        return 0
    bound = max(t_h2d_ms, min(t_v)) * 1.02
    return max(si for si, tv in zip(s, t_v) if tv <= bound)


def arrival_rate(times_ns) -> float:
    """req/s over a window of arrival times: (n - 1) / (t_last - t_first); 0 with < 2 arrivals."""
    if len(times_ns) < 2 or times_ns[-1] <= times_ns[0]:
        return 0.0
    return (len(times_ns) - 1) * 1e9 / (times_ns[-1] - times_ns[0])


def plan(s, t_v, t_p, td_v, td_p, L, td_full=None, tau=2.5):
    """Whole planner: points, frontier, Eq. 3 best, SM_min, alpha per context."""
    pts = enumerate_points(s, t_v, t_p, td_v, td_p, L)
    best = optimal_static(pts)
    front = pareto_frontier(pts)
    if td_full is None:
        td_full = min(min(td_v), min(td_p))
    smin = sm_min_rule(s, td_v, td_p, td_full, tau)
    smin = min(smin, best.s_v, best.s_p)
    return {"points": pts, "frontier": front, "best": best, "sm_min": smin,
            "alpha_dv": alpha_rule(best.s_v, smin), "alpha_dp": alpha_rule(best.s_p, smin)}


def mg1_wait(lam: float, ET: float, ET2: float) -> float:
    """Eq. 6: E[W_q] = lam E[T^2] / (2 (1 - lam E[T]))."""
    rho = lam * ET
    if rho >= 1.0:
        return math.inf
    return lam * ET2 / (2.0 * (1.0 - rho))
