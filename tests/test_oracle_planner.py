"""Pins for oracle/planner.py and oracle/offload.py (CPU only).

Paper-printed values (tests/golden/paper_pins.json), closed forms, brute force
on tiny candidate sets, and a hypothesis property against a sort-sweep
frontier (an independent algorithm).
"""
import itertools
import json
import math
import os

import pytest
from hypothesis import given, settings, strategies as st

from oracle import planner as P
from oracle import offload as O

PINS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_pins.json")))


def test_eq2_eq1_eq4_paper_values():
    sd = PINS["stage_duration_ms"]
    pv, pp = P.prop(sd["vision"], sd["prefill"])
    assert round(pv, 4) == 0.7134 and round(pp, 4) == 0.2866
    assert abs(pv + pp - 1) < 1e-15
    # Eq. 1 with t_d constant (28.9 ms) and L = 50
    assert round(P.expected_e2e(sd["vision"], sd["prefill"], sd["decode"], sd["decode"], 50), 1) == 2575.9
    thr = P.throughput(sd["vision"] / 1000, sd["prefill"] / 1000)
    assert round(thr, 3) == 0.884
    assert abs(thr * (sd["vision"] + sd["prefill"]) / 1000 - 1) < 1e-15


def test_eq5_paper_sequences():
    h = PINS["eq5_hyper"]
    g = h["granularity"]
    dv = [P.adaptive_sm(h["sm_op_dv"], h["sm_min"], h["alpha_dv"], n, g) for n in range(1, 7)]
    dp = [P.adaptive_sm(h["sm_op_dp"], h["sm_min"], h["alpha_dp"], n, g) for n in range(1, 6)]
    assert dv == [24, 20, 16, 12, 12, 12]
    assert dp == [30, 24, 18, 12, 12]
    # "SM_dec will drop to SM_min when the number of pending requests reaches 4"
    n4 = h["reaches_sm_min_at_n_pend"]
    assert P.adaptive_sm(h["sm_op_dv"], h["sm_min"], h["alpha_dv"], n4, g) == h["sm_min"]
    assert P.adaptive_sm(h["sm_op_dv"], h["sm_min"], h["alpha_dv"], n4 - 1, g) > h["sm_min"]
    # the alpha rule reproduces the paper's alphas
    assert P.alpha_rule(h["sm_op_dv"], h["sm_min"]) == h["alpha_dv"]
    assert P.alpha_rule(h["sm_op_dp"], h["sm_min"]) == h["alpha_dp"]
    assert P.adaptive_sm(24, 12, 4, 0, 2) == 24       # n = 0 treated as 1


TOY = dict(s=[8, 16, 24, 32], t_v=[100, 110, 125, 150], t_p=[40, 45, 52, 60],
           td_v=[12, 8, 6, 5.5], td_p=[14, 9, 7, 6], L=10)


def test_worked_example_planner():
    """SURVEY.md 8(c) c6 worked example, computed by hand."""
    r = P.plan(**TOY)
    b = r["best"]
    assert (b.s_v, b.s_p) == (16, 16)
    # by hand: t_v=110, t_p=45, prop_v=110/155 ; e2e = 155 + (110*8+45*9)/155*10
    assert abs(b.e2e - (155 + (110 * 8 + 45 * 9) / 155 * 10)) < 1e-12
    assert round(b.e2e, 3) == 237.903 and round(b.thr, 4) == 6.4516
    fr = [(p.s_v, p.s_p, round(p.e2e, 3)) for p in r["frontier"]]
    assert fr == [(16, 16, 237.903), (16, 8, 246.0), (8, 16, 255.69), (8, 8, 265.714)]
    # decode SMs non-increasing along the frontier as throughput rises
    sums = [p.s_v + p.s_p for p in r["frontier"]]
    assert sums == sorted(sums, reverse=True)


def _brute_best(points):
    m = min(p.e2e for p in points)
    return max((p for p in points if p.e2e == m), key=lambda p: (p.s_v, p.s_p))


def _sweep_frontier(points):
    """Independent algorithm: sort by e2e asc (thr desc), sweep keeping strictly better thr."""
    out, best_thr = [], -math.inf
    for p in sorted(points, key=lambda p: (p.e2e, -p.thr, -p.s_v, -p.s_p)):
        if p.thr > best_thr:
            out.append(p)
            best_thr = p.thr
    return sorted(out, key=lambda p: (p.thr, p.e2e))


curve = st.lists(st.floats(1.0, 500.0, allow_nan=False), min_size=4, max_size=4)


@settings(max_examples=200, deadline=None)
@given(curve, curve, curve, curve, st.integers(1, 80))
def test_frontier_and_eq3_properties(tv, tp, tdv, tdp, L):
    s = [8, 16, 24, 32]
    pts = P.enumerate_points(s, tv, tp, tdv, tdp, L)
    assert len(pts) == 16
    fr = P.pareto_frontier(pts)
    sw = _sweep_frontier(pts)
    assert [(p.e2e, p.thr) for p in fr] == [(p.e2e, p.thr) for p in sw]
    best = P.optimal_static(pts)
    assert best == _brute_best(pts)
    assert any(p.e2e == best.e2e and p.thr >= best.thr for p in fr)   # Eq. 3 point is on the frontier
    for p in fr:
        assert not any(P.dominates(q, p) for q in pts)


def test_sm_min_rule_reaches_paper_choice():
    # paper: SM_min = 12 keeps max TBT < 80 ms ~= 2.8 x 28.9 ms; toy curve with that shape
    s = [6, 8, 10, 12, 14]
    td = [120, 95, 81, 70, 60]
    assert P.sm_min_rule(s, td, td, 28.9, tau=80 / 28.9) == 12


def test_mg1_against_paper_table():
    t = PINS["mg1_table"]
    for lam, T, util, theory in zip(t["lambda"], t["T_s"], t["utilization"], t["theory_s"]):
        assert abs(lam * T - util) <= 0.011          # utilization row = lambda E[T]
        w = P.mg1_wait(lam, T, T * T)                # M/D/1 special case (E[T^2] = E[T]^2)
        if theory is None:
            assert math.isinf(w)                      # rho >= 1: no prediction ("\" in the table)
        else:
            assert abs(w - theory) / theory <= 0.08   # paper's E[T^2] is >= E[T]^2


def test_mg1_closed_forms():
    assert P.mg1_wait(0.0, 1.0, 1.0) == 0.0
    # M/M/1: E[T^2] = 2 E[T]^2 -> W_q = rho/(mu - lam)
    lam, mu = 0.5, 1.0
    assert abs(P.mg1_wait(lam, 1 / mu, 2 / mu ** 2) - (lam / mu) / (mu - lam)) < 1e-15


# ---------------------------------------------------------------- offload (Eq. 7, 8)
def test_eq7_sequences():
    assert O.next_logical_layer(6, 2, 64) == 8
    assert O.next_logical_layer(63, 2, 64) == 1
    # SURVEY 8(c) c6 worked example: K=2, L=4
    assert [x[2] for x in O.load_schedule(2, 4)] == [2, 3, 0, 1]
    # each physical slot cycles through every logical layer congruent to it mod gcd
    for K in (2, 3, 4, 5):
        seq = [O.next_logical_layer(l, K, 32) for l in range(32)]
        assert sorted(seq) == list(range(32))          # every pass loads all L layers once


def test_eq8_paper_value():
    e = PINS["eq8"]
    b = O.required_bandwidth(e["vit_bytes_GB"], e["forward_s_min"], 64, 2)
    assert b <= e["required_GBps_max"] and b > 0.99 * e["required_GBps_max"]
    assert abs(O.required_bandwidth(8, 0.5, 64, 33) - 8.0) < 1e-12
    assert b < e["pcie4_GBps"]


def test_offload_simulation_zero_stall_iff_bandwidth():
    L, K = 32, 2
    compute = [1.0] * L
    S = float(L)                    # 1 unit per layer
    T = sum(compute)
    need = O.required_bandwidth(S, T, L, K)
    _, stall_hi = O.simulate(compute, 1.0, need * 1.05, K, passes=1)
    assert stall_hi == 0
    _, stall_lo = O.simulate(compute, 1.0, need * 0.5, K, passes=1)
    assert stall_lo > 0
    # exact: with bw >= 1 layer per layer-time nothing ever stalls, over many passes
    _, st3 = O.simulate(compute, 1.0, 1.0, K, passes=3)
    assert st3 == 0


def test_layer_vision_memory_accounting():
    """Paper Table layer_vision: resident memory = K * layer_bytes + fixed (constant increments)."""
    t = PINS["layer_vision"]
    inc = [b - a for a, b in zip(t["mem_MB"], t["mem_MB"][1:])]
    assert max(inc) - min(inc) <= 0.1 + 1e-9          # printed to 0.1 MB
    per_layer = sum(inc) / len(inc)
    assert t["vit_layers"] * per_layer <= t["raw_MB"]  # the layer stack fits in the raw footprint


def test_frontier_lookup_pins():
    """Frontier-lookup controller against the paper's own planner pieces:
    at zero load it picks the Eq. 3 optimum (the global E2E minimum lies on the frontier); above
    every point's throughput it picks the highest-throughput point (the smallest front+prefill
    time, i.e. the fewest decode SMs here); picks are monotone in the arrival rate; and the rate
    estimate is exact on evenly spaced arrivals."""
    s = [8, 16, 24, 32]
    pts = P.enumerate_points(s, [100, 110, 125, 150], [40, 45, 52, 60], [12, 8, 6, 5.5], [14, 9, 7, 6], 10)
    fr = P.pareto_frontier(pts)
    best = P.optimal_static(pts)
    assert P.frontier_pick(fr, 0.0)[:2] == (best.s_v, best.s_p)
    top = max(pts, key=lambda p: p.thr)
    assert P.frontier_pick(fr, 1e9)[:2] == (top.s_v, top.s_p) == (8, 8)
    lams = [0.0, 5.0, 6.5, 7.0, 7.05, 7.15, 100.0]
    picks = [P.frontier_pick(fr, lam) for lam in lams]
    for a, b in zip(picks, picks[1:]):
        assert b[3] >= a[3] and b[2] >= a[2]
    for lam, p in zip(lams, picks):   # covers lam whenever some point does
        assert p[3] >= lam or all(q.thr < lam for q in fr)
    assert P.arrival_rate([0, 10_000_000, 20_000_000, 30_000_000]) == 100.0
    assert P.arrival_rate([5]) == 0.0


def test_offload_floor_pins():
    """Offload-aware split: with layer-wise offload a vision pass lasts at
    least its weight streaming time t_h2d (Eq. 8's premise).  The floor is the largest
    decode split whose vision pass on the remaining SMs still fits inside t_h2d: the pass is no
    slower there, and one split more would make it slower."""
    s = [8, 16, 24, 32, 40]
    tv = [10.0, 11.0, 12.5, 15.0, 19.0]
    assert P.offload_floor(s, tv, 12.6) == 24                 # 12.5 <= 12.6 * 1.02 < 15
    assert P.offload_floor(s, tv, 9.0) == 8                   # compute-bound: only the best split
    assert P.offload_floor(s, tv, 100.0) == 40
    # Eq. 8 numbers of the 7B ViT: 32 layers x 39.4 MB streamed at 55 GB/s
    t_h2d = 32 * 39.4e6 / 55e9 * 1e3          # ms
    f = P.offload_floor(s, [t_h2d * x for x in (0.5, 0.8, 0.99, 1.2, 1.5)], t_h2d)
    assert f == 24
    i = s.index(f)
    assert [0.5, 0.8, 0.99, 1.2, 1.5][i] <= 1.02 < [0.5, 0.8, 0.99, 1.2, 1.5][i + 1]
    # the measured B200 curve (profiles/r01_s3_offload.json, K = 2): flat at the PCIe bound to 56
    meas = [22.51, 22.63, 22.65, 22.71, 22.85, 22.87, 22.95, 24.15, 25.55, 30.65]
    assert P.offload_floor([8 * k for k in range(1, 11)], meas, 22.7) == 56
