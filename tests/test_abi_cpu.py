"""CPU tests of the C ABI (no GPU): libnova.so loads and exports every symbol the
headers declare; the pure-host planner (nova_plan, nova_adaptive_sm, Eq. 7/8)
matches the oracle; the C++ Algorithm 1 controller, run on the virtual-time Sim
backend, reproduces the oracle's decisions tick by tick (decision-log replay,
SURVEY.md §8(c) c3) and the hand-derived worked example."""
import os
import random
import re

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from oracle import planner as P
from oracle import scheduler as OS
from synth import TINY

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MS = 1_000_000


@pytest.fixture(scope="module")
def E():
    from paper_2509_21301_b200 import build
    build.build()
    from paper_2509_21301_b200 import engine
    return engine


def _declared_symbols():
    names = set()
    for h in ("nova.h", "nova_ops.h"):
        txt = open(os.path.join(ROOT, "include", h)).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        names |= set(re.findall(r"\b(nova_[a-z0-9_]+)\s*\(", txt))
    return names


def test_library_exports_every_declared_symbol(E):
    import ctypes
    from paper_2509_21301_b200._lib import LIB_PATH
    lb = ctypes.CDLL(LIB_PATH)
    syms = _declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lb, s)]
    assert missing == []


def test_planner_worked_example_and_eq5(E):
    r = E.nova_plan([8, 16, 24, 32], [100, 110, 125, 150], [40, 45, 52, 60], [12, 8, 6, 5.5], [14, 9, 7, 6], 10)
    assert r["best"][:2] == (16, 16) and round(r["best"][2], 3) == 237.903
    fr = sorted([(p[0], p[1]) for p in r["points"] if p[4]])
    assert fr == sorted([(16, 16), (16, 8), (8, 16), (8, 8)])
    assert [E.nova_adaptive_sm(24, 12, 4, n, 2) for n in range(1, 7)] == [24, 20, 16, 12, 12, 12]
    assert [E.nova_adaptive_sm(30, 12, 6, n, 2) for n in range(1, 6)] == [30, 24, 18, 12, 12]
    assert E.nova_next_logical_layer(6, 2, 64) == 8 and E.nova_next_logical_layer(63, 2, 64) == 1
    assert abs(E.nova_required_bandwidth(8e9, 0.5, 64, 2) - 16e9 * 62 / 62) < 1e-3


curve = st.lists(st.floats(1.0, 300.0, allow_nan=False), min_size=5, max_size=5)


@settings(max_examples=60, deadline=None)
@given(curve, curve, curve, curve, st.integers(1, 64))
def test_c_planner_matches_oracle(tv, tp, tdv, tdp, L):
    from paper_2509_21301_b200 import engine as E
    s = [8, 16, 24, 32, 40]
    c = E.nova_plan(s, tv, tp, tdv, tdp, L, tau=2.5, t_d_full=min(tdv + tdp))
    o = P.plan(s, tv, tp, tdv, tdp, L, td_full=min(tdv + tdp), tau=2.5)
    assert c["best"][:2] == (o["best"].s_v, o["best"].s_p)
    assert abs(c["best"][2] - o["best"].e2e) <= 1e-9 * o["best"].e2e
    cf = sorted((p[2], p[3]) for p in c["points"] if p[4])
    of = sorted((p.e2e, p.thr) for p in P.pareto_frontier(o["points"]))
    assert len(set(cf)) == len(of)
    assert all(abs(a[0] - b[0]) <= 1e-9 * b[0] for a, b in zip(sorted(set(cf)), of))
    assert c["sm_min"] == o["sm_min"]
    assert abs(c["alpha_dv"] - o["alpha_dv"]) < 1e-12 and abs(c["alpha_dp"] - o["alpha_dp"]) < 1e-12


def _sim_engine(E, mode, splits, tv, tp, tdv, tdp, solo, beta=0.0, **pol):
    e = E.Engine(TINY, E.EngineOptions(backend=E.BACKEND_SIM, max_requests=512, max_gen=512))
    e.sim_set_curves(splits, tv, tp, tdv, tdp, *solo, beta=beta)
    e.finalize()
    e.set_partition(mode, **pol)
    return e


@settings(max_examples=40, deadline=None)
@given(st.lists(st.floats(1.0, 50.0, allow_nan=False), min_size=6, max_size=6), st.floats(0.5, 200.0))
def test_c_offload_floor_matches_oracle(tv, th):
    from paper_2509_21301_b200 import engine as E
    s = [8, 16, 24, 32, 40, 48]
    tv = sorted(tv)
    assert E.nova_offload_floor(s, tv, th) == P.offload_floor(s, tv, th)


def test_sim_worked_example(E):
    for mode, want in [(E.ADAPTIVE, {1: [14, 15, 16], 2: [28, 29, 30]}), (E.SERIAL, {1: [14, 15, 26], 2: [30, 31, 32]})]:
        e = _sim_engine(E, mode, [8, 16], [10 * MS] * 2, [4 * MS] * 2, [MS] * 2, [MS] * 2, (10 * MS, 4 * MS, MS),
                        sm_op_dv=16, sm_op_dp=16, sm_min=8, alpha_dv=0, alpha_dp=0)
        ids = [e.submit(None, [1], 3, 0, grid=(4, 4)) for _ in range(2)]
        while e.step().events:
            pass
        got = {}
        for rid, idx, tok, t, fl in e.poll_tokens():
            got.setdefault(rid, []).append(t // MS)
        assert got == {ids[0]: want[1], ids[1]: want[2]}


def _replay(log, reqs, pol):
    """Feed the engine's logged events, tick by tick, to the oracle Alg. 1 and compare decisions."""
    alg = OS.Alg1(pol)
    for rid, g in reqs.items():
        if isinstance(g, tuple):   # (gen_len, S): CHUNK mode needs the prefill length
            alg.add_request(rid, g[0], g[1])
        else:
            alg.add_request(rid, g)
    ticks = {}
    for rec in log:
        ticks.setdefault(rec[0], []).append(rec)
    n_dec = 0
    for t in sorted(ticks):
        evs, decs = [], []
        for tick, is_ev, kind, ctx, s, ids, tns in ticks[t]:
            if is_ev:
                payload = list(ids) if kind in (OS.EV_DECODE_DONE, OS.EV_HYBRID_DONE) else ids[0]
                evs.append((kind, min(ids), payload, tns))
            else:
                decs.append((kind, tuple(ids), ctx, s))
        want = alg.tick(evs)
        assert decs == want, f"tick {t}"
        n_dec += len(decs)
    return n_dec


@pytest.mark.parametrize("mode", [0, 1, 2, 3, 4, 5])  # serial, static, adaptive, PF-Limit(5), multi-stream, frontier
@pytest.mark.parametrize("seed", [1, 2])
def test_sim_decision_log_replays_on_oracle(E, mode, seed):
    rnd = random.Random(seed)
    splits = [8 * k for k in range(1, 15)]
    tv = [int(9 * MS * 148 / (148 - s)) for s in splits]
    tp = [int(3 * MS * 148 / (148 - s)) for s in splits]
    td = [int(0.7 * MS * max(1.0, 32 / s)) for s in splits]
    pol = dict(sm_decode_dv=48, sm_decode_dp=40, sm_op_dv=64, sm_op_dp=56, sm_min=16, alpha_dv=16.0,
               alpha_dp=13.3, b_max=8, sm_dv_floor=40 if seed == 2 else 0)   # seed 2: offload-aware floor
    extra = {}
    if mode == OS.FRONTIER:   # Pareto frontier of the same curves (oracle planner), window 8
        ms = lambda xs: [x / MS for x in xs]
        fr = P.pareto_frontier(P.enumerate_points(splits, ms(tv), ms(tp), ms(td), ms(td), 8))
        extra = dict(frontier=[(p.s_v, p.s_p, p.e2e, p.thr) for p in fr], lam_window=8)
        e = E.Engine(TINY, E.EngineOptions(backend=E.BACKEND_SIM, max_requests=512, max_gen=512))
        e.sim_set_curves(splits, tv, tp, td, td, 9 * MS, 3 * MS, int(0.7 * MS), beta=0.03)
        e.finalize()
        e.set_frontier([(a, b, c, d, 1) for a, b, c, d in extra["frontier"]], window=8)
        e.set_partition(mode, **pol)
    else:
        e = _sim_engine(E, mode, splits, tv, tp, td, td, (9 * MS, 3 * MS, int(0.7 * MS)), beta=0.03, **pol)
    t, gens = 0, {}
    for i in range(120):
        t += int(rnd.expovariate(1 / 6.0) * MS) if rnd.random() < 0.8 else 0     # bursts of equal timestamps
        g = rnd.randint(1, 12)
        rid = e.submit(None, [1] * 4, g, t, grid=rnd.choice([(52, 94), (66, 120)]),
                       vis_scale=rnd.choice([1.0, 1.62]), pre_scale=rnd.uniform(0.9, 1.2))
        gens[rid] = g
    while e.step().events:
        pass
    log = e.decision_log()
    opol = OS.Policy(mode=mode, total_sms=148, granularity=8, **pol, **extra)
    n = _replay(log, gens, opol)
    fin = [r for r in log if not r[1] and r[2] == OS.D_FINISH]
    assert len(fin) == len(gens) and n > 3 * len(gens)
    toks = e.poll_tokens(100000)
    assert len(toks) == sum(gens.values())


@pytest.mark.parametrize("budget,seed", [(128, 1), (48, 2), (512 // 4, 3)])
def test_sim_chunk_mode_replays_on_oracle(E, budget, seed):
    """CHUNK (the paper's chunked-prefill baseline, R26): the C++ controller's decision
    log (hybrid passes with their chunk sizes) replays on the oracle state machine, every prefill
    token count is covered exactly by its chunks, and all tokens are emitted."""
    rnd = random.Random(seed)
    e = _sim_engine(E, E.CHUNK, [8, 16], [9 * MS] * 2, [3 * MS] * 2, [MS] * 2, [MS] * 2, (9 * MS, 3 * MS, int(0.7 * MS)),
                    beta=0.03, b_max=8, chunk_budget=budget)
    t, gens = 0, {}
    for i in range(40):
        t += int(rnd.expovariate(1 / 20.0) * MS) if rnd.random() < 0.8 else 0
        g = rnd.randint(1, 10)
        grid = rnd.choice([(8, 12), (52, 94), (4, 6)])
        npr = rnd.randint(1, 30)
        rid = e.submit(None, [1] * npr, g, t, grid=grid)
        gens[rid] = (g, (grid[0] // 2) * (grid[1] // 2) + npr)
    while e.step().events:
        pass
    log = e.decision_log()
    n = _replay(log, gens, OS.Policy(mode=OS.CHUNK, total_sms=148, granularity=8, b_max=8, chunk_budget=budget))
    hyb = [r for r in log if not r[1] and r[2] == OS.D_HYBRID]
    covered = {}
    for r in hyb:
        covered[r[5][0]] = covered.get(r[5][0], 0) + r[4]
        assert 1 <= r[4] <= budget and len(r[5]) - 1 <= 8
        assert r[4] <= max(1, budget - (len(r[5]) - 1))
    assert covered == {rid: gs[1] for rid, gs in gens.items()}
    assert n > len(gens)
    toks = e.poll_tokens(100000)
    assert len(toks) == sum(g for g, _ in gens.values())
    assert sorted(i for rid, i, *_ in toks if rid == min(gens)) == list(range(gens[min(gens)][0]))


def test_sim_chunk_matches_oracle_simulation_times(E):
    """CHUNK through the C++ Sim backend and oracle.scheduler.simulate: identical token times."""
    pol = dict(b_max=4, chunk_budget=64)
    e = _sim_engine(E, E.CHUNK, [8], [9 * MS], [3 * MS], [MS], [MS], (9 * MS, 3 * MS, MS), beta=0.05, **pol)
    rnd = random.Random(9)
    reqs, t = [], 0
    for i in range(25):
        t += int(rnd.expovariate(1 / 9.0) * MS)
        g = rnd.randint(1, 8)
        grid = rnd.choice([(8, 12), (16, 20)])
        rid = e.submit(None, [3, 4, 5], g, t, grid=grid)
        reqs.append(OS.SimRequest(rid, t, g, 1.0, 1.0, S=(grid[0] // 2) * (grid[1] // 2) + 3))
    while e.step().events:
        pass
    got = {}
    for rid, idx, tok, tt, fl in e.poll_tokens(10000):
        got.setdefault(rid, []).append(tt)
    _, want = OS.simulate(OS.Policy(mode=OS.CHUNK, **pol), OS.SimCurves([8], [9 * MS], [3 * MS], [MS], [MS], 9 * MS,
                                                                        3 * MS, MS, beta=0.05), reqs)
    assert got == want


def test_sim_matches_oracle_simulation_times(E):
    """Same trace through the C++ Sim backend and oracle.scheduler.simulate: identical token times."""
    splits = [8, 16, 24, 32]
    tv, tp = [12 * MS, 13 * MS, 15 * MS, 17 * MS], [4 * MS, 4 * MS, 5 * MS, 6 * MS]
    tdv, tdp = [3 * MS, 2 * MS, int(1.5 * MS), MS], [3 * MS, 2 * MS, int(1.6 * MS), MS]
    pol = dict(sm_op_dv=32, sm_op_dp=24, sm_min=8, alpha_dv=8.0, alpha_dp=5.4, b_max=4)
    e = _sim_engine(E, E.ADAPTIVE, splits, tv, tp, tdv, tdp, (10 * MS, 3 * MS, MS), beta=0.05, **pol)
    rnd = random.Random(5)
    reqs, t = [], 0
    for i in range(40):
        t += int(rnd.expovariate(1 / 7.0) * MS)
        g = rnd.randint(1, 9)
        vs = rnd.choice([1.0, 1.5])
        rid = e.submit(None, [3], g, t, grid=(4, 4), vis_scale=vs)
        reqs.append(OS.SimRequest(rid, t, g, vs, 1.0))
    while e.step().events:
        pass
    got = {}
    for rid, idx, tok, tt, fl in e.poll_tokens(10000):
        got.setdefault(rid, []).append(tt)
    _, want = OS.simulate(OS.Policy(mode=OS.ADAPTIVE, **pol), OS.SimCurves(splits, tv, tp, tdv, tdp, 10 * MS, 3 * MS,
                                                                          MS, beta=0.05), reqs)
    assert got == want


def test_submit_validation(E):
    e = _sim_engine(E, E.ADAPTIVE, [8], [MS], [MS], [MS], [MS], (MS, MS, MS))
    with pytest.raises(E.NovaError):
        e.submit(None, [1], 0, 0, grid=(4, 4))        # gen_len < 1
    with pytest.raises(E.NovaError):
        e.submit(None, [1], 2, 0, grid=(3, 4))        # not a multiple of patch*merge
    with pytest.raises(E.NovaError):
        e.set_partition(E.STATIC, sm_decode_dv=0, sm_decode_dp=8)


def test_finished_retention_and_release(E):
    """Bounded memory: finished requests beyond finished_retention are released
    oldest-first; nova_release_request frees one early; unfinished ones cannot be released."""
    e = E.Engine(TINY, E.EngineOptions(backend=E.BACKEND_SIM, max_requests=64, max_gen=64, finished_retention=3))
    e.sim_set_curves([8], [MS], [MS], [MS], [MS], MS, MS, MS)
    e.finalize()
    e.set_partition(E.SERIAL)
    ids = [e.submit(None, [1], 2, i * MS, grid=(4, 4)) for i in range(6)]
    late = e.submit(None, [1], 2, 10_000 * MS, grid=(4, 4))
    while e.step().finished < 6:
        pass
    for rid in ids[:3]:          # released by the retention bound
        with pytest.raises(E.NovaError):
            e.stats(rid)
    assert all(e.stats(rid)["finished"] for rid in ids[3:])
    e.release(ids[3])
    with pytest.raises(E.NovaError):
        e.stats(ids[3])
    with pytest.raises(E.NovaError):
        e.release(late)          # not finished yet
    assert e.stats(late)["finished"] == 0


def test_decision_log_ring_base(E):
    """The decision log is a bounded ring with absolute record indices (base 0 until it wraps)."""
    import ctypes as C
    from paper_2509_21301_b200 import _abi as A
    e = _sim_engine(E, E.SERIAL, [8], [MS], [MS], [MS], [MS], (MS, MS, MS))
    for i in range(4):
        e.submit(None, [1], 3, i * MS, grid=(4, 4))
    while e.step().events:
        pass
    assert e.lib.nova_decision_log_base(e.h) == 0
    log = e.decision_log()
    n, tot = A.I32(), A.I64()
    buf = (A.LogRecord * 8)()
    assert e.lib.nova_decision_log(e.h, 2, buf, 8, C.byref(n), C.byref(tot)) == 0
    assert tot.value == len(log) and n.value == 8 and buf[0].tick == log[2][0]
    assert e.lib.nova_decision_log(e.h, -1, buf, 8, C.byref(n), C.byref(tot)) != 0
