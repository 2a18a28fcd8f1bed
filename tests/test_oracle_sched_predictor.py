"""Pins for oracle/sched.py (a1) and oracle/predictor.py (a8) — CPU only.

Deadlines/slack against the SPEC worked examples (tests/golden/spec_examples.json,
anchored to PAPER Eq. 1-3 and Table 3); the predictor against SPEC's affine
cost-model examples (a special case of the model), hand-worked work queues,
closed forms of the event model, MEASURED per-CTA tile schedules of real
launches, and the inverse-consistency invariant of S:137."""
import json
import math
import os

import numpy as np
import pytest

from oracle import predictor as P
from oracle import sched as S

FX = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


@pytest.mark.parametrize("ex", FX["deadlines"], ids=lambda e: e["cite"])
def test_deadline_examples(ex):
    if ex["fn"] == "first":
        got = S.deadline_first(ex["t_arrival"], ex["slo_ttft"])
    elif ex["fn"] == "token":
        got = S.deadline_token(ex["t_arrival"], ex["slo_ttft"], ex["slo_tbt"], ex["n"])
    else:
        got = S.deadline_total(ex["t_arrival"], ex["slo_ttlt"])
    assert got == pytest.approx(ex["expect"], abs=1e-12)


def test_deadline_invariants():
    assert S.deadline_token(1.0, 6.0, 0.05, 1) == S.deadline_first(1.0, 6.0)       # S:188 n=1 reduces to Eq.1
    assert S.deadline_token(0, 6, 0.05, 2) - S.deadline_token(0, 6, 0.05, 1) == pytest.approx(0.05)
    with pytest.raises(ValueError):
        S.deadline_token(0, 6, 0.05, 0)


@pytest.mark.parametrize("ex", FX["slack"], ids=lambda e: e["cite"])
def test_slack_examples(ex):
    decs = [S.DecodeQoS(**d) for d in ex["decodes"]]
    got = S.min_slack(decs, ex["now"])
    if ex["expect"] == "inf":
        assert got == math.inf
    else:
        assert got == pytest.approx(ex["expect"], abs=1e-12)


SHAPE = P.PredShape(num_q_heads=32, num_kv_heads=8, head_dim=128, elt_bytes=2)
TINY = P.PredShape(num_q_heads=4, num_kv_heads=2, head_dim=64, elt_bytes=4, dtype="f32")
# event-model parameters (tau0, tau_p, tau_d, sigma, r_w, u0, BW, gamma, r_cta, sigma0)
NL = [0.9e-6, 0.05e-6, 0.2e-6, 9.0, 70e9, 1e-9, 8.8e12, 0.15, 96e9, 1.0]


def spec_theta(c0, c1, c2):
    """SPEC affine model as a predictor parameter vector (module docstring)."""
    return np.array([c0, c1, 0.0, c2, 0.0, 0.0] + NL)


def L8(grid=148, np_=0, q=128, small=128):
    return P.Launch(q, small, grid, np_, 12)


def test_spec_cost_model_examples():
    cm = FX["cost_model"]
    th = spec_theta(cm["c0"], cm["c1"], cm["c2"])
    ev = lambda sl, ctx: P.predict(th, P.work(SHAPE, sl, ctx, 128, 128), L8(np_=1 if sl else 0))  # noqa: E731
    assert ev([], []) == pytest.approx(cm["c0"], abs=1e-15)
    t256, t2048 = ev([(0, 256)], []), ev([(0, 2048)], [])
    assert t256 == pytest.approx(cm["chunk256_s"], rel=1e-12)
    assert t2048 == pytest.approx(cm["chunk2048_s"], rel=1e-12)
    assert (256 / t256) / (2048 / t2048) == pytest.approx(cm["throughput_ratio"], abs=5e-4)
    assert t256 == P.affine(cm["c0"], cm["c1"], cm["c2"], [(0, 256)], [])
    # S:115 linearity: one decode of kv_context_len 1000 adds exactly c1 + 1000*c2 (R4: ctx = 1000)
    th2 = spec_theta(cm["c0"], cm["c1"], cm["linearity"]["c2"])
    base = P.predict(th2, P.work(SHAPE, [(0, 256)], [], 128, 128), L8(np_=1))
    more = P.predict(th2, P.work(SHAPE, [(0, 256)], [1000], 128, 128), L8(np_=1))
    assert more - base == pytest.approx(cm["c1"] + 1000 * cm["linearity"]["c2"], rel=1e-9)


def test_spec_max_feasible_chunk_examples():
    cm = FX["cost_model"]

    def t_of(ctx):
        return lambda C: P.affine(cm["c0"], cm["c1"], cm["c2"], [(0, C)] if C else [], ctx)
    assert P.max_feasible_chunk(t_of([]), 10**6, math.inf, 2048) == (2048, False)
    assert P.max_feasible_chunk(t_of([100]), 10**6, 0.001, 2048) == (0, True)
    assert P.max_feasible_chunk(t_of([]), 10**6, cm["inverse"]["slack"], 2048) == (256, False)
    assert P.max_feasible_chunk(t_of([]), 100, math.inf, 2048) == (100, False)                   # remaining caps
    assert P.largest_feasible_chunk(t_of([]), 10**6, cm["inverse"]["slack"], 2048) == (256, False)


# ---- steps 1-2: the work of a batch, hand-worked (causal key ranges; row pieces)

def test_work_hand_worked():
    # TINY: g = 2 -> R = 64 rows per tile; slice (0, 100): q tiles see 100 and 64 keys -> 1 step each, x Hkv 2
    assert P.work(TINY, [(0, 100)], [], 128, 128).tiles == [1, 1, 1, 1]
    # slices by o + c: (0, 300) first (qt 4..0 see 300, 256, 192, 128, 64 keys -> 3, 2, 2, 1, 1), then (100, 50)
    assert P.work(TINY, [(100, 50), (0, 300)], [], 128, 128).tiles == [3, 3, 2, 2, 2, 2, 1, 1, 1, 1, 2, 2]
    assert P.work(TINY, [(7, 0)], [], 128, 128).tiles == []
    # L8B: g = 4 -> R = 32; chunk 512 at 1536 -> 16 tiles x 8 heads, keys 2048 .. 1568 -> 16 .. 13 steps
    w = P.work(SHAPE, [(1536, 512)], [], 128, 128)
    assert len(w.tiles) == 128 and w.tiles[:8] == [16] * 8 and w.tiles[-8:] == [13] * 8
    # decode rows 300 and 129 at q = 128, small = 64 (TINY: Hkv 2, 64 dims x 2 x 4 B = 512 B per token):
    # full pieces 128, 128 (row 300), 128 (row 129); tails 44 (300 - 256) and 1 -> 44, 1
    w = P.work(TINY, [], [129, 300], 128, 64)
    assert w.pieces == [128 * 512.0] * 6 + [44 * 512.0] * 2 + [1 * 512.0] * 2
    assert w.units == 10 and w.sum_ctx == 429 and w.D == 2
    w = P.work(TINY, [], [300], 128, 16)                       # tail 44 keys in 16-key pieces: 16, 16, 12
    assert w.pieces == [128 * 512.0] * 4 + [16 * 512.0] * 4 + [12 * 512.0] * 2


def test_tiles_per_cta_list_schedule():
    w = P.Work(0, 0, 0, 0, tiles=[5, 5, 4, 4, 4, 4, 3, 3, 3, 3, 4, 4], pieces=[])
    # by hand: CTAs (0,0,0) -> 5,5,4 -> 8(+4 on CTA 2)... each tile to the CTA free first
    assert sorted(P.tiles_per_cta(w, L8(np_=3))) == [4, 4, 4]
    assert P.tiles_per_cta(P.Work(0, 0, 0, 0, tiles=[7], pieces=[]), L8(np_=4)) == [1, 0, 0, 0]
    assert sum(P.tiles_per_cta(w, L8(np_=5))) == len(w.tiles)


# ---- step 3: the event model against closed forms

def test_event_model_closed_forms():
    nl = dict(zip(["tau0", "tau_p", "tau_d", "sigma", "r_w", "u0", "bw", "gamma", "r_cta", "sigma0"], NL))
    v = list(NL)
    # (a) prefill only, n <= n_p equal tiles of s steps: all first tiles end together at s + sigma0 steps
    #     of tau0 + tau_p n / NSM
    w = P.Work(64, 0, 0, 0, tiles=[12] * 40, pieces=[])
    assert P.simulate(w, L8(grid=40, np_=40), v) == pytest.approx((12 + nl["sigma0"]) * (nl["tau0"] + nl["tau_p"] * 40 / 148), rel=1e-12)
    # (b) decode only, n <= W equal units of b bytes: rate min(r_w, BW / n, r_cta grid / n)
    b = 64 * 1024.0
    for n, grid in ((100, 148), (1776, 148), (24, 2)):
        w = P.Work(0, 1, 1, n, tiles=[], pieces=[b] * n)
        rate = min(nl["r_w"], nl["bw"] / n, nl["r_cta"] * grid / n)
        assert P.simulate(w, L8(grid=grid), v) == pytest.approx((b + nl["u0"] * nl["r_w"]) / rate, rel=1e-12)
    # (c) two rounds: 2 W units on W warps take twice as long
    w = P.Work(0, 1, 1, 48, tiles=[], pieces=[b] * 48)
    rate = min(nl["r_w"], nl["bw"] / 24, nl["r_cta"] * 2 / 24)
    assert P.simulate(w, L8(grid=2), v) == pytest.approx(2 * (b + nl["u0"] * nl["r_w"]) / rate, rel=1e-12)
    # (d) a prefill CTA's warps join when its tile ends; no coupling (tau_d = gamma = 0, r_w binds):
    #     grid 2, n_p 1, one warp per CTA: warp A runs unit 1 from 0; the tile ends at tp; the
    #     prefill CTA's warp runs unit 2 from tp (tp < the unit time, so warp A is still busy)
    v0 = [nl["tau0"], 0.0, 1e-30, nl["sigma"], 10e9, 0.0, 1e15, 1e-30, 1e15, nl["sigma0"]]
    w = P.Work(32, 2, 2, 2, tiles=[2], pieces=[b, b])
    tp = (2 + nl["sigma0"]) * nl["tau0"]
    tu = b / 10e9
    assert P.simulate(w, P.Launch(128, 128, 2, 1, 1), v0) == pytest.approx(tp + tu, rel=1e-9)
    # (e) coupling: one long unit streams while the tile runs (B = 1 of W = 2 warps) -> step time
    #     tau0 + tau_d / 2; the unit (rate r_w / (1 + gamma / NSM) during the tile) outlasts it
    v1 = [1e-6, 1e-30, 0.4e-6, 0.0 + 1e-30, 1e9, 0.0, 1e15, 0.3, 1e15, 5.0]
    w = P.Work(32, 1, 1, 1, tiles=[10], pieces=[1e6])
    tp = 15 * (1e-6 + 0.4e-6 / 2)
    done = tp * 1e9 / (1 + 0.3 / 148)
    assert P.simulate(w, P.Launch(128, 128, 2, 1, 1), v1) == pytest.approx(tp + (1e6 - done) / 1e9, rel=1e-9)
    # (f) empty batch: T_sim = 0, t_hat = c0
    assert P.predict(spec_theta(3e-5, 1e-9, 1e-10), P.Work(0, 0, 0, 0, [], []), L8()) == pytest.approx(3e-5)


def test_trace_pin_tile_schedule():
    """MEASURED per-CTA tile counts (tests/golden/launch_traces_l8b.json, niyama_debug_trace of 73
    config-3 launches on B200, tools/make_trace_fixture.py) against the model's list schedule of the
    tile queue: the prefill CTA count and the tile total always agree, launches with <= 2 tiles per
    CTA agree exactly, and no CTA runs more than 2 tiles more or fewer than the model says (the real
    CTAs do not all advance at one rate: ~18 CTAs run 1 tile more, ~18 one less)."""
    fx = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "launch_traces_l8b.json")))
    exact = 0
    for L in fx["launches"]:
        q = L["split_len"]
        w = P.work(SHAPE, [(L["offset"], L["chunk"])], L["ctx"], q, min(q, max(256, q // 4)))
        m = P.tiles_per_cta(w, P.Launch(q, 0, 148, L["prefill_ctas"], 12))
        meas = {int(k): v for k, v in L["measured_tiles_per_cta_hist"].items()}
        assert sum(meas.values()) == L["prefill_ctas"] == len(m)
        assert sum(k * v for k, v in meas.items()) == len(w.tiles) == L["tiles"]
        assert min(meas) >= min(m) - 2 and max(meas) <= max(m) + 2
        hm = {}
        for k in m:
            hm[k] = hm.get(k, 0) + 1
        if max(m) <= 2:
            assert hm == meas
        exact += hm == meas
    assert len(fx["launches"]) >= 70 and exact >= 50


def test_bisection_inverse_consistent_and_largest_when_monotone():
    """t(C) <= s < t(C+1) for interior C; equals S:119's scan when t is monotone in C."""
    theta = np.array([1.7e-5, 2.5e-9, 0.0, 1e-10, 6e-10, 1.0] + NL)
    g = np.random.default_rng(5)
    for _ in range(4):
        ctx = [int(x) for x in g.integers(1, 4097, size=int(g.integers(0, 30)))]
        o = int(g.integers(0, 4000))
        cap = 120

        def t_of(C):
            q = 128
            return P.predict(theta, P.work(SHAPE, [(o, C)] if C else [], ctx, q, q), L8(np_=min(148, max(1, C // 4)) if C else 0))
        ts = [t_of(C) for C in range(cap + 1)]
        slack = float(g.uniform(ts[0], ts[-1] * 1.2))
        C, inf = P.max_feasible_chunk(t_of, cap, slack, 2048)
        assert not inf
        assert P.feasible(ts[C], slack)
        if C < cap:
            assert not P.feasible(ts[C + 1], slack)
        if all(b >= a for a, b in zip(ts, ts[1:])):
            assert (C, inf) == P.largest_feasible_chunk(t_of, cap, slack, 2048)
