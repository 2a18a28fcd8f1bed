"""Pins for oracle/sched.py (a1) and oracle/predictor.py (a8) — CPU only.

Deadlines/slack against the SPEC worked examples (tests/golden/spec_examples.json,
anchored to PAPER Eq. 1-3 and Table 3); the predictor against SPEC's affine
cost-model examples (a special case of the feature model), exact recovery of a
known non-negative parameter vector, a brute-force active-set NNLS, and the
monotonicity / inverse-consistency invariants of S:136-137."""
import itertools
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
NONLIN = [1.7e-6, 55e9, 5.6e12]


def spec_theta(c0, c1, c2):
    """SPEC affine model as a schedule-model parameter vector (module docstring)."""
    return np.array([c0, c1, 0.0, c2, 0.0, 0.0] + NONLIN)


def test_spec_cost_model_examples():
    cm = FX["cost_model"]
    th = spec_theta(cm["c0"], cm["c1"], cm["c2"])
    assert P.predict(th, SHAPE, [], []) == pytest.approx(cm["c0"], abs=1e-15)
    t256 = P.predict(th, SHAPE, [(0, 256)], [])
    t2048 = P.predict(th, SHAPE, [(0, 2048)], [])
    assert t256 == pytest.approx(cm["chunk256_s"], rel=1e-12)
    assert t2048 == pytest.approx(cm["chunk2048_s"], rel=1e-12)
    assert (256 / t256) / (2048 / t2048) == pytest.approx(cm["throughput_ratio"], abs=5e-4)
    # S:115 linearity: one decode of kv_context_len 1000 adds exactly c1 + 1000*c2
    # (ctx counts the new token, R4: ctx = 1000 here is 1000 context tokens)
    th2 = spec_theta(cm["c0"], cm["c1"], cm["linearity"]["c2"])
    base = P.predict(th2, SHAPE, [(0, 256)], [])
    more = P.predict(th2, SHAPE, [(0, 256)], [1000])
    assert more - base == pytest.approx(cm["c1"] + 1000 * cm["linearity"]["c2"], rel=1e-9)


def test_spec_max_feasible_chunk_examples():
    cm = FX["cost_model"]
    th = spec_theta(cm["c0"], cm["c1"], cm["c2"])
    assert P.max_feasible_chunk(th, SHAPE, [], 0, 10**6, math.inf, 2048) == (2048, False)
    assert P.max_feasible_chunk(th, SHAPE, [100], 0, 10**6, 0.001, 2048) == (0, True)
    assert P.max_feasible_chunk(th, SHAPE, [], 0, 10**6, cm["inverse"]["slack"], 2048) == (256, False)
    assert P.max_feasible_chunk(th, SHAPE, [], 0, 100, math.inf, 2048) == (100, False)          # remaining caps
    assert P.largest_feasible_chunk(th, SHAPE, [], 0, 10**6, cm["inverse"]["slack"], 2048) == (256, False)


# ---- schedule model, step by step against hand-worked cases

def test_tile_queue_hand_worked():
    # TINY: g = 2 -> R = 64 rows per tile, Hkv = 2 copies of each tile
    assert P.tile_queue(TINY, [(0, 100)]) == [3, 3, 3, 3]          # keys 100 and 64 -> 1 step + 2 setup
    # slices sorted by o + c: (0, 300) [300 keys] before (100, 50) [150 keys]
    # (0,300): qt 4..0 see 300, 256, 192, 128, 64 keys -> 3, 2, 2, 1, 1 steps
    assert P.tile_queue(TINY, [(100, 50), (0, 300)]) == [5, 5, 4, 4, 4, 4, 3, 3, 3, 3, 4, 4]
    assert P.tile_queue(TINY, [(7, 0)]) == []                      # a zero-length slice is no slice
    # L8B: g = 4 -> R = 32; chunk 512 at 1536 -> 16 tiles x 8 heads, keys 2048 .. 1568
    q = P.tile_queue(SHAPE, [(1536, 512)])
    assert len(q) == 128 and q[:8] == [18] * 8 and q[-8:] == [15] * 8


def test_list_schedule_hand_worked():
    # worked by hand: machines (0,0,0) -> ... -> (16,16,14)
    assert P.list_schedule([5, 5, 4, 4, 4, 4, 3, 3, 3, 3, 4, 4], 3) == [14, 16, 16]
    assert P.list_schedule([7], 4) == [0, 0, 0, 7]
    assert P.list_schedule([], 3) == []
    costs = [9, 8, 7, 6, 5, 4, 3]
    assert sum(P.list_schedule(costs, 2)) == sum(costs)            # work is conserved


def test_split_len_and_cta_split_hand_worked():
    assert P.split_len(133674, 4096, 8) == 256        # ceil(1069392 / 4736) = 226 -> nearest 256
    assert P.split_len(77000, 4096, 8) == 128         # raw 131: 128 is nearer than 256
    assert P.split_len(100, 100, 1) == 128            # floor 128
    assert P.split_len(10**7, 8192, 8) == 16384       # ceil(8e7 / 4736) = 16892 -> nearest 16384
    assert P.split_len(10, 600000, 1) == 256          # ceil(600000/128) = 4688 > 4095 -> 256
    assert P.cta_split(4, 0, 12, 0, SHAPE) == (4, 4)
    assert P.cta_split(0, 600, 0, 133674, SHAPE) == (75, 0)
    # wp = 2074*160e3, wd = 133674*4096 -> 148 * 0.3768 = 55.8 -> 56 (floor 32)
    assert P.cta_split(128, 600, 2074, 133674, SHAPE) == (148, 56)
    assert P.cta_split(128, 600, 10, 133674, SHAPE) == (148, 32)   # tile-count floor ceil(128/4)
    # g = 8 (8 decode warps per CTA): wd weighs 1.8x -> wp = 331.84e6, wd = 985.55e6,
    # 148 * 0.25188 = 37.28 -> 38
    shape8 = P.PredShape(num_q_heads=64, num_kv_heads=8, head_dim=128, elt_bytes=2)
    assert P.cta_split(128, 600, 2074, 133674, shape8) == (148, 38)
    # config 4: wp = 59904*160e3 = 9.585e9, wd = 1048576*4096*1.8 = 7.731e9 -> 148 * 0.5535
    # = 81.9 -> 82; the floor is min(ceil(1024/4), ceil(148/2)) = 74
    assert P.cta_split(1024, 7168, 59904, 1048576, shape8) == (148, 82)


def test_fluid_decode_closed_forms():
    S0 = P.Sched(rows=0, D=2, sum_ctx=10, Bd=1e9, grid=100, np_=0, fin=[])
    np.testing.assert_allclose(P.phi(S0, 1e-6, 50e9, 6e12), [1, 2, 2, 10, 1e9 / 5e12, 0])   # min(BW, 100 r)
    # 20 prefill CTAs busy until 1e-4 s: 80 x 50 GB/s = 4 TB/s, then 5 TB/s
    S1 = P.Sched(rows=64, D=2, sum_ctx=10, Bd=1e9, grid=100, np_=20, fin=[100] * 20)
    np.testing.assert_allclose(P.phi(S1, 1e-6, 50e9, 6e12), [1, 66, 2, 10, 1e-4 + 6e8 / 5e12, 1e-4])
    S2 = P.Sched(rows=64, D=2, sum_ctx=10, Bd=1e8, grid=100, np_=20, fin=[100] * 20)
    np.testing.assert_allclose(P.phi(S2, 1e-6, 50e9, 6e12), [1, 66, 2, 10, 1e-4, 1e8 / 4e12])
    # staggered: k = 2, 3, then 4 CTAs at 1 GB/s: 1e5 + 1.5e5 bytes by 1e-4 s, 2.5e5 left at 4 GB/s
    S3 = P.Sched(rows=1, D=1, sum_ctx=1, Bd=5e5, grid=4, np_=2, fin=[50, 100])
    np.testing.assert_allclose(P.phi(S3, 1e-6, 1e9, 1e12), [1, 2, 1, 1, 1e-4 + 2.5e5 / 4e9, 1e-4])
    S4 = P.Sched(rows=1, D=0, sum_ctx=0, Bd=0.0, grid=4, np_=4, fin=[1, 2, 3, 4])
    np.testing.assert_allclose(P.phi(S4, 1e-6, 1e9, 1e12), [1, 1, 0, 0, 4e-6, 0])


def _samples(theta, n, seed):
    g = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        c = int(g.choice([0, 256, 512, 1024, 2048]))
        o = int(g.integers(0, 6000)) if c else 0
        D = int(g.integers(0, 257))
        if c == 0 and D == 0:
            D = 1
        L = int(g.integers(D, D * 4096 + 1)) if D else 0
        s = P.Sample(c, o, D, L, 1.0)
        s.seconds = P.predict(theta, SHAPE, *P.sample_batch(s))
        out.append(s)
    return out


GRID3 = (1.2e-6, 2.0e-6, 0.4e-6, 40e9, 60e9, 10e9, 5.6e12, 6.4e12, 0.4e12)


def test_fit_recovers_known_theta():
    theta = np.array([3e-5, 2e-9, 5e-8, 1.1e-10, 0.9, 0.2, 1.6e-6, 50e9, 6.0e12])
    samp = _samples(theta, 40, 1)
    got = P.fit(SHAPE, samp, GRID3)
    np.testing.assert_allclose(got[6:], theta[6:], rtol=1e-12)
    pred = np.array([P.predict(got, SHAPE, *P.sample_batch(s)) for s in samp])
    np.testing.assert_allclose(pred, [s.seconds for s in samp], rtol=1e-8)


def test_fit_matches_bruteforce_active_set():
    """At one grid point the NNLS optimum == best feasible unconstrained LS over all 2^6 active sets."""
    theta = np.array([3e-5, 2e-9, 5e-8, 1.1e-10, 0.9, 0.2, 1.6e-6, 50e9, 6.0e12])
    samp = _samples(theta, 40, 2)
    g = np.random.default_rng(3)
    for s in samp:
        s.seconds *= float(g.uniform(0.8, 1.2))       # noisy: some weights clamp at 0
    one = (1.6e-6, 1.6e-6, 1e-7, 50e9, 50e9, 1e9, 6e12, 6e12, 1e11)
    got = P.fit(SHAPE, samp, one)
    t = np.array([s.seconds for s in samp])
    Phi = np.stack([P.phi(P.schedule(SHAPE, *P.sample_batch(s)), 1.6e-6, 50e9, 6e12) for s in samp])
    A = Phi / t[:, None]
    colmax = np.abs(A).max(axis=0)
    An = A / colmax
    best_r = math.inf
    for mask in itertools.product([0, 1], repeat=P.NFEAT):
        idx = [i for i in range(P.NFEAT) if mask[i]]
        z = np.zeros(P.NFEAT)
        if idx:
            sol, *_ = np.linalg.lstsq(An[:, idx], np.ones(len(t)), rcond=None)
            if np.any(sol < -1e-12):
                continue
            z[idx] = np.maximum(sol, 0)
        best_r = min(best_r, float(np.sum((An @ z - 1.0) ** 2)))
    assert float(np.sum((A @ got[:6] - 1.0) ** 2)) == pytest.approx(best_r, rel=1e-9, abs=1e-14)


def test_bisection_inverse_consistent_and_largest_when_monotone():
    """t(C) <= s < t(C+1) for interior C; equals S:119's scan when t is monotone in C."""
    theta = np.array([3e-5, 2e-9, 5e-8, 1.1e-10, 0.9, 0.2, 1.6e-6, 50e9, 6.0e12])
    g = np.random.default_rng(5)
    for _ in range(8):
        ctx = [int(x) for x in g.integers(1, 4097, size=int(g.integers(0, 40)))]
        o = int(g.integers(0, 4000))
        cap = 300
        ts = [P.predict(theta, SHAPE, [(o, C)], ctx) for C in range(cap + 1)]
        slack = float(g.uniform(ts[0], ts[-1] * 1.2))
        C, inf = P.max_feasible_chunk(theta, SHAPE, ctx, o, cap, slack, 2048)
        assert not inf
        assert P.feasible(ts[C], slack)
        if C < cap:
            assert not P.feasible(ts[C + 1], slack)
        if all(b >= a for a, b in zip(ts, ts[1:])):
            assert (C, inf) == P.largest_feasible_chunk(theta, SHAPE, ctx, o, cap, slack, 2048)
