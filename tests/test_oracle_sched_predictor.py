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
PER_TOKEN_BYTES = 8 * 128 * 2 * 2


def spec_theta(c0, c1, c2):
    """SPEC affine model as a feature-model parameter vector (module docstring)."""
    return np.array([c0, c1, c1, c2 / PER_TOKEN_BYTES, 0.0, 0.0])


def test_spec_cost_model_examples():
    cm = FX["cost_model"]
    th = spec_theta(cm["c0"], cm["c1"], cm["c2"])
    assert P.predict(th, P.features(SHAPE, [], [])) == pytest.approx(cm["c0"], abs=1e-15)
    t256 = P.predict(th, P.features(SHAPE, [(0, 256)], []))
    t2048 = P.predict(th, P.features(SHAPE, [(0, 2048)], []))
    assert t256 == pytest.approx(cm["chunk256_s"], rel=1e-12)
    assert t2048 == pytest.approx(cm["chunk2048_s"], rel=1e-12)
    assert (256 / t256) / (2048 / t2048) == pytest.approx(cm["throughput_ratio"], abs=5e-4)
    # S:115 linearity: one decode of kv_context_len 1000 adds exactly c1 + 1000*c2
    # (ctx counts the new token, R4: ctx = 1000 here is 1000 context tokens)
    th2 = spec_theta(cm["c0"], cm["c1"], cm["linearity"]["c2"])
    base = P.predict(th2, P.features(SHAPE, [(0, 256)], []))
    more = P.predict(th2, P.features(SHAPE, [(0, 256)], [1000]))
    assert more - base == pytest.approx(cm["c1"] + 1000 * cm["linearity"]["c2"], rel=1e-9)


def test_spec_max_feasible_chunk_examples():
    cm = FX["cost_model"]
    th = spec_theta(cm["c0"], cm["c1"], cm["c2"])
    assert P.max_feasible_chunk(th, SHAPE, [], 0, 10**6, math.inf, 2048) == (2048, False)
    assert P.max_feasible_chunk(th, SHAPE, [100], 0, 10**6, 0.001, 2048) == (0, True)
    assert P.max_feasible_chunk(th, SHAPE, [], 0, 10**6, cm["inverse"]["slack"], 2048) == (256, False)
    assert P.max_feasible_chunk(th, SHAPE, [], 0, 100, math.inf, 2048) == (100, False)          # remaining caps


def _samples(theta, n, seed):
    g = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        c = int(g.choice([0, 256, 512, 1024, 2048]))
        o = int(g.integers(0, 6000)) if c else 0
        D = int(g.integers(0, 257))
        L = int(g.integers(D, D * 4096 + 1)) if D else 0
        s = P.Sample(c, o, D, L, 1.0)
        s.seconds = float(theta @ P.features_sample(SHAPE, s))
        out.append(s)
    return out


def test_fit_recovers_known_theta():
    theta = np.array([4e-6, 2e-9, 5e-8, 1.1e-13, 3e-16, 0.9])
    samp = _samples(theta, 60, 1)
    got = P.fit(SHAPE, samp)
    pred = np.array([got @ P.features_sample(SHAPE, s) for s in samp])
    meas = np.array([s.seconds for s in samp])
    np.testing.assert_allclose(pred, meas, rtol=1e-8)


def test_fit_matches_bruteforce_active_set():
    """NNLS optimum == best feasible unconstrained LS over all 2^6 active sets."""
    theta = np.array([4e-6, -3e-9, 5e-8, 1.1e-13, 3e-16, 0.4])  # one negative truth -> clamped
    samp = _samples(theta, 50, 2)
    for s in samp:
        s.seconds = max(s.seconds, 1e-6)
    A = np.stack([P.features_sample(SHAPE, s) for s in samp])
    t = np.array([s.seconds for s in samp])
    A = A / t[:, None]
    colmax = np.abs(A).max(axis=0)
    An = A / colmax
    best, best_r = None, math.inf
    for mask in itertools.product([0, 1], repeat=P.NFEAT):
        idx = [i for i in range(P.NFEAT) if mask[i]]
        z = np.zeros(P.NFEAT)
        if idx:
            sol, *_ = np.linalg.lstsq(An[:, idx], np.ones(len(t)), rcond=None)
            if np.any(sol < -1e-12):
                continue
            z[idx] = np.maximum(sol, 0)
        r = float(np.sum((An @ z - 1.0) ** 2))
        if r < best_r - 1e-15:
            best, best_r = z, r
    got = P.fit(SHAPE, samp) * colmax
    assert float(np.sum((An @ got - 1.0) ** 2)) == pytest.approx(best_r, rel=1e-9, abs=1e-14)


def test_monotone_and_inverse_consistent():
    """t_hat non-decreasing in c, D, ctx; t(C) <= s < t(C+1) for interior C."""
    theta = np.array([4e-6, 2e-9, 5e-8, 1.1e-13, 3e-16, 0.9])
    g = np.random.default_rng(5)
    for _ in range(20):
        ctx = [int(x) for x in g.integers(1, 4097, size=int(g.integers(0, 40)))]
        o = int(g.integers(0, 4000))
        ts = [P.predict(theta, P.features(SHAPE, [(o, C)], ctx)) for C in range(0, 2049, 64)]
        assert all(b >= a for a, b in zip(ts, ts[1:]))
        slack = float(g.uniform(ts[0], ts[-1] * 1.2))
        C, inf = P.max_feasible_chunk(theta, SHAPE, ctx, o, 2048, slack, 2048)
        assert not inf
        assert P.predict(theta, P.features(SHAPE, [(o, C)], ctx)) <= slack * (1 + 1e-12)
        if C < 2048:
            assert P.predict(theta, P.features(SHAPE, [(o, C + 1)], ctx)) > slack
