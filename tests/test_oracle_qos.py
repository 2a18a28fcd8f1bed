"""Pins for oracle/qos.py (the §8(f)1 QoS scheduler core), CPU only.

Every pin is a SPEC worked example (cited) or a property the paper
states (§3.4), checked against brute force or a library routine.
"""
import itertools
import math

import numpy as np
import pytest

import workloads as W
from oracle import qos as Q

TBL3 = [Q.QoS(True, 6.0, 0.050), Q.QoS(False, slo_ttlt=600.0), Q.QoS(False, slo_ttlt=1800.0)]


def sched(**kw):
    model = kw.pop("model", Q.AffineModel(2e-3, 1.8e-5, 0.0))
    return Q.Scheduler(Q.Config(**kw), model)


def req(i, t, prompt, qos=TBL3[0], low=False, app=0, done=0):
    r = Q.Req(i, t, prompt, qos, low, app)
    r.prefill_done = done
    return r


# ---- decode-length history ----

def test_history_mean_plus_two_std():
    s = sched(decode_token_s=1.0, min_samples=30)
    for _ in range(15):
        s.hist.add(7, 80)
        s.hist.add(7, 120)                         # mean 100, std 20
    r = req(1, 0.0, 10, TBL3[1], app=7)
    assert s.decode_rem(r) == pytest.approx(140.0)                 # S:244 mean+2sigma, 0 decoded
    r.decoded = 200
    assert s.decode_rem(r) == 0.0                                  # S:245 clamp at zero
    assert s.decode_rem(req(2, 0.0, 10, TBL3[1], app=8)) == pytest.approx(415.0 + 600.0)   # S:246 prior


def test_history_welford_matches_numpy():
    g = np.random.default_rng(0)
    x = g.integers(1, 2000, size=500)
    h = Q.History()
    for v in x:
        h.add(0, int(v))
    cfg = Q.Config(min_samples=1)
    assert h.estimate(0, cfg) == pytest.approx(x.mean() + 2 * x.std(), rel=1e-12)


# ---- priorities ----

def test_alpha_zero_is_edf_permutation():
    """SPEC acceptance 1: alpha = 0 induces exactly the EDF order (random sets)."""
    g = np.random.default_rng(1)
    for trial in range(200):
        n = int(g.integers(1, 30))
        rs = [req(i, float(g.random() * 100), int(g.integers(1, 5000)), TBL3[int(g.integers(0, 3))],
                  done=0) for i in range(n)]
        a = sched(policy=Q.NIYAMA, alpha=0.0)
        e = sched(policy=Q.EDF)
        assert sorted(rs, key=a.priority) == sorted(rs, key=e.priority)


def test_alpha_large_is_srpf_permutation():
    """SPEC acceptance 1 / S:252: above alpha > (deadline spread)/(min work gap) the hybrid order
    equals SRPF on interactive sets with distinct remaining work (c0 = 0: Prefill_rem is c1 x tokens)."""
    g = np.random.default_rng(2)
    model = Q.AffineModel(0.0, 1e-4, 0.0)
    for trial in range(200):
        n = int(g.integers(2, 25))
        rem = g.choice(np.arange(1, 4000), size=n, replace=False)
        rs = [req(i, float(g.random() * 50), int(rem[i]) + 100, done=100) for i in range(n)]
        spread = max(r.t_arrival for r in rs) - min(r.t_arrival for r in rs)
        gap = min(abs(int(a) - int(b)) for a, b in itertools.combinations(rem, 2)) * 1e-4
        h = sched(policy=Q.NIYAMA, alpha=2 * spread / gap + 1.0, model=model)
        srpf = sched(policy=Q.SRPF, model=model)
        assert [r.id for r in sorted(rs, key=h.priority)] == [r.id for r in sorted(rs, key=srpf.priority)]


def test_priority_examples():
    s = sched(policy=Q.NIYAMA, alpha=1.0)
    a, b = req(1, 0.0, 100), req(2, 0.0, 1000)                      # S:251 same deadline, 100 vs 1000
    assert sorted([b, a], key=s.priority)[0] is a
    f = sched(policy=Q.FCFS)
    rs = [req(3, 3.0, 10), req(1, 1.0, 10), req(2, 2.0, 10)]
    assert [r.id for r in sorted(rs, key=f.priority)] == [1, 2, 3]
    e = sched(policy=Q.EDF)
    q2 = req(1, 0.0, 10, TBL3[1])
    q1 = req(2, 1.0, 10, TBL3[0])                                    # S:262 Q1 (6 s) after Q2 (600 s)
    assert sorted([q2, q1], key=e.priority)[0] is q1
    sr = sched(policy=Q.SRPF)
    half = req(1, 0.0, 1000, done=500)
    fresh = req(2, 0.0, 600)                                         # S:263 500 < 600
    assert sorted([fresh, half], key=sr.priority)[0] is half


# ---- violation checker ----

def test_check_violation_examples():
    s = sched()
    r = req(1, -1.0, 100, Q.QoS(True, 6.0, 0.05))                   # deadline 5 s
    assert s.status(r, 6.0) == Q.VIOLATED
    r2 = req(2, 0.0, 1000, Q.QoS(True, 6.0, 0.05))
    rem = s.prefill_rem(r2)
    assert rem == pytest.approx(2e-3 + 1.8e-5 * 1000)
    now = 6.0 - rem + 1e-9                                           # deadline = now + rem - eps
    assert s.status(r2, now) == Q.WILL_VIOLATE
    assert s.status(r2, 0.0) == Q.OK


# ---- eager relegation ----

def _violating(i, low):
    return req(i, -10.0, 100, Q.QoS(True, 6.0, 0.05), low=low)      # deadline -4 < now = 0


def test_relegation_examples():
    s = sched()
    s.submit(req(1, 0.0, 100))
    b = s.next_batch(0.0)
    assert b.relegated == []                                          # S:300 no violators
    s = sched()
    s.submit(_violating(1, low=False))
    s.submit(_violating(2, low=True))
    b = s.next_batch(0.0)
    assert b.relegated == [2]                                         # S:301 Low first
    assert s.reqs[1].state == "prefill"
    s = sched()
    s.submit(_violating(1, low=False))
    s.submit(req(3, 0.0, 50, low=True))                               # a Low request that is OK
    b = s.next_batch(0.0)
    assert b.relegated == [1]                                         # S:302 High when no Low violator


def test_relegated_service_order():
    s = sched()
    s.submit(_violating(1, low=True))
    s.submit(req(2, -20.0, 100, Q.QoS(True, 6.0, 0.05), low=True))  # earlier deadline (-14)
    b = s.next_batch(0.0)
    assert sorted(b.relegated) == [1, 2]
    assert [x[0] for x in b.slices] == [2, 1]                         # S:364 earlier deadline first (R28)
    s2 = sched()
    s2.submit(_violating(1, low=True))
    s2.next_batch(0.0)
    s2.complete(0.01, [])
    s2.submit(req(5, 0.01, 100))
    b = s2.next_batch(0.01)
    assert [x[0] for x in b.slices] == [5]                            # S:363 primary queue non-empty: no relegated service


# ---- selective preemption ----

def test_selective_preemption():
    # in-flight non-interactive prefill with a huge slack; urgent interactive arrives
    s = sched(max_chunk=100, policy=Q.EDF, relegation=False)
    s.submit(req(1, 0.0, 1000, TBL3[2]))
    s.next_batch(0.0)
    s.complete(0.01, [])
    assert s.inflight == 1
    s.submit(req(2, 0.01, 100, TBL3[0]))
    b = s.next_batch(0.01)
    assert b.slices[0][0] == 2                                        # S:313 preempted
    # displaced exactly at the WillViolate boundary -> not preempted
    s = sched(max_chunk=100, policy=Q.EDF, relegation=False)
    bulky = req(1, 0.0, 1000, Q.QoS(False, slo_ttlt=1e9))
    s.submit(bulky)
    s.next_batch(0.0)
    s.complete(0.0, [])
    rem = s.prefill_rem(bulky) + s.decode_rem(bulky)
    bulky.qos = Q.QoS(False, slo_ttlt=rem + 1e-9)                    # OK now, WillViolate one iteration later
    assert s.status(bulky, 0.0) == Q.OK
    s.submit(req(2, 0.0, 100, Q.QoS(True, 0.5e-9, 0.05)))             # earlier deadline
    b = s.next_batch(0.0)
    assert b.slices[0][0] == 1
    # never preempt: in-flight first; always: priority order
    for mode, first in ((Q.NEVER, 1), (Q.ALWAYS, 2)):
        s = sched(max_chunk=100, policy=Q.EDF, relegation=False, preemption=mode)
        s.submit(req(1, 0.0, 1000, TBL3[2]))
        s.next_batch(0.0)
        s.complete(0.01, [])
        s.submit(req(2, 0.01, 100, TBL3[0]))
        assert s.next_batch(0.01).slices[0][0] == first


# ---- batch assembly ----

def test_assemble_examples():
    s = sched()
    s.submit(req(1, 0.0, 300))
    b = s.next_batch(0.0)
    assert b.slices == [(1, 0, 300)] and b.budget == 2048
    s = sched(dynamic_chunk=False, fixed_chunk=500, policy=Q.FCFS)
    s.submit(req(1, 0.0, 400))
    s.submit(req(2, 1e-3, 900))
    b = s.next_batch(0.0)
    assert [(x[0], x[2]) for x in b.slices] == [(1, 400), (2, 100)]   # S:326 greedy fill


def test_budget_closed_form_chunk256():
    """S:114 / S:124: c0 = 2 ms, c1 = 0.018 ms; one interactive decode whose next-token deadline
    is c0 + c1 (256 + 1) away -> budget exactly 256 ("256-scale regime")."""
    s = sched(model=Q.AffineModel(2e-3, 1.8e-5, 0.0), relegation=False)
    d = req(1, 0.0, 10, Q.QoS(True, 2e-3 + 1.8e-5 * 257, 0.05))
    d.prefill_done, d.state = 10, "decode"
    s.reqs[1] = d
    s.submit(req(2, 0.0, 5000, TBL3[2]))
    b = s.next_batch(0.0)
    assert b.budget == 256 and b.slices == [(2, 0, 256)] and not b.infeasible
    assert b.predicted <= b.min_slack


# ---- completion ----

def test_lifecycle_examples():
    s = sched(relegation=False)
    s.submit(req(1, 0.0, 100))
    b = s.next_batch(0.0)
    assert b.decodes == []
    s.complete(0.05, [])
    assert s.reqs[1].state == "decode"                                 # S:332 decode queue next iteration
    t = 0.05
    for k in range(10):
        b = s.next_batch(t)
        assert b.decodes == [(1, 100 + k + 1)]                         # R4 ctx incl. the new token
        t += 0.05
        s.complete(t, [1] if k == 9 else [])
    r = s.reqs[1]
    assert r.state == "done" and r.decoded == 10
    assert np.allclose(np.diff(r.tokens), 0.05)                        # S:334 spaced 50 ms
    s = sched()
    s.submit(req(2, 0.0, 10))
    s.next_batch(0.0)
    s.complete(0.01, [])
    s.next_batch(0.01)
    s.complete(0.02, [2])                                               # S:333 decode_tokens = 1
    assert s.reqs[2].state == "done" and s.reqs[2].tokens == [0.02]
    with pytest.raises(ValueError):
        s.complete(0.03, [])


# ---- invariants over whole simulations (acceptance 2 and 9) ----

@pytest.mark.parametrize("qps,policy,dyn", [(2.0, Q.NIYAMA, True), (8.0, Q.NIYAMA, True), (8.0, Q.EDF, False),
                                            (8.0, Q.FCFS, False)])
def test_simulation_invariants(qps, policy, dyn):
    tr = W.qos_trace(60.0, qps, seed=3, max_prompt=4000, max_decode=300)
    model = Q.AffineModel(2e-3, 1.8e-5, 2e-9)
    pre = Q.SELECTIVE if policy == Q.NIYAMA else (Q.NEVER if policy == Q.FCFS else Q.ALWAYS)
    s = Q.Scheduler(Q.Config(policy=policy, alpha=0.5, dynamic_chunk=dyn, relegation=policy == Q.NIYAMA,
                             preemption=pre), model)
    seen_prefill = {}
    log = Q.simulate(s, tr, lambda b: TBL3[b])
    for now, b, dt in log:
        if dyn and b.decodes and math.isfinite(b.min_slack) and b.min_slack > 0:
            assert b.predicted <= b.min_slack * (1 + 1e-12)             # slack safety
        assert sum(n for _, _, n in b.slices) <= (2048 if dyn else 256)
        for rid, o, n in b.slices:
            assert n > 0 and o == seen_prefill.get(rid, 0)               # monotone progress
            seen_prefill[rid] = o + n
    assert all(r.state == "done" for r in s.reqs.values())              # conservation
    assert len(s.reqs) == len(tr)
    for r in s.reqs.values():
        t = next(x for x in tr if x.id == r.id)
        assert r.decoded == t.decode and len(r.tokens) == t.decode and r.prefill_done == r.prompt
        assert all(a < b for a, b in zip(r.tokens, r.tokens[1:]))


def test_trace_generator_properties():
    tr = W.qos_trace(3600.0, 1.0, seed=11)
    assert abs(len(tr) - 3600) <= 4 * 60                                # S:60 Poisson concentration
    assert W.qos_trace(3600.0, 1.0, seed=11) == tr                       # determinism
    tr = W.qos_trace(20000.0, 0.5, seed=12)
    share = np.bincount([r.bucket for r in tr], minlength=3) / len(tr)
    assert np.all(np.abs(share - 1 / 3) < 0.02)                          # S:61 thirds
    low = np.mean([r.low for r in tr])
    assert abs(low - 0.2) < 0.02
    assert abs(np.median([r.prompt for r in tr]) / 1730 - 1) < 0.05      # Table 1 p50
    sched_ = W.diurnal_schedule(3600.0, 2.0, 6.0)
    assert sched_ == [(0.0, 2.0), (900.0, 6.0), (1800.0, 2.0), (2700.0, 6.0)]
