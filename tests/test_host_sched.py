"""§8(f)1 QoS scheduler core: the C++ scheduler (niyama_sched_*, through the C ABI)
against the oracle (oracle/qos.py) on the same traces, decision by decision.

Both use SPEC's affine cost model — for the C++ side the a8 predictor's
special case theta_lin = (c0, c1, 0, c2, 0, 0) (R16) — so every predicted
latency is the same fp64 expression on both sides and the batches must agree
exactly: slices, decodes, budget, infeasible flag, relegations, predicted latency,
min slack.  CPU only (the scheduler is host code).
"""
import math

import pytest

import paper_2503_22562_b200 as ny
import workloads as W
from oracle import qos as Q

C0, C1, C2 = 2e-3, 1.8e-5, 2e-9
TBL3 = [Q.QoS(True, 6.0, 0.050), Q.QoS(False, slo_ttlt=600.0), Q.QoS(False, slo_ttlt=1800.0)]


def affine_predictor():
    cfg = ny.Predictor.shape_cfg(32, 8, 128, "bf16")
    return ny.Predictor.from_params(cfg, [C0, C1, 0.0, C2, 0.0, 0.0] + list(ny.DEFAULT_THETA[6:]))


def scale_qos(q, s):
    return Q.QoS(q.interactive, q.slo_ttft * s, q.slo_tbt * s, q.slo_ttlt * s)


def run_both(trace, qos, cfg: Q.Config, max_iters=200000):
    """The SPEC event loop (oracle.qos.simulate's rules) driving both schedulers in lockstep."""
    pred = affine_predictor()
    cs = ny.Scheduler(pred, policy=cfg.policy, preemption=cfg.preemption, dynamic_chunk=cfg.dynamic_chunk,
                      fixed_chunk=cfg.fixed_chunk, max_chunk=cfg.max_chunk, relegation=cfg.relegation,
                      multi_fill=cfg.multi_fill, history_min_samples=cfg.min_samples, alpha=cfg.alpha,
                      prior_mean=cfg.prior_mean, prior_std=cfg.prior_std, decode_token_s=cfg.decode_token_s,
                      layers=cfg.layers, fixed_s=cfg.fixed_s, kv_token_budget=cfg.kv_token_budget)
    os_ = Q.Scheduler(cfg, Q.AffineModel(C0, C1, C2))
    reqs = sorted(trace, key=lambda r: (r.t_arrival, r.id))
    truth = {r.id: r.decode for r in reqs}
    now, i, iters = 0.0, 0, 0
    for _ in range(max_iters):
        while i < len(reqs) and reqs[i].t_arrival <= now:
            r = reqs[i]
            q = qos[r.bucket]
            cs.submit(r.id, r.t_arrival, r.prompt, q.interactive, q.slo_ttft, q.slo_tbt, q.slo_ttlt, r.low, r.app,
                      r.bucket)
            os_.submit(Q.Req(r.id, r.t_arrival, r.prompt, q, r.low, r.app))
            i += 1
        a = cs.next_batch(now)
        b = os_.next_batch(now)
        assert a.slices == b.slices, (iters, a.slices, b.slices)
        assert a.decodes == b.decodes, iters
        assert a.relegated == b.relegated, iters
        assert (a.budget, a.infeasible) == (b.budget, b.infeasible), iters
        assert a.predicted == b.predicted, iters
        assert a.min_slack == b.min_slack or (math.isinf(a.min_slack) and math.isinf(b.min_slack)), iters
        if a.empty:
            os_.last = None
            if i >= len(reqs):
                break
            now = max(now, reqs[i].t_arrival)
            continue
        iters += 1
        now += b.predicted
        fin = [rid for rid, _ in b.decodes if os_.reqs[rid].decoded + 1 == truth[rid]]
        cs.complete(now, fin)
        os_.complete(now, fin)
    for r in reqs:
        got = cs.request(r.id)
        want = os_.reqs[r.id]
        assert got["state"] == want.state and got["relegated"] == want.relegated
        assert got["decoded"] == want.decoded and got["prefill_done"] == want.prefill_done
    return iters, os_


@pytest.mark.parametrize("name,cfg,qps,scale", [
    ("niyama", Q.Config(alpha=0.5), 4.0, 0.05),
    ("niyama-overload", Q.Config(alpha=2.0), 30.0, 0.02),
    ("niyama-no-multifill", Q.Config(alpha=0.0, multi_fill=False), 12.0, 0.05),
    ("edf-fixed", Q.Config(policy=Q.EDF, dynamic_chunk=False, relegation=False, preemption=Q.ALWAYS), 12.0, 0.05),
    ("fcfs-fixed", Q.Config(policy=Q.FCFS, dynamic_chunk=False, relegation=False, preemption=Q.NEVER), 12.0, 0.05),
    ("srpf", Q.Config(policy=Q.SRPF, relegation=False, preemption=Q.ALWAYS), 12.0, 0.05),
    ("sjf-never", Q.Config(policy=Q.SJF, relegation=True, preemption=Q.NEVER), 12.0, 0.05),
    ("niyama-layers", Q.Config(alpha=0.5, layers=4.0, fixed_s=1e-4), 3.0, 0.1),
    ("niyama-kvbudget", Q.Config(alpha=0.5, kv_token_budget=60000), 12.0, 0.05),
])
def test_sched_matches_oracle(name, cfg, qps, scale):
    cfg.min_samples = 5
    cfg.decode_token_s = 0.01
    tr = W.qos_trace(20.0, qps, seed=7, max_prompt=3000, max_decode=200)
    qos = [scale_qos(q, scale) for q in TBL3]
    iters, os_ = run_both(tr, qos, cfg)
    assert iters > 100
    if name == "niyama-overload":
        assert any(r.relegated for r in os_.reqs.values())      # the overload case exercises relegation


def test_sched_validation_and_state_errors():
    pred = affine_predictor()
    s = ny.Scheduler(pred)
    with pytest.raises(ny.NiyamaError):
        s.submit(1, 0.0, 0, True, 6.0, 0.05)                   # prompt < 1
    s.submit(1, 0.0, 10, True, 6.0, 0.05)
    with pytest.raises(ny.NiyamaError):
        s.submit(1, 0.0, 10, True, 6.0, 0.05)                  # duplicate id
    with pytest.raises(ny.NiyamaError):
        s.complete(0.0, [])                                     # nothing outstanding
    b = s.next_batch(0.0)
    assert b.slices == [(1, 0, 10)] and not b.decodes
    with pytest.raises(ny.NiyamaError):
        s.next_batch(0.0)                                       # outstanding batch
    s.complete(0.01, [])
    b = s.next_batch(0.01)
    assert b.decodes == [(1, 11)]
    with pytest.raises(ny.NiyamaError):
        s.complete(0.02, [99])                                  # not a decode of the batch
    s.complete(0.02, [1])
    assert s.request(1)["state"] == "done" and s.counts()["done"] == 1
    assert s.next_batch(0.02).empty
    with pytest.raises(ny.NiyamaError):
        ny.Scheduler(pred, alpha=-1.0)


def test_sched_priority_and_status_through_abi():
    pred = affine_predictor()
    s = ny.Scheduler(pred, alpha=1.0)
    s.submit(1, 0.0, 1000, True, 6.0, 0.05)
    k, st = s.priority(1, 0.0)
    assert k == pytest.approx(6.0 + (C0 + C1 * 1000))          # Eq. 4 with Prefill_rem of one chunk
    assert st == 0
    assert s.priority(1, 7.0)[1] == 1                            # Violated (deadline 6 < 7)
    assert s.priority(1, 6.0 - (C0 + C1 * 1000) + 1e-9)[1] == 2  # WillViolate
