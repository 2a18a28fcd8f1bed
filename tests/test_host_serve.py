"""serve.replay on the predictor-driven executor (no GPU): the serving loop of PAPER.md P:205
steps 1-7 with SPEC's event loop and report.  Checks what holds for any
trace: every request finishes, each request gets exactly its decode count of tokens at
non-decreasing times, the replica clock is the sum of the iteration times, the recorded
batch descriptors are the batches the executor ran (their prediction IS the iteration time
under ModelExecutor), and refitting the predictor on those descriptors against a known
scaling of the times recovers that scaling (the calibration replay_qos.py --calibrate does
on the GPU's measured launches)."""
import numpy as np
import pytest

import paper_2503_22562_b200 as ny
from paper_2503_22562_b200 import serve
import workloads as W


def _setup(seed=3, duration=6.0, qps=6.0, name="niyama"):
    s = W.L8B
    cfg = ny.Predictor.shape_cfg(s.num_q_heads, s.num_kv_heads, s.head_dim, "bf16")
    pred = ny.Predictor.from_params(cfg, list(ny.DEFAULT_THETA))
    layers, fixed = 32, 32 * 9e-6
    ref = W.BatchDesc([0], [1536], [256], list(range(1, 65)), [2048] * 64)
    t_ref = fixed + layers * pred.predict(ref)
    sc = t_ref / 0.050
    buckets = [serve.QoSBucket(True, 6.0 * sc, 0.050 * sc), serve.QoSBucket(False, slo_ttlt=600.0 * sc),
               serve.QoSBucket(False, slo_ttlt=1800.0 * sc)]
    pol = {"niyama": dict(policy="niyama", preemption="selective", dynamic_chunk=True, relegation=True, alpha=0.0),
           "edf": dict(policy="edf", preemption="always", dynamic_chunk=False, fixed_chunk=256, relegation=False)}
    sched = ny.Scheduler(pred, max_chunk=2048, layers=layers, fixed_s=fixed, decode_token_s=t_ref,
                         history_min_samples=30, **pol[name])
    trace = W.qos_trace(duration * sc, qps / sc, seed=seed, max_prompt=4096, max_decode=256)
    return cfg, pred, layers, fixed, buckets, sched, trace


@pytest.mark.parametrize("name", ["niyama", "edf"])
def test_replay_invariants_and_record(name):
    cfg, pred, layers, fixed, buckets, sched, trace = _setup(name=name)
    rec = []
    it, recs = serve.replay(sched, serve.ModelExecutor(pred, layers, fixed), trace, buckets, record=rec)
    assert len(trace) > 10 and len(recs) == len(trace)
    assert len(rec) == len(it) > 0
    for r in recs.values():
        assert len(r.tokens) == r.decode                        # every request ran to its EOS
        assert all(b >= a for a, b in zip(r.tokens, r.tokens[1:]))
        assert r.tokens[0] > r.t_arrival
    for a, b in zip(it, it[1:]):                                 # the clock never runs backwards
        assert b.t_start >= a.t_start + a.seconds - 1e-12
    for x, d in zip(it, rec):                                    # the recorded batch is the executed one
        assert x.seconds == pytest.approx(fixed + layers * pred.predict(d), rel=1e-12)
        assert x.prefill_tokens == int(d.pl.sum()) and x.decodes == len(d.ds)
    s = serve.summarize(it, recs, buckets, fixed_s=fixed)
    assert s["finished"] == len(trace) and s["iterations"] == len(it)
    assert sum(s["chunk_histogram"].values()) == len(it)


def test_replay_calibration_recovers_scaling():
    cfg, pred, layers, fixed, buckets, sched, trace = _setup(seed=4)
    rec = []
    it, _ = serve.replay(sched, serve.ModelExecutor(pred, layers, fixed), trace, buckets, record=rec)
    # "measured" attention per layer: the model's time x 1.08 (a uniformly slower device)
    secs = [1.08 * pred.predict(d) for d in rec]
    step = max(1, len(rec) // 400)
    p2 = ny.Predictor.fit_batches(cfg, rec[::step], secs[::step], start=list(ny.DEFAULT_THETA))
    err = np.array([p2.predict(d) / t - 1.0 for d, t in zip(rec, secs)])
    assert np.median(np.abs(err)) < 0.02 and abs(err.mean()) < 0.02
    # the uncalibrated predictor is off by the 8 % by construction
    err0 = np.array([pred.predict(d) / t - 1.0 for d, t in zip(rec, secs)])
    assert np.median(np.abs(err0)) > 0.07
