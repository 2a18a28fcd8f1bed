"""serve.replay on the real kernels (GpuExecutor: plan -> per layer append + attention, timed
with CUDA events), the config-5 loop at a size that runs in seconds: every request reaches
its EOS, the KV blocks come back, the launch count is 2 per layer per iteration, the
attention launches are part of the iteration time, and the recorded descriptors are the
executed batches."""
import pytest

import paper_2503_22562_b200 as ny
from paper_2503_22562_b200 import serve
import workloads as W

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["niyama", "edf"])
def test_gpu_replay_small(name):
    s = W.L8B
    cfg = ny.Predictor.shape_cfg(s.num_q_heads, s.num_kv_heads, s.head_dim, "bf16")
    layers, blocks = 2, 4000
    ex = serve.GpuExecutor(s, layers, blocks, max_rows=2048 + 512)
    pred = ny.Predictor.from_params(cfg, list(ny.DEFAULT_THETA)).bind(ex.kv)
    fixed = layers * 9e-6
    ref = W.BatchDesc([0], [1536], [256], list(range(1, 65)), [2048] * 64)
    t_ref = fixed + layers * pred.predict(ref)
    sc = t_ref / 0.050
    buckets = [serve.QoSBucket(True, 6.0 * sc, 0.050 * sc), serve.QoSBucket(False, slo_ttlt=600.0 * sc),
               serve.QoSBucket(False, slo_ttlt=1800.0 * sc)]
    pol = {"niyama": dict(policy="niyama", preemption="selective", dynamic_chunk=True, relegation=True, alpha=0.0),
           "edf": dict(policy="edf", preemption="always", dynamic_chunk=False, fixed_chunk=256, relegation=False)}
    sched = ny.Scheduler(pred, max_chunk=2048, layers=layers, fixed_s=fixed, decode_token_s=t_ref,
                         history_min_samples=30, kv_token_budget=int(blocks * 16 * 0.9), **pol[name])
    trace = W.qos_trace(4.0 * sc, 8.0 / sc, seed=11, max_prompt=3000, max_decode=64)
    free0 = ex.kv.num_free()
    rec = []
    it, recs = serve.replay(sched, ex, trace, buckets, record=rec)
    assert len(trace) >= 10 and len(it) == len(rec) > 0
    assert all(len(r.tokens) == r.decode for r in recs.values())
    assert ex.launches == 2 * layers * len(it)
    assert ex.kv.num_free() == free0                      # every finished sequence released its blocks
    for x, d in zip(it, rec):
        assert 0.0 < x.attention_s < x.seconds
        assert x.prefill_tokens == int(d.pl.sum()) and x.decodes == len(d.ds)
    summ = serve.summarize(it, recs, buckets, fixed_s=fixed)
    assert summ["finished"] == len(trace)
    assert summ["predictor_rel_err_attention_only"]["p50"] < 0.5   # sanity: same order as measured
