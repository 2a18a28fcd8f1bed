"""Config 5 — QoS trace replay (SURVEY §8(d) "Config 5 inputs"; §8(f) rank 1).

Three Table-3 tiers, ShareGPT lengths (Table 1), Poisson arrivals with
a diurnal low/high step, 20% low-priority requests.  The CPU scheduler
(niyama_sched_*) picks each iteration's batch and the real kernels run it through
n_layers layers on one B200 (paper_2503_22562_b200/serve.py).

Time scale: the engine is attention-only, so the SLOs are scaled by s = (predicted
iteration time of a 256-token chunk + 64 decodes at ctx ~2K) / 50 ms — the strict tier's
TBT becomes the time of that iteration, the way P:420 picked chunk 256 for 50 ms — and
every SLO, the diurnal period and the arrival rate scale with it.  Capacity (the
largest QPS with <= 1% violations) is searched on the predictor-driven simulator (no GPU);
the diurnal trace alternates 0.5x and 1.5x of it ("50% above capacity").

    python tools/replay_qos.py [--layers 32] [--phases 4] [--policies niyama,edf] [--out ...]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2503_22562_b200 as ny  # noqa: E402
from paper_2503_22562_b200 import serve  # noqa: E402
import workloads as W  # noqa: E402

POLICIES = {
    # Niyama: hybrid priority, dynamic chunking, eager relegation, selective preemption
    "niyama": dict(policy="niyama", preemption="selective", dynamic_chunk=True, relegation=True, alpha=0.0),
    # Sarathi-EDF: EDF, fixed chunk 256, no relegation
    "edf": dict(policy="edf", preemption="always", dynamic_chunk=False, fixed_chunk=256, relegation=False),
    # Sarathi-FCFS
    "fcfs": dict(policy="fcfs", preemption="never", dynamic_chunk=False, fixed_chunk=256, relegation=False),
}


def buckets_scaled(s):
    return [serve.QoSBucket(True, 6.0 * s, 0.050 * s), serve.QoSBucket(False, slo_ttlt=600.0 * s),
            serve.QoSBucket(False, slo_ttlt=1800.0 * s)]


def make_sched(pred, name, layers, fixed_s, decode_token_s):
    return ny.Scheduler(pred, max_chunk=2048, layers=layers, fixed_s=fixed_s, decode_token_s=decode_token_s,
                        history_min_samples=30, **POLICIES[name])


def capacity(pred, layers, fixed_s, s, buckets, duration, seed, lo, hi, tol, tdec):
    """S:395 bisection on uniform-load Poisson traces, predictor as the executor."""
    probes = []

    def viol(qps):
        tr = W.qos_trace(duration, qps, seed=seed, max_prompt=8192, max_decode=2048)
        sched = make_sched(pred, "niyama", layers, fixed_s, tdec)
        it, recs = serve.replay(sched, serve.ModelExecutor(pred, layers, fixed_s), tr, buckets, until=duration * 1.5)
        v = serve.summarize(it, recs, buckets, t_end=duration * 1.5)["violations_pct"]
        probes.append((qps, v))
        return v
    if viol(lo) > 1.0:
        return lo, probes
    while hi - lo > tol:
        mid = 0.5 * (lo + hi)
        if viol(mid) <= 1.0:
            lo = mid
        else:
            hi = mid
    return lo, probes


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--phases", type=int, default=4, help="diurnal phases (low, high, ...), 15 min x s each")
    ap.add_argument("--policies", default="niyama,edf")
    ap.add_argument("--seed", type=int, default=5)
    ap.add_argument("--capacity-only", action="store_true")
    ap.add_argument("--capacity", type=float, default=0.0, help="skip the search: use this capacity (QPS)")
    ap.add_argument("--model-only", action="store_true", help="replay on the predictor (no GPU)")
    ap.add_argument("--full", action="store_true",
                    help="full Llama-3-8B iterations: cuBLAS linear layers around every layer's append + attention, "
                         "scheduled with the full-iteration predictor (profiles/iteration_fit.json's sweep)")
    ap.add_argument("--calibrate", action="store_true",
                    help="after the runs, refit the attention predictor on the measured attention launches of the "
                         "first policy's replay (the engine's own profile, as Vidur profiling feeds the paper's "
                         "predictor) and replay every policy again with it (same trace)")
    ap.add_argument("--head-start-us", type=float, default=0.0,
                    help="GpuExecutor head start: the host enqueues each iteration before the GPU starts it, so the "
                         "replica clock and the attention times hold no host launch gaps (serve.py)")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "replay_config5.json"))
    args = ap.parse_args()
    shape = W.L8B
    cfg = ny.Predictor.shape_cfg(shape.num_q_heads, shape.num_kv_heads, shape.head_dim, "bf16")
    def make_pred(kv=None):
        p = ny.Predictor.from_params(cfg, list(ny.DEFAULT_THETA))
        if kv is not None:
            p.bind(kv)
        if args.full:
            sw = json.load(open(os.path.join(ROOT, json.load(open(os.path.join(ROOT, "profiles", "iteration_fit.json")))["sweep"])))
            lin = sorted(sw["linear"], key=lambda x: x["T"])
            p.set_iteration(args.layers, [x["T"] for x in lin], [x["seconds"] for x in lin])
            tr = [x for x in sw["points"] if (x["kind"] == "grid" and x["seed"] != 2) or x["kind"] == "random"]
            dd = [W.BatchDesc([0] if x["chunk"] else [], [x["offset"]] if x["chunk"] else [],
                              [x["chunk"]] if x["chunk"] else [], list(range(1, x["D"] + 1)), list(x["ctx"])) for x in tr]
            p.fit_iteration(dd, [x["seconds"] for x in tr])
        return p
    pred = make_pred()
    if args.full:   # the predictor returns whole iterations
        layers_s, fixed_s = 1, 0.0
    else:
        layers_s, fixed_s = args.layers, args.layers * 9e-6   # + per-layer KV append launch (profiles/r01)
    ref = W.BatchDesc([0], [1536], [256], list(range(1, 65)), [2048] * 64)
    t_ref = fixed_s + layers_s * pred.predict(ref)
    s = t_ref / 0.050
    buckets = buckets_scaled(s)
    tdec = t_ref                                        # R25: a decode iteration ~ the reference iteration
    out = {"layers": args.layers, "head_start_us": args.head_start_us, "engine": "full iteration (cuBLAS linear layers + attention)" if args.full
           else "attention-only (append + attention per layer)", "scale": s, "strict_tbt_s": 0.050 * s, "ttft_s": 6.0 * s,
           "ttlt_s": [600.0 * s, 1800.0 * s], "fixed_s_per_iteration": fixed_s, "reference_iteration_s": t_ref}
    t0 = time.time()
    if args.capacity > 0:
        cap, probes = args.capacity, "given (--capacity)"
    else:
        cap, probes = capacity(pred, layers_s, fixed_s, s, buckets, duration=3600.0 * s, seed=args.seed,
                               lo=0.5 / s, hi=20.0 / s, tol=0.05 / s, tdec=tdec)
    out["capacity_qps"] = cap
    out["capacity_probes"] = probes
    out["capacity_search_s"] = time.time() - t0
    print(json.dumps({k: out[k] for k in ("scale", "strict_tbt_s", "capacity_qps")}), flush=True)
    if args.capacity_only:
        json.dump(out, open(args.out, "w"), indent=1)
        return
    period = 900.0 * s
    duration = period * args.phases
    sched_qps = W.diurnal_schedule(duration, 0.5 * cap, 1.5 * cap, period)
    trace = W.qos_trace(duration, sched_qps, seed=args.seed + 1, max_prompt=8192, max_decode=2048)
    out["diurnal"] = {"period_s": period, "duration_s": duration, "qps": sched_qps, "requests": len(trace)}
    out["runs"] = {}
    gpu = None
    if not args.model_only:
        import torch  # noqa: F401
        blocks = 60000
        gpu = dict(blocks=blocks)
    cal = {"theta": None}
    recorded = []

    def run_policy(name, tag, theta):
        t1 = time.time()
        sched = make_sched(pred, name, layers_s, fixed_s, tdec)
        if args.model_only:
            ex = serve.ModelExecutor(pred, layers_s, fixed_s)
        else:
            linear = None
            if args.full:
                sys.path.insert(0, os.path.join(ROOT, "tools"))
                from sweep_iteration import LinearLayers
                linear = LinearLayers(max_t=2048 + 2048)
            ex = serve.GpuExecutor(shape, args.layers, gpu["blocks"], max_rows=2048 + 2048, linear=linear,
                                   head_start_us=args.head_start_us)
            pred_b = make_pred(ex.kv) if theta is None else ny.Predictor.from_params(cfg, theta).bind(ex.kv)
            sched = ny.Scheduler(pred_b, max_chunk=2048, layers=layers_s, fixed_s=fixed_s, decode_token_s=tdec,
                                 history_min_samples=30, kv_token_budget=int(gpu["blocks"] * 16 * 0.9),
                                 **POLICIES[name])
        rec = [] if (args.calibrate and theta is None and not recorded and not args.model_only) else None
        it, recs = serve.replay(sched, ex, trace, buckets, until=duration * 1.25, record=rec)
        if rec is not None:
            recorded.append((rec, [x.attention_s / args.layers for x in it]))
        summ = serve.summarize(it, recs, buckets, t_end=duration * 1.25, fixed_s=fixed_s)
        if args.full:   # the scheduler's prediction is the whole iteration: no attention-only comparison
            summ.pop("predictor_rel_err_attention_only", None)
        summ["wall_s"] = time.time() - t1
        if not args.model_only:
            summ["gpu_launches"] = ex.launches
        out["runs"][tag] = summ
        print(tag, json.dumps(summ), flush=True)
        os.makedirs(os.path.dirname(args.out), exist_ok=True)
        json.dump(out, open(args.out, "w"), indent=1)   # after every policy (long runs)
        del ex

    for name in args.policies.split(","):
        run_policy(name, name, None)
    if args.calibrate and recorded:
        descs, secs = recorded[0]
        keep = [i for i, x in enumerate(secs) if x == x and x > 0]
        step = max(1, len(keep) // 3000)
        keep = keep[::step]
        t1 = time.time()
        p_cal = ny.Predictor.fit_batches(cfg, [descs[i] for i in keep], [secs[i] for i in keep],
                                         start=list(ny.DEFAULT_THETA))
        cal["theta"] = [float(x) for x in p_cal.params()]
        err = np.abs([p_cal.predict(descs[i]) / secs[i] - 1.0 for i in keep])
        out["calibration"] = {"iterations": len(keep), "fit_s": time.time() - t1, "theta": cal["theta"],
                              "in_sample_rel_err": {"p50": float(np.median(err)), "p95": float(np.percentile(err, 95)),
                                                    "max": float(err.max())}}
        print("calibration", json.dumps(out["calibration"]["in_sample_rel_err"]), flush=True)
        for name in args.policies.split(","):
            run_policy(name, name + "@calibrated", cal["theta"])
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(out, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
