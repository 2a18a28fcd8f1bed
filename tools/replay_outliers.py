"""Where does the attention predictor miss on a served trace?  One config-5 replay (Niyama,
32 layers, the real kernels) records every batch descriptor with its measured attention
time; prints the error distribution by iteration shape and the worst iterations.

    python tools/replay_outliers.py [--phases 1] [--capacity 23.434] [--out gpurun_out/replay_outliers.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np  # noqa: E402

import paper_2503_22562_b200 as ny  # noqa: E402
from paper_2503_22562_b200 import serve  # noqa: E402
import workloads as W  # noqa: E402
from replay_qos import POLICIES, buckets_scaled  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--phases", type=int, default=1)
    ap.add_argument("--capacity", type=float, default=23.434116172784805)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--head-start-us", type=float, default=0.0, help="GpuExecutor head start (see serve.py)")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "replay_outliers.json"))
    args = ap.parse_args()
    s = W.L8B
    L = args.layers
    cfg = ny.Predictor.shape_cfg(s.num_q_heads, s.num_kv_heads, s.head_dim, "bf16")
    ex = serve.GpuExecutor(s, L, 60000, max_rows=2048 + 2048, head_start_us=args.head_start_us)
    pred = ny.Predictor.from_params(cfg, list(ny.DEFAULT_THETA)).bind(ex.kv)
    fixed = L * 9e-6
    ref = W.BatchDesc([0], [1536], [256], list(range(1, 65)), [2048] * 64)
    t_ref = fixed + L * ny.Predictor.from_params(cfg, list(ny.DEFAULT_THETA)).predict(ref)
    sc = t_ref / 0.050
    buckets = buckets_scaled(sc)
    period = 900.0 * sc
    dur = period * args.phases
    trace = W.qos_trace(dur, W.diurnal_schedule(dur, 0.5 * args.capacity, 1.5 * args.capacity, period), seed=6,
                        max_prompt=8192, max_decode=2048)
    sched = ny.Scheduler(pred, max_chunk=2048, layers=L, fixed_s=fixed, decode_token_s=t_ref, history_min_samples=30,
                         kv_token_budget=int(60000 * 16 * 0.9), **POLICIES["niyama"])
    rec = []
    it, _ = serve.replay(sched, ex, trace, buckets, until=dur * 1.25, record=rec)
    rows = []
    for k, (x, d) in enumerate(zip(it, rec)):
        meas = x.attention_s / L
        p = pred.predict(d)
        rows.append(dict(i=k, chunk=int(d.pl.sum()), slices=len(d.pl), D=len(d.ds),
                         sum_ctx=int(d.dc.sum()) if len(d.dc) else 0,
                         max_off=int((d.po + d.pl).max()) if len(d.pl) else 0, meas_us=meas * 1e6, pred_us=p * 1e6,
                         err=p / meas - 1.0))
    err = np.array([r["err"] for r in rows])
    print(f"{len(rows)} iterations: |err| p50 {np.median(np.abs(err)):.4f} p95 {np.percentile(np.abs(err), 95):.4f} "
          f"max {np.abs(err).max():.4f} mean {err.mean():+.4f}")
    groups = {}
    for r in rows:
        c = r["chunk"]
        cb = "0" if c == 0 else "1-64" if c <= 64 else "65-256" if c <= 256 else "257-1024" if c <= 1024 else ">1024"
        db = "D0" if r["D"] == 0 else "D1-8" if r["D"] <= 8 else "D9-32" if r["D"] <= 32 else "D>32"
        groups.setdefault((cb, db), []).append(r["err"])
    summ = {}
    for k in sorted(groups):
        e = np.array(groups[k])
        summ[f"{k[0]}|{k[1]}"] = dict(n=len(e), mean=float(e.mean()), p50=float(np.median(np.abs(e))),
                                      p95=float(np.percentile(np.abs(e), 95)), max=float(np.abs(e).max()))
        print(f"chunk {k[0]:>9} {k[1]:>6}: n {len(e):6d} mean {e.mean():+.4f} |err| p50 {np.median(np.abs(e)):.4f} "
              f"p95 {np.percentile(np.abs(e), 95):.4f} max {np.abs(e).max():.4f}")
    worst = sorted(rows, key=lambda r: -abs(r["err"]))[:25]
    for r in worst:
        print(json.dumps(r))
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump({"iterations": len(rows), "by_shape": summ, "worst": worst,
               "first_20": rows[:20]}, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
