"""§8(f) rank 4 — full-iteration predictor and the Fig. 4 analogue, from tools/sweep_iteration.py
(CPU only).

Predictors compared on the same held-out points (grid seed 2 + off-grid; training = grid
seeds 0, 1 + random):
  * analytic (the library's): measured linear-layer table lin(T) + layers x the attention
    event model (profiles/predictor_fit.json) + c0 + c1 T fitted by least squares
    (niyama_predictor_set_iteration / niyama_predictor_fit_iteration);
  * random forest on (c, o, D, sum ctx, max ctx, T) — the paper's predictor family (P:319
    "random forest on Vidur profiles"), scikit-learn, log-time target;
  * lookup table (P:744 draft "profile lookup table"): nearest training point in
    normalised (c, D, sum ctx) space, scaled by T.
Fig. 4 analogue ("28% lower" throughput at small chunk): full-iteration
tokens/s against chunk size, mean over the grid's decode counts and seeds.

    python tools/fit_iteration.py gpurun_out/iteration_sweep.json [--out profiles/iteration_fit.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2503_22562_b200 as ny  # noqa: E402
import workloads as W  # noqa: E402


def desc(r):
    c = r["chunk"]
    return W.BatchDesc(prefill_seq=[0] if c else [], prefill_offset=[r["offset"]] if c else [],
                       prefill_len=[c] if c else [], decode_seq=list(range(1, r["D"] + 1)), decode_ctx=list(r["ctx"]))


def stats(e):
    e = np.abs(np.asarray(e))
    return {"p50": float(np.median(e)), "p95": float(np.percentile(e, 95)), "max": float(e.max()), "n": int(len(e))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("sweep")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "iteration_fit.json"))
    args = ap.parse_args()
    sw = json.load(open(args.sweep))
    pts = sw["points"]
    train = [r for r in pts if (r["kind"] == "grid" and r["seed"] != 2) or r["kind"] == "random"]
    held = [r for r in pts if r["kind"] == "offgrid" or (r["kind"] == "grid" and r["seed"] == 2)]
    fit = json.load(open(os.path.join(ROOT, "profiles", "predictor_fit.json")))
    cfg = ny.Predictor.shape_cfg(32, 8, 128, "bf16")
    pr = ny.Predictor.from_params(cfg, fit["theta"])
    lin = sorted(sw["linear"], key=lambda x: x["T"])
    pr.set_iteration(sw["layers"], [x["T"] for x in lin], [x["seconds"] for x in lin])
    pr.fit_iteration([desc(r) for r in train], [r["seconds"] for r in train])
    analytic = {id(r): pr.predict(desc(r)) for r in pts}
    res = {"analytic": {"train": stats([analytic[id(r)] / r["seconds"] - 1 for r in train]),
                        "heldout": stats([analytic[id(r)] / r["seconds"] - 1 for r in held])}}
    # attention share of the iteration (what the linear layers dilute)
    pr0 = ny.Predictor.from_params(cfg, fit["theta"])
    share = [sw["layers"] * pr0.predict(desc(r)) / r["seconds"] for r in pts]

    def feats(r):
        return [r["chunk"], r["offset"], r["D"], r["sum_ctx"], max(r["ctx"]) if r["ctx"] else 0, r["T"]]
    try:
        from sklearn.ensemble import RandomForestRegressor
        X = np.array([feats(r) for r in train])
        y = np.log([r["seconds"] for r in train])
        rf = RandomForestRegressor(n_estimators=300, min_samples_leaf=2, random_state=0).fit(X, y)
        rfp = {id(r): float(np.exp(rf.predict(np.array([feats(r)]))[0])) for r in pts}
        res["random_forest"] = {"train": stats([rfp[id(r)] / r["seconds"] - 1 for r in train]),
                                "heldout": stats([rfp[id(r)] / r["seconds"] - 1 for r in held])}
    except ImportError:  # pragma: no cover
        res["random_forest"] = None
    Z = np.array([[r["chunk"] / 2048, r["D"] / 128, r["sum_ctx"] / 5e5] for r in train])

    def lut(r):
        z = np.array([r["chunk"] / 2048, r["D"] / 128, r["sum_ctx"] / 5e5])
        j = int(np.argmin(((Z - z) ** 2).sum(1)))
        return train[j]["seconds"] * r["T"] / train[j]["T"]
    res["lookup_table"] = {"heldout": stats([lut(r) / r["seconds"] - 1 for r in held])}
    perf = {}
    for c in (256, 512, 1024, 2048):
        rs = [r for r in pts if r["kind"] == "grid" and r["chunk"] == c]
        perf[c] = float(np.mean([r["T"] / r["seconds"] for r in rs]))
    out = {"sweep": os.path.relpath(args.sweep, ROOT), "layers": sw["layers"], "model": sw["model"],
           "timing": sw["timing"], "device": sw.get("device"),
           "iteration_model": "c0 + c1 T + lin(T) + layers x attention event model (include/niyama.h)",
           "linear_table": lin,
           "train_points": len(train), "heldout_points": len(held), "errors": res,
           "attention_share_of_iteration": {"min": float(min(share)), "median": float(np.median(share)),
                                            "max": float(max(share))},
           "fig4_tokens_per_s_by_chunk": perf,
           "fig4_chunk256_vs_2048_throughput_ratio": perf[256] / perf[2048],
           "paper_context": "P:71: 28% lower full-model throughput at small chunk (ratio ~0.72, A100, Llama3-8B)",
           "points": [{k: r[k] for k in ("kind", "seed", "chunk", "offset", "D", "sum_ctx", "T", "seconds")} |
                      {"analytic": analytic[id(r)]} for r in pts]}
    json.dump(out, open(args.out, "w"), indent=1)
    print(json.dumps({k: v for k, v in out.items() if k not in ("points", "linear_table")}, indent=1))


if __name__ == "__main__":
    main()
