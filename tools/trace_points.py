"""Per-CTA launch timelines (niyama_debug_trace) of chosen config-3 sweep points, for the a8
schedule-model pins and diagnosis.  Points are (kind, seed, chunk, D) of tools/sweep_predictor.py.

    python tools/trace_points.py --out gpurun_out/traces.json grid:2:256:16 grid:2:512:16 ...
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from sweep_predictor import Rig, point_desc, plan_fields  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("points", nargs="+")
    args = ap.parse_args()
    rig = Rig(W.L8B, num_blocks=256 * 8192 // 16 + 8192)
    rig.want_trace = True
    out = []
    for p in args.points:
        kind, seed, chunk, D = p.split(":")
        seed, chunk, D = int(seed), int(chunk), int(D)
        o, ctx = point_desc(max(chunk, 1), D, seed)
        if chunk == 0:
            o = 0
        t, T = rig.measure(chunk, o, ctx, args.reps)
        out.append(dict(kind=kind, seed=seed, chunk=chunk, offset=o, D=D, ctx=ctx, sum_ctx=int(sum(ctx)), seconds=t,
                        trace=rig.last_trace, **plan_fields(rig)))
        print(f"{p}: o={o} t={t * 1e6:.1f} us", flush=True)
    json.dump(out, open(args.out, "w"))


if __name__ == "__main__":
    main()
