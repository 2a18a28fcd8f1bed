"""Build tests/golden/launch_traces_l8b.json: MEASURED per-CTA prefill tile counts of traced
config-3 launches (niyama_debug_trace, tools/sweep_predictor.py --trace-every), with each
launch's batch and plan configuration.  Pins the a8 model's tile schedule (oracle
predictor.tiles_per_cta) against the kernel's real dynamic queue.

    python tools/make_trace_fixture.py profiles/r02/predictor_sweep_l8b.json
"""
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    src = sys.argv[1]
    pts = [r for r in json.load(open(src))["points"] if "trace" in r and r["chunk"] > 0]
    out = []
    for r in pts:
        tiles = r["trace"]["tiles"]
        hist = collections.Counter(int(x) for x in tiles if x > 0)
        out.append({"chunk": r["chunk"], "offset": r["offset"], "ctx": r["ctx"], "split_len": r["split_len"],
                    "prefill_ctas": r["prefill_ctas"], "tiles": r["tiles"], "ctas_traced": len(tiles),
                    "measured_tiles_per_cta_hist": {str(k): v for k, v in sorted(hist.items())}})
    dst = os.path.join(ROOT, "tests", "golden", "launch_traces_l8b.json")
    json.dump({"source": os.path.relpath(src, ROOT), "shape": "L8B (Hq 32, Hkv 8, d 128, bf16, B 16)",
               "what": "per launch: how many prefill CTAs ran k tiles (measured, globaltimer trace)",
               "launches": out}, open(dst, "w"), indent=0)
    print(f"{len(out)} launches -> {dst}")


if __name__ == "__main__":
    main()
