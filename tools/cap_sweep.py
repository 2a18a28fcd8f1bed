"""Prefill-CTA share sweep: attention launch time vs the niyama_tuning prefill_ctas cap for several
batch shapes (diagnostic for the runtime's prefill/decode CTA split policy)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from sweep_predictor import Rig  # noqa: E402

SHAPES = [  # (chunk, offset, D)
    (512, 1536, 64), (2048, 4096, 16), (1024, 1024, 64), (256, 1280, 256), (2048, 2048, 128),
    (512, 1536, 0), (2048, 0, 0), (256, 0, 16), (1024, 3072, 16),
    (256, 1536, 16), (512, 1536, 16), (256, 1536, 64), (1024, 1024, 16), (512, 3584, 128), (2048, 2048, 32),
]
CAPS = [0, 8, 16, 24, 32, 40, 48, 56, 64, 80, 96, 112, 128, 148]


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/cap_sweep.json"
    caps = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else CAPS
    res = {}
    for cap in caps:
        rig = Rig(W.L8B, num_blocks=256 * 4096 // 16 + 8192)
        rig.kv.set_tuning(prefill_ctas=cap)
        for (c, o, D) in SHAPES:
            ctx = W.l8b_decode_ctx(D).tolist() if D else []
            t, T = rig.measure(c, o, ctx, 9)
            if cap == 0:
                print("   prefill_ctas", rig.last_info.prefill_ctas, "grid tiles", rig.last_info.num_prefill_tiles)
            res.setdefault(f"c{c}_o{o}_D{D}", {})[cap] = t * 1e6
            print(f"cap={cap:3d} c={c:5d} o={o:5d} D={D:3d} t={t*1e6:8.1f}us", flush=True)
        rig.kv.close()
        del rig
        torch.cuda.empty_cache()
    json.dump(res, open(out, "w"), indent=1)
    for k, v in res.items():
        best = min(v, key=v.get)
        print(f"{k:22s} default={v.get(0, float('nan')):7.1f} best cap={best} {v[best]:7.1f}  " +
              " ".join(f"{cp}:{v[cp]:.0f}" for cp in caps if cp))


if __name__ == "__main__":
    main()
