import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import workloads as W
from tests.gpu_harness import Run, oracle_for, to_host_f64
wl = W.random_hybrid(W.L8B, seed=5, num_prefill=1, max_chunk=256, num_decode=8, max_ctx=2000, q_scale=8.0)
for rep in range(3):
    r = Run(wl)
    o, lse = r.attention()
    oo = to_host_f64(o, "bf16")
    bad = ~np.isfinite(oo)
    print("rep", rep, "nonfinite", bad.sum(), "rows", sorted(set(np.nonzero(bad)[1].tolist()))[:20], "heads", sorted(set(np.nonzero(bad)[0].tolist())))
    d = wl.final.desc
    print("T", d.num_rows, "prefill", d.prefill_offset, d.prefill_len, "dec", d.decode_ctx)
