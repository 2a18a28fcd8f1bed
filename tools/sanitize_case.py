"""One hybrid-batch case through the C ABI, for compute-sanitizer runs
(tools/sanitize.sh): append + attention (and the fused append variant), checked
against the oracle so a sanitizer-clean run is also a correct one."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from tests.gpu_harness import Run, assert_close, oracle_for, to_host_f64  # noqa: E402

CASES = {
    "tiny": lambda: W.config1_tiny("unaligned"),
    "ragged": lambda: W.random_hybrid(W.L8B, seed=3, num_prefill=2, max_chunk=150, num_decode=6, max_ctx=900),
    "g8": lambda: W.random_hybrid(W.Shape(16, 2, 128, 16, "bf16"), seed=8, num_prefill=1, max_chunk=100,
                                  num_decode=5, max_ctx=2500),
    "config2": lambda: W.config2_l8b(),
    "dec": lambda: W.hybrid(W.L8B, "dec", prefill_offset=0, chunk=0, decode_ctx=[300, 17, 1000, 45], seed=7),
}

if __name__ == "__main__":
    name = sys.argv[1]
    fused = "fused" in sys.argv[2:]
    tuning = dict(decode_path=2) if "path2" in sys.argv[2:] else None
    if "pairs" in sys.argv[2:]:
        tuning = dict(prefill_pairs=1)
    wl = CASES[name]()
    r = Run(wl, fused=fused, tuning=tuning)
    o, lse = r.attention()
    o2, _ = r.attention()      # second launch of the same plan (epoch counters, self-reset queues)
    torch.cuda.synchronize()
    rows = None if name != "config2" else list(range(480, 576))
    _, _, O, L = oracle_for(wl, rows=rows)
    og = to_host_f64(o2, wl.shape.dtype)
    lg = lse.cpu().numpy().astype(np.float64)
    if rows is not None:
        m = np.zeros(og.shape[1], bool)
        m[rows] = True
        og, O, lg, L = og[:, m], O[:, m], lg[:, m], L[:, m]
    tol = {} if wl.shape.dtype == "bf16" else dict(max_abs=1e-5, rel_l2=1e-5, lse_tol=1e-5)
    ma, rl = assert_close(og, O, lg, L, **tol)
    print(f"{name}{' fused' if fused else ''}: OK max_abs={ma:.2e} rel_l2={rl:.2e}")
