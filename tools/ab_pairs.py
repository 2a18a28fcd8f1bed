"""A/B of niyama_tuning.prefill_pairs (2 = one q tile per CTA, 1 = CTA pairs with multicast
K/V) on the prefill-heavy set (median of back-to-back launches, tools/kbench.time_it)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from kbench import time_it  # noqa: E402

cases = [W.hybrid(W.L70B, "l70b-prefill-c2048-o6144", prefill_offset=6144, chunk=2048, decode_ctx=[], seed=4),
         W.config4_l70b(),
         W.hybrid(W.L8B, "l8b-prefill-c2048-o2048", prefill_offset=2048, chunk=2048, decode_ctx=[], seed=4),
         W.hybrid(W.L8B, "l8b-prefill-c512-o1536", prefill_offset=1536, chunk=512, decode_ctx=[], seed=2),
         W.config2_l8b()]
for wl in cases:
    for v in (2, 1, 2, 1):
        print(f"pairs={v}", end=" ")
        time_it(wl, reps=30, tuning=dict(prefill_pairs=v))
