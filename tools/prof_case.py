"""Run one workload's attention launch a few times (for ncu -k regex:hybrid_attn).

    python tools/prof_case.py {prefill|decode|mixed|l70b} [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from kbench import setup  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "mixed"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if case == "prefill":
    wl = W.hybrid(W.L8B, "prefill-only", prefill_offset=1536, chunk=512, decode_ctx=[], seed=2)
elif case == "decode":
    wl = W.hybrid(W.L8B, "decode-only", prefill_offset=0, chunk=0, decode_ctx=W.l8b_decode_ctx(), seed=2)
elif case == "l70b":
    wl = W.config4_l70b()
elif case == "l70bp":
    wl = W.hybrid(W.L70B, "l70b-prefill-c2048-o6144", prefill_offset=6144, chunk=2048, decode_ctx=[], seed=4)
else:
    wl = W.config2_l8b()
kv, plan, q, o, lse = setup(wl)
for _ in range(reps):
    kv.attention(plan, 0, q, o, lse)
torch.cuda.synchronize()
print("done", case)
