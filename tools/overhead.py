"""Fixed cost of the fused launch: near-empty batches, cooperative (split rows) or not."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from kbench import time_it  # noqa: E402

if __name__ == "__main__":
    time_it(W.hybrid(W.L8B, "1 decode ctx 16 (no split)", prefill_offset=0, chunk=0, decode_ctx=[16], seed=2), trace=True)
    time_it(W.hybrid(W.L8B, "1 decode ctx 200 (split 64 -> coop)", prefill_offset=0, chunk=0, decode_ctx=[200],
                     seed=2), trace=True)
    time_it(W.hybrid(W.L8B, "64 decodes ctx 64 (no split)", prefill_offset=0, chunk=0, decode_ctx=[64] * 64,
                     seed=2), trace=True)
    time_it(W.hybrid(W.L8B, "1 prefill tile c32 o0", prefill_offset=0, chunk=32, decode_ctx=[], seed=2), trace=True)
    time_it(W.hybrid(W.L8B, "148 decodes ctx 2048", prefill_offset=0, chunk=0, decode_ctx=[2048] * 148, seed=2),
            trace=True)
