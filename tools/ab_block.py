"""Block size A/B on prefill-heavy launches (§8(f) rank 3): a prefill step's K / V^T bulk
copies are one per paged block, so larger blocks mean fewer copy issues per 128-key step
(B = 16: 8 + 8 copies of 4 KB; B = 64: 2 + 2 of 16 KB).  Median of back-to-back launches
(tools/kbench.time_it) for L70B / L8B shapes at B = 16, 32, 64, 128.

    python tools/ab_block.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from kbench import time_it  # noqa: E402


def main():
    for B in (16, 32, 64, 128):
        l70 = W.Shape(64, 8, 128, B, "bf16")
        l8 = W.Shape(32, 8, 128, B, "bf16")
        for wl in (W.hybrid(l70, f"l70b-prefill-c2048-o6144-B{B}", prefill_offset=6144, chunk=2048, decode_ctx=[],
                            seed=4),
                   W.hybrid(l70, f"l70b-config4-B{B}", prefill_offset=6144, chunk=2048, decode_ctx=[8192] * 128,
                            seed=4),
                   W.hybrid(l8, f"l8b-prefill-c2048-o2048-B{B}", prefill_offset=2048, chunk=2048, decode_ctx=[],
                            seed=4),
                   W.hybrid(l8, f"l8b-config2-B{B}", prefill_offset=1536, chunk=512, decode_ctx=W.l8b_decode_ctx(),
                            seed=2)):
            time_it(wl, reps=30)


if __name__ == "__main__":
    main()
