"""Small hybrid batches (few decodes): launch time vs split length (niyama_tuning split_len)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from kbench import time_it  # noqa: E402

if __name__ == "__main__":
    for D, c, o in [(16, 256, 1536), (16, 1024, 1024), (32, 512, 1024), (8, 0, 0), (16, 0, 0), (32, 0, 0)]:
        ctx = W.l8b_decode_ctx(D, seed=D).tolist()
        for sl in (0, 128, 256):
            time_it(W.hybrid(W.L8B, f"D{D}-c{c}-o{o}-split{sl}", prefill_offset=o, chunk=c, decode_ctx=ctx, seed=2),
                    tuning={"split_len": sl})
