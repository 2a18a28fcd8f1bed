"""A/B of prefill split-K (niyama_tuning.prefill_split: 0 off (default), 1 on) on small prefill-heavy launches."""
import os, sys
sys.path.insert(0, '/root/repo/tools'); sys.path.insert(0, '/root/repo')
import workloads as W
from kbench import time_it
for wl in (W.hybrid(W.L8B, "prefill-only-c100-o3000", prefill_offset=3000, chunk=100, decode_ctx=[], seed=31),
           W.hybrid(W.L8B, "prefill-only-c256-o2048", prefill_offset=2048, chunk=256, decode_ctx=[], seed=31),
           W.hybrid(W.L8B, "mixed-c64-o2000-D3", prefill_offset=2000, chunk=64, decode_ctx=[700, 33, 1500], seed=32),
           W.hybrid(W.L8B, "prefill-only-c512-o1536", prefill_offset=1536, chunk=512, decode_ctx=[], seed=2)):
    for split in (0, 1):
        print(f"prefill_split={split}", end=" ")
        time_it(wl, tuning=dict(prefill_split=split))
