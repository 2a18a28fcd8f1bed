"""Oracle: paged KV cache bookkeeping.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper delegates KV management to vLLM PagedAttention (§3.6:
"maintaining compatibility with vLLM's efficient tensor parallelism and
PagedAttention mechanisms") and keeps a request's KV on the GPU across
iterations (§3.4 selective preemption).  It never writes the
allocator down; readings fix it:

  R9  fixed block size B (default 16); a sequence of n tokens owns
      ceil(n/B) blocks; new blocks are the SMALLEST free ids, ascending;
      reservation walks the descriptor in order (prefill slices, then
      decodes) and is all-or-nothing; release returns the blocks.
  R4  decode_ctx counts keys visible after appending the new token, so the
      decode's new token goes to position ctx-1 and the cache must hold
      exactly ctx-1 tokens before the batch.
  R6  batch rows: prefill slice rows first (position offset+i), then decodes.

Stored values keep their representation (bf16 as uint16 bits, fp32 as
float32) so read-back comparisons are bitwise.
"""
from __future__ import annotations

import bisect
from dataclasses import dataclass
from typing import Dict, List, Tuple

import numpy as np

OK, EINVAL, ENOBLOCKS, ENOSEQ, ESTATE = 0, 1, 2, 3, 4


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


@dataclass
class Plan:
    """One iteration's bookkeeping result.

    rows[r] = (seq, position, visible) for batch row r: the new token of row r
    is written at logical `position`; attention for row r sees keys
    [0, visible) with visible = position + 1 (causal, P:118 chunked prefill;
    decode row sees its whole context).
    slots[r] = (physical block, slot within block) that receives row r's K/V.
    """

    rows: List[Tuple[int, int, int]]
    slots: List[Tuple[int, int]]
    tables: Dict[int, List[int]]


class KVPool:
    def __init__(self, num_layers: int, num_kv_heads: int, head_dim: int, block_size: int,
                 num_blocks: int, dtype: str = "bf16"):
        if block_size < 1 or num_blocks < 1 or head_dim < 1 or num_kv_heads < 1 or num_layers < 1:
            raise OracleError(EINVAL, "bad pool shape")
        self.L, self.H, self.d, self.B, self.N = num_layers, num_kv_heads, head_dim, block_size, num_blocks
        self.dtype = dtype
        store = np.uint16 if dtype == "bf16" else np.float32
        # [layer][K=0/V=1][block][kv head][slot][d]
        self.data = np.zeros((num_layers, 2, num_blocks, num_kv_heads, block_size, head_dim), dtype=store)
        self.free: List[int] = list(range(num_blocks))  # kept sorted ascending
        self.table: Dict[int, List[int]] = {}
        self.length: Dict[int, int] = {}

    # -- R9 allocation ------------------------------------------------------
    def _need(self, seq: int, new_len: int) -> int:
        have = len(self.table.get(seq, []))
        want = -(-new_len // self.B)  # ceil
        return max(0, want - have)

    def plan(self, desc) -> Plan:
        """Validate a batch descriptor, reserve blocks, advance lengths (a2).

        Errors leave the pool untouched (validation precedes any mutation)."""
        P, D = desc.num_prefill, desc.num_decode
        if not (len(desc.prefill_offset) == len(desc.prefill_len) == P and len(desc.decode_ctx) == D):
            raise OracleError(EINVAL, "descriptor arrays disagree in length")
        if desc.tier is not None and len(desc.tier) != P + D:
            raise OracleError(EINVAL, "tier array length")
        seen = set()
        for s in list(desc.prefill_seq) + list(desc.decode_seq):
            if s in seen:
                raise OracleError(EINVAL, f"seq {s} appears twice in one batch")
            seen.add(s)
        new_len: List[Tuple[int, int]] = []
        for s, o, c in zip(desc.prefill_seq, desc.prefill_offset, desc.prefill_len):
            if o < 0 or c < 0:
                raise OracleError(EINVAL, "negative prefill offset/len")
            cur = self.length.get(s, 0)
            if cur != o:
                raise OracleError(ESTATE, f"seq {s}: cached {cur} != prefill offset {o}")
            new_len.append((s, o + c))
        for s, ctx in zip(desc.decode_seq, desc.decode_ctx):
            if ctx < 1:
                raise OracleError(EINVAL, "decode ctx < 1")
            if s not in self.length:
                raise OracleError(ENOSEQ, f"decode of unknown seq {s}")
            if self.length[s] != ctx - 1:
                raise OracleError(ESTATE, f"seq {s}: cached {self.length[s]} != ctx-1 {ctx - 1}")
            new_len.append((s, ctx))
        total = sum(self._need(s, n) for s, n in new_len)
        if total > len(self.free):
            raise OracleError(ENOBLOCKS, f"need {total} blocks, {len(self.free)} free")
        # commit: smallest free ids, descriptor order
        for s, n in new_len:
            k = self._need(s, n)
            take, self.free = self.free[:k], self.free[k:]
            self.table.setdefault(s, []).extend(take)
            self.length[s] = n
        rows, slots = [], []
        for s, o, c in zip(desc.prefill_seq, desc.prefill_offset, desc.prefill_len):
            for i in range(c):
                p = o + i
                rows.append((s, p, p + 1))
                slots.append((self.table[s][p // self.B], p % self.B))
        for s, ctx in zip(desc.decode_seq, desc.decode_ctx):
            p = ctx - 1
            rows.append((s, p, ctx))
            slots.append((self.table[s][p // self.B], p % self.B))
        return Plan(rows=rows, slots=slots, tables={s: list(self.table[s]) for s, _ in new_len})

    def release(self, seq: int) -> None:
        if seq not in self.length:
            raise OracleError(ENOSEQ, f"release of unknown seq {seq}")
        for b in self.table.pop(seq):
            bisect.insort(self.free, b)
        del self.length[seq]

    def truncate(self, seq: int, new_len: int) -> None:
        """Keep the first new_len tokens; blocks past ceil(new_len/B) are freed (R9)."""
        if seq not in self.length:
            raise OracleError(ENOSEQ, f"truncate of unknown seq {seq}")
        if new_len < 0 or new_len > self.length[seq]:
            raise OracleError(EINVAL, "truncate: new_len outside [0, len]")
        keep = -(-new_len // self.B)
        for b in self.table[seq][keep:]:
            bisect.insort(self.free, b)
        self.table[seq] = self.table[seq][:keep]
        self.length[seq] = new_len

    # -- a3 append ----------------------------------------------------------
    def append(self, layer: int, plan: Plan, k_new: np.ndarray, v_new: np.ndarray) -> None:
        """pool[table[s][p//B]][h][p%B][:] = K_new[row][h][:] (bit copy), same for V."""
        for r, (blk, slot) in enumerate(plan.slots):
            self.data[layer, 0, blk, :, slot, :] = k_new[r]
            self.data[layer, 1, blk, :, slot, :] = v_new[r]

    # -- read back ----------------------------------------------------------
    def gather(self, layer: int, seq: int, n: int) -> Tuple[np.ndarray, np.ndarray]:
        """Logical K, V of `seq` positions [0, n): [n][Hkv][d] in stored representation."""
        tbl = self.table[seq]
        t = np.arange(n)
        blk = np.asarray(tbl, dtype=np.int64)[t // self.B] if n else np.zeros(0, np.int64)
        slot = t % self.B
        k = self.data[layer, 0, blk, :, slot, :]
        v = self.data[layer, 1, blk, :, slot, :]
        return k, v
