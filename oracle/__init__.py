"""fp64 CPU ORACLE for the Niyama hybrid-batch paged-attention path.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import anything in
this package.  The product path (`paper_2503_22562_b200`, `include/niyama.h`)
never imports, links or calls it, and this package never imports the product:
the two share no code.  Inputs come from `workloads.py` (seeded generators,
no method arithmetic).

Contents (each function cites the passage it follows; PAPER.md = P:n,
SPEC.md = S:n, readings R1..R19):

- kvcache.py   a2/a3  block-table KV pool: reserve, plan, append, gather
- attention.py a4-a6  causal GQA softmax attention over each row's logical
                      KV sequence (the plain definition), LSE, split merge
- predictor.py a8     iteration-time predictor: features, NNLS fit, eval,
                      max feasible chunk (brute force over C)
- sched.py     a1     deadlines Eq. 1-3, slack, min slack over decodes
- shard.py     a7     KV-head sharding and head all-gather (concatenation)

Parity status: every function here is pinned by a `-m "not gpu"` test against
something other than itself (brute force, a library special case, closed
forms, invariants, SPEC worked examples).  See DESIGN.md §"Oracle pins".
"""
