"""CPU oracle for the AutoOverlap hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (its `cpu_baseline` leg and
`--impl reference`) may import anything under oracle/.  The product package
(paper_2601_20595_b200/) never imports it; there is no CPU fallback.

  numeric.py   fp64 AG-GEMM / GEMM-RS / GEMM-AR definitions
  schedule.py  brute-force chunk schedule + canonical JSON (§5.1-§5.2)
  a2a.py       fp64 MoE All-to-All dispatch + expert GEMM and its chunk-ordered tile list (NEXT-3)
  attn.py      fp64 sequence-parallel attention over the all-gathered KV (NEXT-4)
"""
