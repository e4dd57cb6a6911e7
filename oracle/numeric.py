"""CPU fp64 numerical oracle for the AutoOverlap hot path (AG-GEMM and GEMM-RS).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
`cpu_baseline` / `--impl reference` legs may import this module.  It shares no code with
the CUDA path (paper_2601_20595_b200/), and the CUDA path never imports it.

Every function states the passage it follows.  `P:n` = /root/reference/PAPER.md line n,
`S:n` = /root/reference/SPEC.md line n.  The method reaches exactly (up to rounding
order) the plain collective-then-GEMM result, so the oracle is that definition written
out in float64 ("Numerical result"):

  AG-GEMM  ("AllGather--GEMM"; "gather = concatenation of shards"):
      C_r = concat_p(A_p) . B_r^T
  GEMM-AR  ("GEMM--AllReduce", NEXT-1):  C = sum_s A_s . B_s^T on every rank
  GEMM-RS  ("GEMM--ReduceScatter"; S:165/S:168 owner rows are contiguous blocks;
            S:604 "ascending source rank" accumulation order):
      C_shard_r = ( sum_{s=0..W-1} A_s . B_s^T )[r*S:(r+1)*S, :]

Operand layouts follow Lst.1: A [rows, K], B [N, K], result = A . B^T.
Inputs are the bf16 tensors from synthetic/inputs.py widened exactly to float64.

Pins (tests/test_oracle_numeric.py, `-m "not gpu"`): exact rational arithmetic on
sampled elements, the K-unsharded closed form for RS, exact-integer provenance
patterns, and W=1 reduction to a plain matmul.
"""
from __future__ import annotations

import numpy as np


def all_gather(shards):
    """AllGather of row shards: concatenation in rank order (Lst.2 P:249-265:
    rank r's local region is shard(r); after the plan every rank holds every shard(p)
    at its own position)."""
    return np.concatenate([np.asarray(s, dtype=np.float64) for s in shards], axis=0)


def gemm(A, B):
    """Local kernel of Lst.1: accumulator = tl.dot(a, b.T) over all K."""
    A = np.asarray(A, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    return A @ B.T


def ag_gemm(A_shards, B_r):
    """AllGather->GEMM at one rank: C_r = concat_p(A_p) . B_r^T."""
    return gemm(all_gather(A_shards), B_r)


def ag_gemm_all_ranks(A_shards, Bs):
    """Simulates every rank r of AG-GEMM (north star: "simulates the ranks, forms the
    gathered ... tensors and computes the GEMM in fp64")."""
    A_full = all_gather(A_shards)
    return [gemm(A_full, B) for B in Bs]


def reduce_scatter(partials, rank: int):
    """ReduceScatter of full-size partials: owner `rank` receives the elementwise sum,
    accumulated in ascending source rank, of its contiguous row block (S:168:
    "rank 0 reduces [0:128), rank 1 reduces [128:256)")."""
    W = len(partials)
    M = partials[0].shape[0]
    assert M % W == 0
    S = M // W
    acc = np.zeros_like(np.asarray(partials[0], dtype=np.float64)[rank * S:(rank + 1) * S])
    for s in range(W):
        acc = acc + np.asarray(partials[s], dtype=np.float64)[rank * S:(rank + 1) * S]
    return acc


def gemm_rs(As, Bs, rank: int):
    """GEMM->ReduceScatter at owner `rank`: every rank s forms its partial A_s . B_s^T
    (K-sharded, row-parallel), then the partials are reduce-scattered."""
    partials = [gemm(A, B) for A, B in zip(As, Bs)]
    return reduce_scatter(partials, rank)


def gemm_rs_all_ranks(As, Bs):
    partials = [gemm(A, B) for A, B in zip(As, Bs)]
    return [reduce_scatter(partials, r) for r in range(len(As))]


def gemm_ar(As, Bs):
    """GEMM->AllReduce ("GEMM--AllReduce"; Fig.4d P:311 partition-based AllReduce):
    every rank receives the full sum of the partials, C = sum_s A_s . B_s^T (ascending s)."""
    acc = None
    for A, B in zip(As, Bs):
        p = gemm(A, B)
        acc = p if acc is None else acc + p
    return acc


def gemm_rows(A, B, rows):
    """Selected output rows of A . B^T (used for sampled checks at full size, where the
    oracle computes the outputs one row block at a time)."""
    A = np.asarray(A, dtype=np.float64)
    return A[rows] @ np.asarray(B, dtype=np.float64).T


def ag_gemm_rows(A_shards, B_r, rows):
    """Rows `rows` (global row ids) of the AG-GEMM result, computed from the gathered A."""
    return gemm_rows(all_gather(A_shards), B_r, rows)


def gemm_rs_rows(As, Bs, rank: int, local_rows):
    """Rows `local_rows` (indices inside owner `rank`'s block) of the GEMM-RS result."""
    W = len(As)
    M = np.asarray(As[0]).shape[0]
    S = M // W
    g = rank * S + np.asarray(local_rows)
    acc = None
    for s in range(W):
        p = gemm_rows(As[s], Bs[s], g)
        acc = p if acc is None else acc + p
    return acc


def gemm_rs_from_rows(A_rows, Bs):
    """GEMM-RS output rows given, for every source s, the same rows of A_s (already
    selected): sum_s A_rows[s] . B_s^T in ascending s."""
    acc = None
    for a, b in zip(A_rows, Bs):
        p = gemm(a, b)
        acc = p if acc is None else acc + p
    return acc


def check_tolerance(gpu, ref, elem_rel=1e-2, frob_rel=2e-3):
    """BASELINE.json north star acceptance: per element |gpu - oracle| <= 1e-2 *
    max(1, |oracle|) and relative Frobenius error <= 2e-3.  Returns (ok, max_elem, frob)."""
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if ref.size == 0:
        return True, 0.0, 0.0
    err = np.abs(gpu - ref)
    elem = float(np.max(err / np.maximum(1.0, np.abs(ref))))
    denom = float(np.linalg.norm(ref))
    frob = float(np.linalg.norm(gpu - ref) / denom) if denom > 0 else float(np.linalg.norm(gpu - ref))
    return (elem <= elem_rel and frob <= frob_rel), elem, frob
