"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no gather, no GEMM, no reduction, no
schedule logic).  It only draws random numbers and builds the structured
"provenance" patterns of SURVEY.md §8(c) ("What pins each part").  Both the CUDA path
and the CPU oracle consume exactly the tensors produced here.

Recipe (SURVEY.md §8(d) "Value distributions and seeds"):
  * A ~ N(0, 1), B ~ N(0, 1) / sqrt(K_total), drawn in fp32 with torch.Generator,
    seeds A_r = 1000 + r + salt, B_r = 2000 + r + salt, then rounded to bf16 (RNE, torch
    `.to(torch.bfloat16)`).  Outputs are then ~N(0, 1) like real activations.
  * Layouts follow Lst.1 (`b_desc.load([offs_bn, offs_k])`,
    `tl.dot(a, b.T)`): A [rows, K] row-major, B [N, K] row-major (nn.Linear layout).
"""
from __future__ import annotations

import math

import torch

BF16 = torch.bfloat16


def _randn(shape, seed: int, scale: float = 1.0) -> torch.Tensor:
    g = torch.Generator(device="cpu")
    g.manual_seed(seed)
    x = torch.randn(*shape, generator=g, dtype=torch.float32)
    if scale != 1.0:
        x = x * scale
    return x.to(BF16)


def ag_inputs(world_size: int, M: int, K: int, N_loc: int, salt: int = 0):
    """AllGather->GEMM inputs (BASELINE.json configs[1] shape family).

    Returns (A_shards, Bs): A_shards[r] is rank r's row shard [M/W, K] bf16, Bs[r] is
    rank r's column-sharded weight [N_loc, K] bf16 (B ~ N(0,1)/sqrt(K))."""
    assert M % world_size == 0
    S = M // world_size
    A = [_randn((S, K), 1000 + r + salt) for r in range(world_size)]
    B = [_randn((N_loc, K), 2000 + r + salt, 1.0 / math.sqrt(max(K, 1))) for r in range(world_size)]
    return A, B


def rs_inputs(world_size: int, M: int, K_loc: int, N: int, salt: int = 0):
    """GEMM->ReduceScatter inputs (BASELINE.json configs[2] shape family).

    Returns (As, Bs): As[s] is rank s's K-shard of the activation [M, K_loc], Bs[s] is
    rank s's row-parallel weight shard [N, K_loc]; B ~ N(0,1)/sqrt(W*K_loc)."""
    K_total = max(world_size * K_loc, 1)
    A = [_randn((M, K_loc), 1000 + s + salt) for s in range(world_size)]
    B = [_randn((N, K_loc), 2000 + s + salt, 1.0 / math.sqrt(K_total)) for s in range(world_size)]
    return A, B


def rs_weights(world_size: int, K_loc: int, N: int, salt: int = 0):
    """Only the weight shards of rs_inputs (same seeds, same values)."""
    K_total = max(world_size * K_loc, 1)
    return [_randn((N, K_loc), 2000 + s + salt, 1.0 / math.sqrt(K_total)) for s in range(world_size)]


def ag_provenance_inputs(world_size: int, M: int, K: int, N_loc: int, epoch: int = 0):
    """Exact-integer provenance pattern for AG ("Gather semantics").

    A[i, 0..2] = base-32 digits of the global row id i (each <= 31, exact in bf16),
    A[i, 3] = epoch mod 32, every other element 0.  B[n, k] = 1 iff k == n mod 4.
    Then C[i, n] = A[i, n mod 4] exactly, so decoding C gives back row id and epoch."""
    assert K >= 4 and M < 32 ** 3
    S = M // world_size
    shards = []
    for r in range(world_size):
        a = torch.zeros(S, K, dtype=torch.float32)
        rows = torch.arange(r * S, (r + 1) * S)
        a[:, 0] = (rows % 32).float()
        a[:, 1] = ((rows // 32) % 32).float()
        a[:, 2] = ((rows // 1024) % 32).float()
        a[:, 3] = float(epoch % 32)
        shards.append(a.to(BF16))
    Bs = []
    for r in range(world_size):
        b = torch.zeros(N_loc, K, dtype=torch.float32)
        n = torch.arange(N_loc)
        b[n, n % 4] = 1.0
        Bs.append(b.to(BF16))
    return shards, Bs


def rs_provenance_inputs(world_size: int, M: int, K_loc: int, N: int):
    """Bitmask provenance pattern for RS ("RS numerics").

    Rank s uses A_s[:, 0] = 1 and B_s[:, 0] = 2**s, everything else 0, so every output
    element equals sum_s 2**s = 2**W - 1 exactly; a missing or duplicated contribution
    shows up as a wrong bit."""
    As, Bs = [], []
    for s in range(world_size):
        a = torch.zeros(M, K_loc, dtype=torch.float32)
        a[:, 0] = 1.0
        b = torch.zeros(N, K_loc, dtype=torch.float32)
        b[:, 0] = float(2 ** s)
        As.append(a.to(BF16))
        Bs.append(b.to(BF16))
    return As, Bs


def moe_inputs(world_size: int, T: int, H: int, N: int, topk: int = 2, zipf: float = 0.0, salt: int = 0):
    """MoE dispatch + expert GEMM inputs (BASELINE.json configs[3]; SURVEY.md §8(d)
    "Mixtral (NEXT-3): router logits N(0,1) with seed 3000, top-2, plus a Zipf-skewed
    variant").  One expert per rank (expert e lives on rank e).

    Returns (Xs, idxs, Bs): Xs[s] [T, H] bf16 tokens of rank s (N(0,1)); idxs[s] [T, topk]
    int32 expert ids of each token: the top-k of N(0,1) router logits (seed 3000 + s +
    salt), or with zipf > 0 k distinct experts drawn with probability ~ 1 / (e + 1)**zipf;
    Bs[e] [N, H] bf16 expert weight (N(0,1)/sqrt(H); Mixtral w1||w3 when N = 2 * 14336)."""
    X = [_randn((T, H), 1000 + s + salt) for s in range(world_size)]
    B = [_randn((N, H), 2000 + e + salt, 1.0 / math.sqrt(max(H, 1))) for e in range(world_size)]
    idx = []
    for s in range(world_size):
        g = torch.Generator(device="cpu")
        g.manual_seed(3000 + s + salt)
        if zipf > 0:
            p = 1.0 / torch.arange(1, world_size + 1, dtype=torch.float64) ** zipf
            sel = torch.multinomial(p.expand(T, world_size), topk, replacement=False, generator=g)
        else:
            logits = torch.randn(T, world_size, generator=g, dtype=torch.float32)
            sel = torch.topk(logits, topk, dim=1).indices
        idx.append(sel.to(torch.int32).contiguous())
    return X, idx, B


def moe_provenance_inputs(world_size: int, T: int, H: int, N: int, idxs, epoch: int = 0):
    """Exact-integer provenance for A2A: X_s[t, 0..2] = base-32 digits of the global token
    id s*T + t, X_s[t, 3] = epoch mod 32, other elements 0; B_e[n, k] = 1 iff k == n mod 4,
    so Y_e[i, n] = A_e[i, n mod 4] exactly and every output row names the token it came
    from.  `idxs` (routing) is passed through unchanged."""
    assert H >= 4 and world_size * T < 32 ** 3
    X = []
    for s in range(world_size):
        a = torch.zeros(T, H, dtype=torch.float32)
        gid = torch.arange(s * T, (s + 1) * T)
        a[:, 0] = (gid % 32).float()
        a[:, 1] = ((gid // 32) % 32).float()
        a[:, 2] = ((gid // 1024) % 32).float()
        a[:, 3] = float(epoch % 32)
        X.append(a.to(BF16))
    B = []
    for e in range(world_size):
        b = torch.zeros(N, H, dtype=torch.float32)
        n = torch.arange(N)
        b[n, n % 4] = 1.0
        B.append(b.to(BF16))
    return X, idxs, B


def attn_inputs(world_size: int, H: int, S_loc: int, d: int, salt: int = 0):
    """Sequence-parallel attention inputs (NEXT-4; Llama-3 attention shapes: d = 128): per
    rank Q_r, K_r, V_r [H, S_loc, d] bf16, N(0,1) (seeds 4000/5000/6000 + r + salt).
    With N(0,1) q and k the scaled scores q.k/sqrt(d) are ~N(0,1), like trained models'."""
    Q = [_randn((H, S_loc, d), 4000 + r + salt) for r in range(world_size)]
    K = [_randn((H, S_loc, d), 5000 + r + salt) for r in range(world_size)]
    V = [_randn((H, S_loc, d), 6000 + r + salt) for r in range(world_size)]
    return Q, K, V


def to_f64(t: torch.Tensor):
    """bf16 -> float64 numpy (exact widening; no rounding happens here)."""
    return t.to(torch.float64).numpy()
