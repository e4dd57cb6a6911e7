"""CPU fp64 oracle for sequence-parallel attention with all-gathered (ring-ordered) KV
("sequence-parallel (SP) schedules, including the
overlapped RingAttention", Fig.4(c) ring AllGather P:310).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
`cpu_baseline` / `--impl reference` legs may import this module.  It shares no code with
the CUDA path (paper_2601_20595_b200/), and the CUDA path never imports it.

Reading (Q27): W ranks split the sequence; rank r holds Q_r, K_r, V_r of its
S_loc tokens for all H heads, laid out [H, S_loc, d].  Non-causal scaled dot-product
attention (Vaswani et al., the paper's attention workloads P:459) over the full sequence:

    O_r[h] = softmax( Q_r[h] . K[h]^T * scale ) . V[h],   K[h] = concat_s K_s[h] (rank order)

with scale = 1/sqrt(d).  The ring order in which the GPU consumes the KV shards does not
change the exact result (softmax over a set); the oracle uses the plain definition.

Causal (ring attention for decoders): query i of rank r is token r*S_loc + i and sees keys
at positions <= its own.

Pins (tests/test_oracle_attn.py): constant scores give the mean of V, a one-hot score
selects one V row, permutation invariance over KV rows, W = 1 reduces to single-device
attention computed with an explicit per-element loop, exact rational arithmetic on a
tiny case.
"""
from __future__ import annotations

import numpy as np


def attention(Q, K, V, scale: float, q_pos=None, k_pos=None):
    """Single-device attention, fp64: softmax(Q K^T * scale) V per head.  Q [H, Sq, d],
    K/V [H, Sk, d].  With q_pos / k_pos (global token positions) the causal mask: query i
    sees key j iff k_pos[j] <= q_pos[i] (Vaswani et al.'s decoder masking)."""
    Q = np.asarray(Q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    S = np.einsum("hqd,hkd->hqk", Q, K) * scale
    if q_pos is not None:
        S = np.where(np.asarray(k_pos)[None, None, :] <= np.asarray(q_pos)[None, :, None], S, -np.inf)
    S = S - S.max(axis=-1, keepdims=True)
    P = np.exp(S)
    P /= P.sum(axis=-1, keepdims=True)
    return np.einsum("hqk,hkd->hqd", P, V)


def sp_attention(Q_list, K_list, V_list, rank: int, scale: float, causal: bool = False):
    """Rank `rank`'s output of sequence-parallel attention: its queries against the
    all-gathered keys/values (concatenation of the shards in rank order).  causal:
    rank r's query i is global token r*S_loc + i and sees keys up to that position."""
    K = np.concatenate([np.asarray(k, dtype=np.float64) for k in K_list], axis=1)
    V = np.concatenate([np.asarray(v, dtype=np.float64) for v in V_list], axis=1)
    if not causal:
        return attention(Q_list[rank], K, V, scale)
    S_loc = np.asarray(Q_list[rank]).shape[1]
    return attention(Q_list[rank], K, V, scale, np.arange(S_loc) + rank * S_loc, np.arange(K.shape[1]))


def sp_attention_rows(Q_list, K_list, V_list, rank: int, scale: float, heads, rows, causal: bool = False,
                      p_bf16: bool = False):
    """Selected (head, row) outputs (full-size sampled checks); p_bf16: attention_p_bf16."""
    K = np.concatenate([np.asarray(k, dtype=np.float64) for k in K_list], axis=1)
    V = np.concatenate([np.asarray(v, dtype=np.float64) for v in V_list], axis=1)
    Q = np.asarray(Q_list[rank], dtype=np.float64)
    S_loc = Q.shape[1]
    qp = (np.asarray(rows) + rank * S_loc) if causal else None
    kp = np.arange(K.shape[1]) if causal else None
    out = []
    for h in heads:
        f = attention_p_bf16 if p_bf16 else attention
        out.append(f(Q[h:h + 1, rows], K[h:h + 1], V[h:h + 1], scale, qp, kp)[0])
    return np.stack(out)


def round_bf16(x):
    """Round-to-nearest-even to bfloat16 (8-bit significand), returned as float64: the
    float32 value's low 16 bits rounded away (inputs here are finite and in float32 range)."""
    f = np.asarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def attention_p_bf16(Q, K, V, scale: float, q_pos=None, k_pos=None):
    """The attention above in the arithmetic of a bf16-in / fp32-accumulate P.V contraction
    (Q27): the unnormalised probabilities p = exp(s - max s) enter the product with
    V rounded to bf16, the normaliser l = sum p is not rounded.  Everything else fp64.  This
    is the floor any kernel that feeds P to a bf16 tensor-core MMA shares; not the
    definition (that is `attention`)."""
    Q = np.asarray(Q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    S = np.einsum("hqd,hkd->hqk", Q, K) * scale
    if q_pos is not None:
        S = np.where(np.asarray(k_pos)[None, None, :] <= np.asarray(q_pos)[None, :, None], S, -np.inf)
    S = S - S.max(axis=-1, keepdims=True)
    P = np.exp(S)
    l = P.sum(axis=-1, keepdims=True)
    return np.einsum("hqk,hkd->hqd", round_bf16(P), V) / l


def sp_attention_p_bf16(Q_list, K_list, V_list, rank: int, scale: float, causal: bool = False):
    """sp_attention with attention_p_bf16."""
    K = np.concatenate([np.asarray(k, dtype=np.float64) for k in K_list], axis=1)
    V = np.concatenate([np.asarray(v, dtype=np.float64) for v in V_list], axis=1)
    if not causal:
        return attention_p_bf16(Q_list[rank], K, V, scale)
    S_loc = np.asarray(Q_list[rank]).shape[1]
    return attention_p_bf16(Q_list[rank], K, V, scale, np.arange(S_loc) + rank * S_loc, np.arange(K.shape[1]))
