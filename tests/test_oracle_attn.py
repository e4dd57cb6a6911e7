"""Pins of the SP-attention oracle (oracle/attn.py) against facts that do not come from it."""
from fractions import Fraction

import numpy as np
import pytest

from oracle import attn as oa
from synthetic import inputs as si


def _np(ts):
    return [si.to_f64(t) for t in ts]


def test_constant_scores_give_mean_of_v():
    rng = np.random.default_rng(0)
    H, Sq, Sk, d = 2, 3, 7, 4
    Q = np.zeros((H, Sq, d))
    K = rng.standard_normal((H, Sk, d))
    V = rng.standard_normal((H, Sk, d))
    np.testing.assert_allclose(oa.attention(Q, K, V, 0.5), np.broadcast_to(V.mean(axis=1, keepdims=True), (H, Sq, d)),
                               rtol=0, atol=1e-14)


def test_one_hot_score_selects_a_row():
    H, Sk, d = 1, 5, 4
    K = np.zeros((H, Sk, d))
    K[0, 3, 0] = 1.0
    Q = np.zeros((H, 1, d))
    Q[0, 0, 0] = 1e4  # score 1e4 * scale on row 3, 0 elsewhere
    V = np.arange(Sk * d, dtype=np.float64).reshape(H, Sk, d)
    np.testing.assert_allclose(oa.attention(Q, K, V, 1.0), V[:, 3:4], rtol=0, atol=1e-12)


def test_kv_order_invariance_and_ring_gather():
    W, H, S, d = 4, 2, 8, 16
    Q, K, V = (_np(x) for x in si.attn_inputs(W, H, S, d, salt=3))
    ref = oa.sp_attention(Q, K, V, 1, d ** -0.5)
    perm = [2, 0, 3, 1]  # any KV order (e.g. the ring arrival order) gives the same softmax
    alt = oa.sp_attention(Q, [K[p] for p in perm], [V[p] for p in perm], 1, d ** -0.5)
    np.testing.assert_allclose(alt, ref, rtol=1e-12, atol=1e-12)


def test_single_rank_matches_element_loop():
    H, S, d = 2, 6, 8
    Q, K, V = (_np(x) for x in si.attn_inputs(1, H, S, d, salt=5))
    scale = d ** -0.5
    got = oa.sp_attention(Q, K, V, 0, scale)
    for h in range(H):
        for i in range(S):
            s = [sum(Q[0][h, i, x] * K[0][h, j, x] for x in range(d)) * scale for j in range(S)]
            m = max(s)
            e = [np.exp(v - m) for v in s]
            z = sum(e)
            for x in range(d):
                assert abs(got[h, i, x] - sum(e[j] * V[0][h, j, x] for j in range(S)) / z) < 1e-12


def test_exact_rational_tiny():
    """scale = ln 2 and integer q.k make every weight a power of two: exact rationals."""
    import math
    H, d = 1, 2
    Q = np.array([[[1.0, 0.0], [0.0, 1.0]]])
    K = np.array([[[0.0, 0.0], [1.0, 0.0], [2.0, 1.0]]])
    V = np.array([[[1.0, 0.0], [0.0, 4.0], [3.0, 3.0]]])
    got = oa.attention(Q, K, V, math.log(2.0))
    for i in range(2):
        w = [Fraction(2) ** int(np.dot(Q[0, i], K[0, j])) for j in range(3)]
        z = sum(w)
        for x in range(d):
            want = sum(w[j] * Fraction(V[0, j, x]) for j in range(3)) / z
            assert abs(got[0, i, x] - float(want)) < 1e-14


def test_sampled_rows_match():
    W, H, S, d = 2, 3, 16, 8
    Q, K, V = (_np(x) for x in si.attn_inputs(W, H, S, d, salt=7))
    full = oa.sp_attention(Q, K, V, 1, d ** -0.5)
    rows = np.array([0, 5, 15])
    np.testing.assert_allclose(oa.sp_attention_rows(Q, K, V, 1, d ** -0.5, [0, 2], rows), full[[0, 2]][:, rows],
                               rtol=1e-13, atol=1e-13)


def test_causal_single_rank_element_loop_and_first_row():
    """Causal: row i averages V over keys 0..i with softmax weights (element loop); the first
    query of the sequence returns V[0] exactly."""
    W, H, S, d = 2, 1, 4, 8
    Q, K, V = (_np(x) for x in si.attn_inputs(W, H, S, d, salt=11))
    scale = d ** -0.5
    Kf = np.concatenate(K, 1)
    Vf = np.concatenate(V, 1)
    for r in range(W):
        got = oa.sp_attention(Q, K, V, r, scale, causal=True)
        for i in range(S):
            n = r * S + i + 1  # visible keys
            s = [sum(Q[r][0, i, x] * Kf[0, j, x] for x in range(d)) * scale for j in range(n)]
            m = max(s)
            e = [np.exp(v - m) for v in s]
            for x in range(d):
                assert abs(got[0, i, x] - sum(e[j] * Vf[0, j, x] for j in range(n)) / sum(e)) < 1e-12
    np.testing.assert_array_equal(oa.sp_attention(Q, K, V, 0, scale, causal=True)[0, 0], V[0][0, 0])


def test_causal_last_rank_last_row_equals_full():
    """The last token of the sequence sees every key: causal == non-causal on that row."""
    W, H, S, d = 3, 2, 8, 16
    Q, K, V = (_np(x) for x in si.attn_inputs(W, H, S, d, salt=13))
    c = oa.sp_attention(Q, K, V, W - 1, d ** -0.5, causal=True)
    f = oa.sp_attention(Q, K, V, W - 1, d ** -0.5)
    np.testing.assert_allclose(c[:, -1], f[:, -1], rtol=1e-13, atol=1e-13)
    rows = np.array([0, 3, 7])
    np.testing.assert_allclose(oa.sp_attention_rows(Q, K, V, 1, d ** -0.5, [1], rows, causal=True),
                               oa.sp_attention(Q, K, V, 1, d ** -0.5, causal=True)[[1]][:, rows], rtol=1e-13, atol=1e-13)


# ---- bf16-P arithmetic floor (Q27) --------------------------------------------
def test_round_bf16_matches_torch():
    import torch
    x = np.random.default_rng(1).standard_normal(200000).astype(np.float32) * 37.0
    x[:4] = [0.0, 1.0, 2.0 ** -130, 65504.0]
    assert np.array_equal(oa.round_bf16(x), torch.from_numpy(x).bfloat16().double().numpy())


def test_p_bf16_variant_reduces_to_exact_when_p_is_representable():
    # Q = 0: every score 0, p = 1 exactly (bf16-representable): both variants give mean(V)
    rng = np.random.default_rng(2)
    Q = np.zeros((2, 8, 128))
    K = rng.standard_normal((2, 64, 128))
    V = rng.standard_normal((2, 64, 128))
    a = oa.attention(Q, K, V, 128 ** -0.5)
    b = oa.attention_p_bf16(Q, K, V, 128 ** -0.5)
    assert np.allclose(a, b, rtol=0, atol=1e-13)
    assert np.allclose(a, V.mean(axis=1, keepdims=True).repeat(8, axis=1), atol=1e-13)


def test_bf16_p_floor_exceeds_the_gemm_bound():
    """With P rounded to bf16 (the P.V MMA's input) and the output rounded to bf16, the
    relative Frobenius error against the exact fp64 result is ~2.2e-3 on the bench's
    N(0,1) scores -- above the north star's 2e-3 for GEMM outputs.  This is why the attention
    tests bound the kernel by the measured floor of this arithmetic, not by 2e-3."""
    from synthetic import inputs as si
    Q, K, V = si.attn_inputs(8, 1, 256, 128, salt=81)
    Qn, Kn, Vn = ([si.to_f64(t) for t in x] for x in (Q, K, V))
    a = oa.sp_attention(Qn, Kn, Vn, 0, 128 ** -0.5)
    b = oa.round_bf16(oa.sp_attention_p_bf16(Qn, Kn, Vn, 0, 128 ** -0.5))
    frob = np.linalg.norm(b - a) / np.linalg.norm(a)
    assert 2.0e-3 < frob < 3.0e-3, frob
    # the P rounding alone: ~2^-9 relative per probability, averaged over the keys
    p_only = oa.sp_attention_p_bf16(Qn, Kn, Vn, 0, 128 ** -0.5)
    assert 1.0e-3 < np.linalg.norm(p_only - a) / np.linalg.norm(a) < 2.0e-3
