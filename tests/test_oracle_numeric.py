"""Pins of the fp64 numerical oracle (oracle/numeric.py) to things other than itself.

Each pin is chosen so that a plausible oracle mistake (a dropped rank, a transposed
operand, a wrong row slice, a wrong gather order) fails at least one test:
  * exact rational arithmetic (fractions.Fraction) on sampled elements, compared within
    the fp64 summation error bound gamma_K * sum|a_k b_k|      -> transposes / indices
  * RS closed form: sum_s A_s B_s^T == A_catK . B_catK^T (K-unsharded), owner rows
                                                               -> row slice / dropped rank
  * exact-integer provenance (row ids + epoch decode exactly)  -> gather order
  * bitmask provenance (every output == 2^W - 1)                -> dropped / doubled rank
  * W = 1 special case == a plain library matmul
"""
from fractions import Fraction

import numpy as np
import pytest

from oracle import numeric as on
from synthetic import inputs as si

U64 = 2.0 ** -53


def _exact_dot(a_row, b_row):
    s = Fraction(0)
    for x, y in zip(a_row.tolist(), b_row.tolist()):
        if x != 0.0 and y != 0.0:
            s += Fraction(x) * Fraction(y)
    return s


def _sample_rows(M, chunk, rng, extra=24):
    """Every chunk-boundary row (first and last row of each chunk) + random rows."""
    rows = set()
    for g0 in range(0, M, chunk):
        rows.add(g0)
        rows.add(g0 + chunk - 1)
    rows.update(rng.integers(0, M, size=extra).tolist())
    return sorted(rows)


def test_ag_gemm_exact_rational_tiny():
    # BASELINE.json configs[0]: W=2, M=256/rank, K=512, N=512, chunk=64
    W, M, K, N, C = 2, 512, 512, 512, 64
    A, B = si.ag_inputs(W, M, K, N)
    A64 = [si.to_f64(a) for a in A]
    B64 = [si.to_f64(b) for b in B]
    rng = np.random.default_rng(7)
    Afull_rows = np.concatenate(A64, axis=0)  # only used to fetch exact row values
    for r in range(W):
        Cr = on.ag_gemm(A64, B64[r])
        assert Cr.shape == (M, N)
        rows = _sample_rows(M, C, rng, extra=8)
        cols = rng.integers(0, N, size=len(rows))
        for i, n in zip(rows, cols):
            # exact value of row i of the gathered A (shard i // S, local row i % S)
            S = M // W
            a = A64[i // S][i % S]
            assert np.array_equal(a, Afull_rows[i])
            exact = _exact_dot(a, B64[r][n])
            bound = K * U64 * float(np.sum(np.abs(a * B64[r][n]))) + 1e-300
            assert abs(Cr[i, n] - float(exact)) <= bound, (r, i, n)


def test_gemm_rs_exact_rational_tiny():
    W, M, K_loc, N, C = 2, 512, 256, 512, 64
    A, B = si.rs_inputs(W, M, K_loc, N)
    A64 = [si.to_f64(a) for a in A]
    B64 = [si.to_f64(b) for b in B]
    rng = np.random.default_rng(11)
    S = M // W
    for r in range(W):
        Cs = on.gemm_rs(A64, B64, r)
        assert Cs.shape == (S, N)
        rows = _sample_rows(S, C, rng, extra=8)
        cols = rng.integers(0, N, size=len(rows))
        for i, n in zip(rows, cols):
            g = r * S + i
            exact = sum((_exact_dot(A64[s][g], B64[s][n]) for s in range(W)), Fraction(0))
            mag = sum(float(np.sum(np.abs(A64[s][g] * B64[s][n]))) for s in range(W))
            bound = (W * K_loc + W) * U64 * mag + 1e-300
            assert abs(Cs[i, n] - float(exact)) <= bound, (r, i, n)


@pytest.mark.parametrize("W", [1, 2, 4, 8])
def test_gemm_rs_equals_k_unsharded_closed_form(W):
    M, K_loc, N = 64 * W, 48, 40
    A, B = si.rs_inputs(W, M, K_loc, N, salt=W)
    A64 = [si.to_f64(a) for a in A]
    B64 = [si.to_f64(b) for b in B]
    A_cat = np.concatenate(A64, axis=1)  # [M, W*K_loc]
    B_cat = np.concatenate(B64, axis=1)  # [N, W*K_loc]
    full = np.einsum("mk,nk->mn", A_cat, B_cat)
    S = M // W
    outs = on.gemm_rs_all_ranks(A64, B64)
    for r in range(W):
        np.testing.assert_allclose(outs[r], full[r * S:(r + 1) * S], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("W", [1, 2, 4, 8])
def test_ag_provenance_decodes_row_and_epoch(W):
    M, K, N = 128 * W, 64, 24
    for epoch in (0, 5, 31):
        A, B = si.ag_provenance_inputs(W, M, K, N, epoch=epoch)
        outs = on.ag_gemm_all_ranks([si.to_f64(a) for a in A], [si.to_f64(b) for b in B])
        for r in range(W):
            Cr = outs[r]
            # decode: C[i, n] = A[i, n mod 4]
            rid = Cr[:, 0] + 32 * Cr[:, 1] + 1024 * Cr[:, 2]
            assert np.array_equal(rid, np.arange(M, dtype=np.float64))
            assert np.all(Cr[:, 3] == epoch % 32)
            assert np.array_equal(Cr[:, 4:8], Cr[:, 0:4])


@pytest.mark.parametrize("W", [1, 2, 4, 8])
def test_rs_bitmask_provenance(W):
    M, K_loc, N = 32 * W, 16, 24
    A, B = si.rs_provenance_inputs(W, M, K_loc, N)
    outs = on.gemm_rs_all_ranks([si.to_f64(a) for a in A], [si.to_f64(b) for b in B])
    for r in range(W):
        assert outs[r].shape == (M // W, N)
        assert np.all(outs[r] == 2 ** W - 1)


def test_world_size_one_is_plain_matmul():
    M, K, N = 96, 80, 56
    A, B = si.ag_inputs(1, M, K, N, salt=3)
    a, b = si.to_f64(A[0]), si.to_f64(B[0])
    ref = np.einsum("mk,nk->mn", a, b)
    np.testing.assert_allclose(on.ag_gemm([a], b), ref, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(on.gemm_rs([a], [b], 0), ref, rtol=1e-13, atol=1e-13)


def test_sampled_rows_match_full():
    W, M, K, N = 4, 256, 64, 48
    A, B = si.ag_inputs(W, M, K, N, salt=9)
    A64 = [si.to_f64(a) for a in A]
    B64 = [si.to_f64(b) for b in B]
    rows = [0, 63, 64, 200, 255]
    np.testing.assert_array_equal(on.ag_gemm_rows(A64, B64[2], rows), on.ag_gemm(A64, B64[2])[rows])
    As, Bs = si.rs_inputs(W, M, K, N, salt=9)
    As64 = [si.to_f64(a) for a in As]
    Bs64 = [si.to_f64(b) for b in Bs]
    local = [0, 5, 63]
    full = on.gemm_rs(As64, Bs64, 3)
    np.testing.assert_allclose(on.gemm_rs_rows(As64, Bs64, 3, local), full[local], rtol=1e-13, atol=1e-13)
    g = [3 * (M // W) + i for i in local]
    np.testing.assert_allclose(on.gemm_rs_from_rows([a[g] for a in As64], Bs64), full[local], rtol=1e-13, atol=1e-13)


def test_tolerance_checker_rejects_perturbation():
    ref = np.linspace(-3, 3, 1000).reshape(10, 100)
    ok, e, f = on.check_tolerance(ref.copy(), ref)
    assert ok and e == 0 and f == 0
    bad = ref.copy()
    bad[3, 3] += 0.05  # one element off by 5e-2 > 1e-2 * max(1, |x|)
    ok, e, _ = on.check_tolerance(bad, ref)
    assert not ok and e > 1e-2
    drift = ref * (1 + 3e-3)  # Frobenius 3e-3 > 2e-3
    ok, _, f = on.check_tolerance(drift, ref)
    assert not ok and f > 2e-3


@pytest.mark.parametrize("W", [1, 2, 3, 8])
def test_gemm_ar_equals_k_unsharded_closed_form(W):
    """GEMM-AR (NEXT-1): every rank's result is the full K-unsharded GEMM (all rows)."""
    M, K_loc, N = 16 * W, 40, 24
    A, B = si.rs_inputs(W, M, K_loc, N, salt=50 + W)
    A64 = [si.to_f64(a) for a in A]
    B64 = [si.to_f64(b) for b in B]
    full = np.concatenate(A64, axis=1) @ np.concatenate(B64, axis=1).T
    np.testing.assert_allclose(on.gemm_ar(A64, B64), full, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("W", [1, 2, 4, 8])
def test_gemm_ar_bitmask_provenance(W):
    M, K_loc, N = 32 * W, 16, 24
    A, B = si.rs_provenance_inputs(W, M, K_loc, N)
    out = on.gemm_ar([si.to_f64(a) for a in A], [si.to_f64(b) for b in B])
    assert out.shape == (M, N) and np.all(out == 2 ** W - 1)
