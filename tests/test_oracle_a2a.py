"""Pins of the A2A-GEMM oracle (oracle/a2a.py) against facts that do not come from it:
an independent per-token matvec path, conservation of routed rows, closed forms of
structured routings, exact-integer provenance, and a brute-force enumeration."""
import numpy as np
import pytest
import torch

from oracle import a2a as oa
from synthetic import inputs as si


def _np(ts):
    return [si.to_f64(t) for t in ts]


def _ids(ts):
    return [t.numpy().astype(np.int64) for t in ts]


@pytest.mark.parametrize("W,T,k,zipf", [(2, 16, 1, 0.0), (4, 32, 2, 0.0), (8, 64, 2, 0.0), (8, 64, 2, 1.2), (3, 20, 2, 0.0)])
def test_combine_identity_independent_path(W, T, k, zipf):
    """sum_j Y_{e_j}[pos[s,t,j]] == X_s[t] . (sum_j B_{e_j})^T per token, the right side
    computed token by token with no dispatch (catches misplaced rows, wrong positions,
    wrong block order and dropped tokens)."""
    H, N = 24, 16
    X, idx, B = si.moe_inputs(W, T, H, N, topk=k, zipf=zipf, salt=W * T)
    Xn, In, Bn = _np(X), _ids(idx), _np(B)
    Y = oa.a2a_gemm(Xn, In, Bn)
    pos = oa.route_positions(In)
    for s in range(W):
        for t in range(T):
            lhs = sum(Y[In[s][t, j]][pos[s][t, j]] for j in range(k))
            rhs = np.zeros(N)
            for j in range(k):
                Be = Bn[In[s][t, j]]
                rhs += np.array([float(np.dot(Xn[s][t], Be[n])) for n in range(N)])
            np.testing.assert_allclose(lhs, rhs, rtol=1e-12, atol=1e-12)


def test_conservation_of_routed_rows():
    W, T, k, H = 4, 40, 2, 8
    X, idx, _ = si.moe_inputs(W, T, H, 8, topk=k, salt=5)
    Xn, In = _np(X), _ids(idx)
    A = oa.dispatch(Xn, In)
    assert sum(a.shape[0] for a in A) == W * T * k
    got = np.concatenate(A, 0)
    want = np.concatenate([np.repeat(Xn[s], k, axis=0) for s in range(W)], 0)
    key = lambda m: m[np.lexsort(m.T[::-1])]
    np.testing.assert_array_equal(key(got), key(want))
    cnt = oa.counts(In, W)
    assert cnt.sum() == W * T * k and (cnt.sum(axis=1) == T * k).all()


def test_all_local_routing_is_plain_gemm():
    W, T, H, N = 4, 16, 8, 12
    X, _, B = si.moe_inputs(W, T, H, N, topk=1, salt=9)
    idx = [np.full((T, 1), s) for s in range(W)]
    Xn, Bn = _np(X), _np(B)
    Y = oa.a2a_gemm(Xn, idx, Bn)
    for e in range(W):
        np.testing.assert_array_equal(oa.dispatch(Xn, idx)[e], Xn[e])
        np.testing.assert_allclose(Y[e], Xn[e] @ Bn[e].T, rtol=0, atol=0)
        np.testing.assert_array_equal(oa.route_positions(idx)[e][:, 0], np.arange(T))


def test_shifted_routing_closed_form():
    W, T, H = 5, 12, 6
    X, _, _ = si.moe_inputs(W, T, H, 4, topk=1, salt=11)
    idx = [np.full((T, 1), (s + 1) % W) for s in range(W)]
    A = oa.dispatch(_np(X), idx)
    for e in range(W):
        np.testing.assert_array_equal(A[e], _np(X)[(e - 1) % W])


def test_round_robin_top2_counts_and_blocks():
    """idx[t] = (t mod W, (t+1) mod W): block s of A_e holds the tokens t with
    t = e or t = e - 1 (mod W), ascending; every count is 2T/W."""
    W, T, H = 4, 16, 4
    X, _, _ = si.moe_inputs(W, T, H, 4, topk=2, salt=13)
    idx = [np.stack([np.arange(T) % W, (np.arange(T) + 1) % W], 1) for _ in range(W)]
    cnt = oa.counts(idx, W)
    assert (cnt == 2 * T // W).all()
    A = oa.dispatch(_np(X), idx)
    for e in range(W):
        toks = [t for t in range(T) if t % W == e or t % W == (e - 1) % W]
        want = np.concatenate([_np(X)[s][toks] for s in range(W)], 0)
        np.testing.assert_array_equal(A[e], want)


def test_provenance_decodes_sorted_token_ids():
    W, T, H, N = 4, 48, 8, 8
    _, idx, _ = si.moe_inputs(W, T, H, N, topk=2, salt=17)
    X, idx, B = si.moe_provenance_inputs(W, T, H, N, idx, epoch=3)
    In = _ids(idx)
    Y = oa.a2a_gemm(_np(X), In, _np(B))
    for e in range(W):
        gid = Y[e][:, 0] + 32 * Y[e][:, 1] + 1024 * Y[e][:, 2]
        want = [s * T + t for s in range(W) for t in range(T) if e in In[s][t]]
        np.testing.assert_array_equal(gid, want)  # source-rank blocks, ascending tokens
        assert (Y[e][:, 3] == 3).all()


def test_brute_force_enumeration_tiny():
    """A_e rebuilt by walking every (source, token, choice) triple in a dictionary keyed by
    destination, independent of the vectorised send sets."""
    W, T, H = 3, 10, 5
    X, idx, _ = si.moe_inputs(W, T, H, 4, topk=2, salt=19)
    Xn, In = _np(X), _ids(idx)
    rows = {e: [] for e in range(W)}
    for s in range(W):
        for t in range(T):
            for j in range(2):
                rows[int(In[s][t, j])].append((s, t))
    A = oa.dispatch(Xn, In)
    pos = oa.route_positions(In)
    for e in range(W):
        order = sorted(rows[e])
        np.testing.assert_array_equal(A[e], np.array([Xn[s][t] for s, t in order]).reshape(-1, H))
        for i, (s, t) in enumerate(order):
            j = int(np.nonzero(In[s][t] == e)[0][0])
            assert pos[s][t, j] == i


def test_sampled_rows_match_full():
    W, T, H, N = 4, 32, 16, 8
    X, idx, B = si.moe_inputs(W, T, H, N, topk=2, zipf=1.0, salt=23)
    Xn, In, Bn = _np(X), _ids(idx), _np(B)
    Y = oa.a2a_gemm(Xn, In, Bn)
    for e in range(W):
        rows = np.arange(0, Y[e].shape[0], 3)
        np.testing.assert_allclose(oa.a2a_gemm_rows(Xn, In, Bn[e], e, rows), Y[e][rows], rtol=0, atol=0)


def test_generator_routing_is_distinct_topk():
    W, T = 8, 256
    for zipf in (0.0, 1.5):
        _, idx, _ = si.moe_inputs(W, T, 4, 4, topk=2, zipf=zipf)
        for t in idx:
            a = t.numpy()
            assert ((a >= 0) & (a < W)).all() and (a[:, 0] != a[:, 1]).all()
    _, idx, _ = si.moe_inputs(W, 4096, 4, 4, topk=2, zipf=1.5)
    c = np.bincount(np.concatenate([t.numpy().ravel() for t in idx]), minlength=W)
    assert c[0] > 2 * c[W - 1]  # skewed toward expert 0


def test_schedule_is_a_permutation_and_follows_arrival():
    """Every tile exactly once; with GROUP_M = 1 the arrival position of a tile's latest
    chunk never decreases along the order; own rows (position 0) first."""
    W, T, C, BM = 8, 256, 64, 128
    _, idx, _ = si.moe_inputs(W, T, 8, 8, topk=2, zipf=1.1, salt=29)
    cnt = oa.counts(_ids(idx), W)
    for e in range(W):
        for gm in (1, 4):
            sch = oa.schedule(cnt, e, T, C, BM, n_nb=3, gm=gm)
            R = int(cnt[:, e].sum())
            nmb = -(-R // BM)
            assert sorted(sch) == [(mb, nb) for mb in range(nmb) for nb in range(3)]
        sch = oa.schedule(cnt, e, T, C, BM, n_nb=3, gm=1)
        starts = np.concatenate([[0], np.cumsum(cnt[:, e])])
        def latest(mb):
            rows = range(mb * BM, min((mb + 1) * BM, starts[-1]))
            best = -1
            for r in rows:
                s = int(np.searchsorted(starts, r, side="right") - 1)
                best = max(best, ((e - s) % W) * (T // C) + (r - starts[s]) // C)
            return best
        keys = [latest(mb) for mb, _ in sch]
        assert keys == sorted(keys)
        if cnt[e, e] >= BM:
            assert sch[0][0] == starts[e] // BM  # a block of the own rows runs first


def test_schedule_closed_form_uniform():
    """cnt = 2T/W everywhere, C = BM = block size: expert e's blocks arrive own block
    first, then the blocks of sources e-1, e-2, ... (the rotation), each block once."""
    W, T, C = 4, 128, 64
    cnt = np.full((W, W), C, dtype=np.int64)  # every source sends exactly one chunk to every expert
    for e in range(W):
        sch = oa.schedule(cnt, e, T, C, BM=C, n_nb=2, gm=1)
        want_blocks = [(e - d) % W for d in range(W)]  # block index == source index here
        assert [mb for mb, nb in sch[::2]] == want_blocks
        assert [nb for _, nb in sch] == [0, 1] * W
