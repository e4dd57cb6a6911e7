"""CPU fp64 oracle for the A2A-GEMM workload (MoE dispatch + expert GEMM; SURVEY.md §8(f)
NEXT-3, BASELINE.json configs[3]: "Mixtral-8x7B MoE All-to-All dispatch + grouped expert
GEMM, 8 experts over 8 GPUs, top-2, 8192 tokens").

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
`cpu_baseline` / `--impl reference` legs may import this module.  It shares no code with
the CUDA path (paper_2601_20595_b200/), and the CUDA path never imports it.

The paper names A2A-GEMM as one of its communication-heavy operators ("A2A-GEMM and
GEMM-AR ... benefit from intermediate split factors"; P:529 split-factor study) and lists
All-to-All among the collectives its plans contain, but prints no
definition.  The reading taken (Q25) is the standard expert-parallel dispatch
(one expert per rank, expert e lives on rank e) followed by the expert GEMM:

  * rank s holds tokens X_s [T, H] and routing idx_s [T, k] (k distinct expert ids per
    token, the top-k of its router logits);
  * send set  S(s -> e) = the token ids t (ascending) with e in idx_s[t, :];
  * All-to-All (the `all_to_all_single` concatenation, source-rank order):
        A_e = concat_{s = 0..W-1} X_s[S(s -> e)]                     [R_e, H]
  * route position of (s, t, j): the row of token t of rank s in A_{idx_s[t, j]}
        pos_s[t, j] = sum_{s' < s} |S(s' -> e)| + #{t' in S(s -> e) : t' < t},  e = idx_s[t, j]
  * expert GEMM (Lst.1's local kernel):  Y_e = A_e . B_e^T  with B_e [N, H].

Pins (tests/test_oracle_a2a.py): per-token combine identity through an independent
matvec path, conservation of the routed rows, closed forms of structured routings
(all-local, shifted, round-robin top-2), exact-integer provenance, brute force.
"""
from __future__ import annotations

import numpy as np


def send_sets(idx, W: int):
    """S(s -> e) for one source: ascending token ids routed to each expert e < W."""
    idx = np.asarray(idx)
    return [np.nonzero((idx == e).any(axis=1))[0] for e in range(W)]


def counts(idx_list, W: int):
    """cnt[s][e] = |S(s -> e)| (the count matrix every rank learns before placing rows)."""
    return np.array([[len(x) for x in send_sets(idx, W)] for idx in idx_list], dtype=np.int64)


def dispatch(X_list, idx_list):
    """All-to-All dispatch: A_e = concat_s X_s[S(s -> e)] for every expert rank e."""
    W = len(X_list)
    sets = [send_sets(idx, W) for idx in idx_list]
    out = []
    for e in range(W):
        parts = [np.asarray(X_list[s], dtype=np.float64)[sets[s][e]] for s in range(W)]
        out.append(np.concatenate(parts, axis=0))
    return out


def route_positions(idx_list):
    """pos_s[t, j]: row of (s, t) in A_{idx_s[t, j]} (definition in the module docstring)."""
    W = len(idx_list)
    cnt = counts(idx_list, W)
    res = []
    for s, idx in enumerate(idx_list):
        idx = np.asarray(idx)
        pos = np.zeros(idx.shape, dtype=np.int64)
        sets = send_sets(idx, W)
        for e in range(W):
            base = int(cnt[:s, e].sum())
            rank_in_set = {int(t): i for i, t in enumerate(sets[e])}
            for t, j in zip(*np.nonzero(idx == e)):
                pos[t, j] = base + rank_in_set[int(t)]
        res.append(pos)
    return res


def a2a_gemm(X_list, idx_list, B_list):
    """Y_e = A_e . B_e^T in float64 for every expert rank e (the op's numerical result)."""
    return [A @ np.asarray(B, dtype=np.float64).T for A, B in zip(dispatch(X_list, idx_list), B_list)]


def a2a_gemm_rows(X_list, idx_list, B_e, e: int, rows):
    """Selected rows of Y_e (full-size sampled checks): rows of A_e located through the
    count matrix, then one row block of the GEMM."""
    W = len(X_list)
    cnt = counts(idx_list, W)
    rows = np.asarray(rows)
    starts = np.concatenate([[0], np.cumsum(cnt[:, e])])
    A = np.zeros((len(rows), np.asarray(X_list[0]).shape[1]), dtype=np.float64)
    for i, r in enumerate(rows):
        s = int(np.searchsorted(starts, r, side="right") - 1)
        t = send_sets(idx_list[s], W)[e][r - starts[s]]
        A[i] = np.asarray(X_list[s][t], dtype=np.float64)
    return A @ np.asarray(B_e, dtype=np.float64).T


def schedule(cnt, e: int, T: int, C: int, BM: int, n_nb: int, gm: int):
    """The chunk-ordered tile list of expert e (Q26), row by row:

      * chunk (s, j) = rows j*C .. (j+1)*C - 1 of source s's block (S(s -> e) in the
        receive layout), arrival position pos(s, j) = ((e - s) mod W) * maxJ + j with
        maxJ = ceil(T / C) (the push rotation of Lst.2 P:249-265: own rows first, then the
        sources e-1, e-2, ... as each pushes to its next peer);
      * row block mb (rows mb*BM .. of the R_e received rows) depends on every chunk that
        one of its rows belongs to (chunk_before_tile) and joins the latest of them
        (S:430);
      * row blocks are ordered by that position (ties by block index), then tiles follow
        Triton's GROUP_M swizzle over the ordered blocks (Fig.6).

    Returns [(mb, nb), ...] in execution order."""
    cnt = np.asarray(cnt)
    W = cnt.shape[0]
    maxJ = -(-T // C)
    owner_of_row = []  # (source, chunk) of every received row, by walking the blocks
    for s in range(W):
        for i in range(int(cnt[s, e])):
            owner_of_row.append((s, i // C))
    R = len(owner_of_row)
    nmb = -(-R // BM)
    key = []
    for mb in range(nmb):
        key.append(max(((e - s) % W) * maxJ + j for s, j in owner_of_row[mb * BM:(mb + 1) * BM]))
    blocks = sorted(range(nmb), key=lambda mb: (key[mb], mb))
    out = []
    per = gm * n_nb
    for k in range(nmb * n_nb):
        first = (k // per) * gm
        size = min(nmb - first, gm)
        r = k % per
        out.append((blocks[first + r % size], r // size))
    return out
