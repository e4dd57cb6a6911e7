"""GPU parity of SP attention (NEXT-4: sequence-parallel attention over all-gathered KV,
consumed in ring/arrival order) vs the fp64 oracle (oracle/attn.py), through the C ABI.

Tolerance: the north-star bound (1e-2 per element relative to max(1, |ref|)); Frobenius:
2e-3, or -- P enters the P.V MMA as bf16 (bf16-in / fp32-accumulate, Q27) and the
output is bf16 -- 1.15x the floor of that arithmetic when it is higher: the relative
Frobenius error of the bf16-P oracle variant (oracle/attn.py attention_p_bf16, pinned in
tests/test_oracle_attn.py) rounded to bf16, against the exact fp64 result, computed for the
same inputs (measured ~2.2-2.3e-3 on N(0,1) scores; the kernels measure ~2.3e-3)."""
import numpy as np
import pytest
import torch

from oracle import attn as oatt
from oracle import numeric as on
from synthetic import inputs as si

pytestmark = pytest.mark.gpu
SMS = 148
FROB = 2e-3  # north star; raised to 1.15x the bf16-P floor per case (see _frob_bound)


def _frob_bound(ref, ref_p_bf16):
    floor = np.linalg.norm(oatt.round_bf16(ref_p_bf16) - ref) / np.linalg.norm(ref)
    return max(FROB, 1.15 * floor)


def _check_full(got, Qn, Kn, Vn, r, causal, what):
    ref = oatt.sp_attention(Qn, Kn, Vn, r, 128 ** -0.5, causal=causal)
    refb = oatt.sp_attention_p_bf16(Qn, Kn, Vn, r, 128 ** -0.5, causal=causal)
    ok, e, f = on.check_tolerance(got, ref, frob_rel=_frob_bound(ref, refb))
    assert ok, f"{what}: max elem err {e:.3e}, frob {f:.3e} (bound {_frob_bound(ref, refb):.3e})"


def _check_rows(got, Qn, Kn, Vn, r, heads, rows, causal, what):
    ref = oatt.sp_attention_rows(Qn, Kn, Vn, r, 128 ** -0.5, heads, rows, causal=causal)
    refb = oatt.sp_attention_rows(Qn, Kn, Vn, r, 128 ** -0.5, heads, rows, causal=causal, p_bf16=True)
    ok, e, f = on.check_tolerance(got, ref, frob_rel=_frob_bound(ref, refb))
    assert ok, f"{what}: max elem err {e:.3e}, frob {f:.3e} (bound {_frob_bound(ref, refb):.3e})"


@pytest.fixture(scope="module")
def ao():
    from paper_2601_20595_b200 import build
    build.build(verbose=False)
    import paper_2601_20595_b200.api as api
    return api


def _world(ao, W, H, S, C, n_cta, **kw):
    d = dict(op="sp_attn", world_size=W, M=S, N=H, K=128, chunk_rows=C, backend="ce", n_cta=n_cta,
             timeout_ns=2_000_000_000)
    d.update(kw)
    ctxs = ao.loopback_world(0, W, ao.workspace_bytes(d))
    return ctxs, [ao.Plan(ctxs[r], dict(d, rank=r)) for r in range(W)]


def _run(ao, ctxs, plans, Q, K, V):
    O = [torch.full_like(q, float("nan"), device="cuda") for q in Q]
    ao.sp_attn_group(plans, [q.cuda() for q in Q], [k.cuda() for k in K], [v.cuda() for v in V], O)
    torch.cuda.synchronize()
    for c in ctxs:
        c.check_async()
    return O


def _check(O, Q, K, V, what):
    Qn, Kn, Vn = ([si.to_f64(t) for t in x] for x in (Q, K, V))
    for r in range(len(O)):
        _check_full(O[r].float().cpu().numpy(), Qn, Kn, Vn, r, False, f"{what} rank {r}")


@pytest.mark.parametrize("W,H,S,C", [(1, 1, 128, 128), (1, 2, 256, 128), (2, 2, 256, 256), (4, 2, 128, 128),
                                     (8, 1, 256, 128)])
def test_sp_attn_vs_oracle(ao, W, H, S, C):
    Q, K, V = si.attn_inputs(W, H, S, 128, salt=W * 10 + H)
    ctxs, plans = _world(ao, W, H, S, C, max(1, SMS // W))
    O = _run(ao, ctxs, plans, Q, K, V)
    _check(O, Q, K, V, f"sp_attn W={W} H={H} S={S} C={C}")


@pytest.mark.parametrize("W", [2, 4])
def test_sp_attn_timesliced_and_epochs(ao, W):
    H, S = 3, 256
    ctxs, plans = _world(ao, W, H, S, 256, SMS)
    for it in range(3):  # both parities, flags re-armed by the epoch
        Q, K, V = si.attn_inputs(W, H, S, 128, salt=100 + it)
        O = _run(ao, ctxs, plans, Q, K, V)
        _check(O, Q, K, V, f"sp_attn ts W={W} it={it}")


def test_sp_attn_few_ctas_many_items(ao):
    """More items than CTAs (each CTA loops over several (head, q-block) items and
    several KV blocks per source): the barrier phases across items."""
    W, H, S = 2, 4, 512
    Q, K, V = si.attn_inputs(W, H, S, 128, salt=7)
    ctxs, plans = _world(ao, W, H, S, 512, 3)
    O = _run(ao, ctxs, plans, Q, K, V)
    _check(O, Q, K, V, "sp_attn few ctas")


def test_sp_attn_llama_sampled(ao):
    """Llama-3-8B attention shape, SP over 8 ranks (loopback, time-sliced): 32 heads,
    d = 128, 16384 tokens (2048 per rank); sampled rows of three heads vs fp64."""
    W, H, S = 8, 32, 2048
    Q, K, V = si.attn_inputs(W, H, S, 128)
    ctxs, plans = _world(ao, W, H, S, 2048, SMS, timeout_ns=10_000_000_000)
    O = _run(ao, ctxs, plans, Q, K, V)
    Qn, Kn, Vn = ([si.to_f64(t) for t in x] for x in (Q, K, V))
    rows = np.array([0, 127, 128, 1000, 2047])
    for r in (0, 5):
        got = O[r][[0, 13, 31]][:, rows].float().cpu().numpy()
        _check_rows(got, Qn, Kn, Vn, r, [0, 13, 31], rows, False, f"llama sampled rank {r}")


@pytest.mark.parametrize("W,H,S", [(1, 2, 256), (2, 2, 256), (4, 1, 512), (8, 2, 256)])
@pytest.mark.parametrize("ts", [False, True])
def test_sp_attn_causal_vs_oracle(ao, W, H, S, ts):
    """Causal ring attention: rank r's queries see the shards of ranks <= r (own shard
    masked on the diagonal blocks); per-rank work differs (rank 0 has the least)."""
    Q, K, V = si.attn_inputs(W, H, S, 128, salt=70 + W)
    ctxs, plans = _world(ao, W, H, S, S, SMS if ts else max(1, SMS // W), causal=1)
    O = _run(ao, ctxs, plans, Q, K, V)
    Qn, Kn, Vn = ([si.to_f64(t) for t in x] for x in (Q, K, V))
    for r in range(W):
        _check_full(O[r].float().cpu().numpy(), Qn, Kn, Vn, r, True, f"causal W={W} H={H} S={S} ts={ts} rank {r}")


def test_sp_attn_causal_llama_sampled(ao):
    W, H, S = 8, 32, 2048
    Q, K, V = si.attn_inputs(W, H, S, 128, salt=3)
    ctxs, plans = _world(ao, W, H, S, 2048, SMS, causal=1, timeout_ns=10_000_000_000)
    O = _run(ao, ctxs, plans, Q, K, V)
    Qn, Kn, Vn = ([si.to_f64(t) for t in x] for x in (Q, K, V))
    rows = np.array([0, 127, 128, 255, 256, 1000, 2047])
    for r in (0, 3, 7):
        got = O[r][[0, 31]][:, rows].float().cpu().numpy()
        _check_rows(got, Qn, Kn, Vn, r, [0, 31], rows, True, f"causal llama rank {r}")


@pytest.mark.parametrize("causal", [0, 1])
def test_sp_attn_per_rank_calls_on_separate_streams(ao, causal):
    """One ao_sp_attn call per rank (n_group = 1), each on its own stream with its own
    copy-engine chain, as with one process per GPU."""
    W, H, S = 2, 2, 512
    Q, K, V = si.attn_inputs(W, H, S, 128, salt=90 + causal)
    ctxs, plans = _world(ao, W, H, S, 512, 32, causal=causal)
    streams = [torch.cuda.Stream() for _ in range(W)]
    dQ, dK, dV = [q.cuda() for q in Q], [k.cuda() for k in K], [v.cuda() for v in V]
    Qn, Kn, Vn = ([si.to_f64(t) for t in x] for x in (Q, K, V))
    for it in range(2):
        O = [torch.empty_like(q) for q in dQ]
        for r in (1, 0) if it % 2 else (0, 1):
            ao.sp_attn(plans[r], dQ[r], dK[r], dV[r], O[r], stream=streams[r])
        torch.cuda.synchronize()
        for c in ctxs:
            c.check_async()
        for r in range(W):
            _check_full(O[r].float().cpu().numpy(), Qn, Kn, Vn, r, bool(causal),
                        f"per-rank attn causal={causal} it={it} r{r}")


@pytest.mark.parametrize("S,causal", [(256, 0), (256, 1), (128, 0)])
def test_sp_attn_peaked_scores_rescale_and_underflow(ao, S, causal):
    """Sharp softmax: q scaled by 6 and rank s's keys by (s + 1) / 2, so scaled scores reach
    ~+-60 (the row max moves by more than the 2^8 lazy-rescale threshold between KV blocks
    in ring order, and most exponentials underflow to 0 in the ftz exp2).  S = 128 runs
    the one-tile kernel, S = 256 the ping-pong kernel."""
    W, H = 4, 2
    Q, K, V = si.attn_inputs(W, H, S, 128, salt=200 + S + causal)
    Q = [(q.float() * 6.0).to(torch.bfloat16) for q in Q]
    K = [(k.float() * (0.5 * (s + 1))).to(torch.bfloat16) for s, k in enumerate(K)]
    ctxs, plans = _world(ao, W, H, S, S, SMS, causal=causal)
    O = _run(ao, ctxs, plans, Q, K, V)
    Qn, Kn, Vn = ([si.to_f64(t) for t in x] for x in (Q, K, V))
    for r in range(W):
        _check_full(O[r].float().cpu().numpy(), Qn, Kn, Vn, r, bool(causal), f"peaked S={S} causal={causal} rank {r}")


@pytest.mark.parametrize("causal", [0, 1])
def test_sp_attn_bitwise_repeatable(ao, causal):
    """The kernels' order of operations is fixed (KV blocks in ring order, fixed-tree row
    sums), so repeated calls on the same inputs are bit-identical.  This also guards the
    MMA warp's reliance on in-order tcgen05 execution (S_x(n+1) overwrites P_x(n) in TMEM
    without a completion wait): a race there would make the runs differ."""
    W, H, S = 8, 4, 512
    Q, K, V = si.attn_inputs(W, H, S, 128, salt=300 + causal)
    ctxs, plans = _world(ao, W, H, S, S, SMS, causal=causal)
    first = _run(ao, ctxs, plans, Q, K, V)
    for it in range(4):
        again = _run(ao, ctxs, plans, Q, K, V)
        for r in range(W):
            assert torch.equal(first[r], again[r]), f"causal={causal} run {it} rank {r} differs"


def test_sp_attn_causal_epochs_without_host_sync(ao):
    """Causal ring attention, per-rank calls on separate streams, 4 epochs back to back
    with different K/V each epoch and no host synchronisation in between.  A causal rank
    waits only on lower ranks, so without the done-word ordering rank 0 (the shortest
    kernels) could push epoch e+2's K/V into a higher rank's parity-(e % 2) buffer while
    that rank's epoch-e kernel still reads it (Q11)."""
    W, H, S, E = 3, 2, 256, 4
    ctxs, plans = _world(ao, W, H, S, 256, 32, causal=1)
    streams = [torch.cuda.Stream() for _ in range(W)]
    ins, outs = [], []
    for e in range(E):
        Q, K, V = si.attn_inputs(W, H, S, 128, salt=300 + e)
        ins.append((Q, K, V))
        dQ, dK, dV = [q.cuda() for q in Q], [k.cuda() for k in K], [v.cuda() for v in V]
        outs.append(([torch.empty_like(q) for q in dQ], dQ, dK, dV))
    torch.cuda.synchronize()
    for e in range(E):  # collective order: every rank issues epoch e before epoch e+1
        O, dQ, dK, dV = outs[e]
        for r in range(W):
            ao.sp_attn(plans[r], dQ[r], dK[r], dV[r], O[r], stream=streams[r])
    torch.cuda.synchronize()
    for c in ctxs:
        c.check_async()
    for e in range(E):
        Q, K, V = ins[e]
        Qn, Kn, Vn = ([si.to_f64(t) for t in x] for x in (Q, K, V))
        for r in range(W):
            _check_full(outs[e][0][r].float().cpu().numpy(), Qn, Kn, Vn, r, True, f"causal epoch {e} rank {r}")


# ---- head-parallel (Ulysses) attention: the same result, computed per head group ---------
def _hp_world(ao, W, H, S, C, n_cta, **kw):
    d = dict(op="hp_attn", world_size=W, M=S, N=H, K=128, chunk_rows=C, backend="ce", n_cta=n_cta,
             timeout_ns=2_000_000_000)
    d.update(kw)
    ctxs = ao.loopback_world(0, W, ao.workspace_bytes(d))
    return ctxs, [ao.Plan(ctxs[r], dict(d, rank=r)) for r in range(W)]


def _run_hp(ao, ctxs, plans, Q, K, V):
    O = [torch.full_like(q, float("nan"), device="cuda") for q in Q]
    ao.hp_attn_group(plans, [q.cuda() for q in Q], [k.cuda() for k in K], [v.cuda() for v in V], O)
    torch.cuda.synchronize()
    for c in ctxs:
        c.check_async()
    return O


@pytest.mark.parametrize("causal", [0, 1])
@pytest.mark.parametrize("ts", [False, True])
@pytest.mark.parametrize("W,H,S,C", [(1, 2, 256, 256), (2, 2, 256, 256), (2, 4, 512, 128), (4, 4, 256, 128),
                                     (8, 8, 256, 256), (4, 8, 512, 256)])
def test_hp_attn_vs_oracle(ao, W, H, S, C, ts, causal):
    """HP attention (DeepSpeed-Ulysses): rank r computes heads [r*H/W, (r+1)*H/W) for
    every source's queries over every source's keys (all-to-all in, output tiles written
    straight to their owners); the result equals SP attention's (same oracle)."""
    Q, K, V = si.attn_inputs(W, H, S, 128, salt=500 + 10 * W + H + causal)
    ctxs, plans = _hp_world(ao, W, H, S, C, SMS if ts else max(1, SMS // W), causal=causal)
    O = _run_hp(ao, ctxs, plans, Q, K, V)
    Qn, Kn, Vn = ([si.to_f64(t) for t in x] for x in (Q, K, V))
    for r in range(W):
        _check_full(O[r].float().cpu().numpy(), Qn, Kn, Vn, r, bool(causal),
                    f"hp W={W} H={H} S={S} ts={ts} causal={causal} rank {r}")
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("causal", [0, 1])
def test_hp_attn_per_rank_calls_epochs_without_host_sync(ao, causal):
    """One ao_hp_attn call per rank on its own stream (as with one process per GPU), three
    epochs back to back with different inputs and no host synchronisation: the return
    buffers and flags are reused across the epoch parities (Q11)."""
    W, H, S, E = 2, 4, 512, 3
    ctxs, plans = _hp_world(ao, W, H, S, 256, 32, causal=causal)
    streams = [torch.cuda.Stream() for _ in range(W)]
    ins, outs = [], []
    for e in range(E):
        Q, K, V = si.attn_inputs(W, H, S, 128, salt=600 + e + 10 * causal)
        ins.append((Q, K, V))
        dQ, dK, dV = [q.cuda() for q in Q], [k.cuda() for k in K], [v.cuda() for v in V]
        outs.append(([torch.empty_like(q) for q in dQ], dQ, dK, dV))
    torch.cuda.synchronize()
    for e in range(E):
        O, dQ, dK, dV = outs[e]
        for r in (range(W) if e % 2 == 0 else reversed(range(W))):
            ao.hp_attn(plans[r], dQ[r], dK[r], dV[r], O[r], stream=streams[r])
    torch.cuda.synchronize()
    for c in ctxs:
        c.check_async()
    for e in range(E):
        Q, K, V = ins[e]
        Qn, Kn, Vn = ([si.to_f64(t) for t in x] for x in (Q, K, V))
        for r in range(W):
            _check_full(outs[e][0][r].float().cpu().numpy(), Qn, Kn, Vn, r, bool(causal),
                        f"hp per-rank causal={causal} epoch {e} rank {r}")
    for c in ctxs:
        c.close()


def test_hp_attn_llama_sampled(ao):
    """Llama-3-8B attention, 32 heads over 8 ranks (4 per rank), 2048 tokens per rank
    (16384 total), time-sliced loopback; sampled rows of three heads vs fp64."""
    W, H, S = 8, 32, 2048
    Q, K, V = si.attn_inputs(W, H, S, 128, salt=7)
    ctxs, plans = _hp_world(ao, W, H, S, 2048, SMS, timeout_ns=10_000_000_000)
    O = _run_hp(ao, ctxs, plans, Q, K, V)
    Qn, Kn, Vn = ([si.to_f64(t) for t in x] for x in (Q, K, V))
    rows = np.array([0, 127, 128, 1000, 2047])
    for r in (0, 5):
        got = O[r][[0, 13, 31]][:, rows].float().cpu().numpy()
        _check_rows(got, Qn, Kn, Vn, r, [0, 13, 31], rows, False, f"hp llama sampled rank {r}")
    for c in ctxs:
        c.close()
