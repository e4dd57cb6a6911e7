"""Worker of tests/test_gpu_multiproc.py: ONE RANK PER PROCESS (the production deployment,
DESIGN.md §11), several processes sharing the one GPU of the test box.

Launched by torch.distributed.run; the process group (gloo: NCCL refuses two ranks on one
GPU) only exchanges the IPC handles (api.dist_world -> cudaIpcOpenMemHandle).  Every op
runs through the C ABI with n_group = 1 per process; results are checked in each process
against the fp64 oracle (tolerance of the north star), provenance decodes bit-exactly.
Prints one JSON line per case; exits 1 on the first failure."""
import json
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2601_20595_b200 as ao  # noqa: E402
from oracle import a2a as oa  # noqa: E402
from oracle import attn as oatt  # noqa: E402
from oracle import numeric as on  # noqa: E402
from synthetic import inputs as si  # noqa: E402

TMO = 30_000_000_000


def log(rank, case, ok, **kw):
    print(json.dumps(dict(rank=rank, case=case, ok=ok, **kw)), flush=True)


def check(gpu, ref, what):
    ok, e, f = on.check_tolerance(gpu.float().cpu().numpy(), ref)
    assert ok, f"{what}: elem {e:.3e} frob {f:.3e}"


def main():
    dist.init_process_group("gloo")
    rank, W = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    cases = sys.argv[1].split(",") if len(sys.argv) > 1 else ["all"]
    n_cta = max(2, 148 // W // 2)  # per process: all processes. CTAs fit the SMs together
    ws = 64 << 20
    ctx = ao.dist_world(0, ws)
    stream = torch.cuda.Stream()

    def want(c):
        return "all" in cases or c in cases

    def run(name, fn):
        print(json.dumps(dict(rank=rank, case=name, start=True)), flush=True)
        try:
            with torch.cuda.stream(stream):
                extra = fn() or {}
            torch.cuda.synchronize()
            ctx.check_async()
            log(rank, name, True, **extra)
        except Exception as e:  # noqa: BLE001
            log(rank, name, False, err=f"{type(e).__name__}: {e}", tb=traceback.format_exc()[-800:])
            dist.barrier()
            sys.exit(1)
        dist.barrier()

    M, K, N, C = 256 * W, 256, 384, 64
    # ---- AG-GEMM: every backend, push (and CE pull), random data vs oracle + provenance epochs
    for backend, dirn in (("ce", "push"), ("tma", "push"), ("ldst", "push"), ("ce", "pull"), ("ldst", "pull")):
        name = f"ag_{backend}_{dirn}"
        if not want("ag") and not want(name):
            continue

        def f(backend=backend, dirn=dirn):
            d = dict(op="ag_gemm", world_size=W, rank=rank, M=M, N=N, K=K, chunk_rows=C, backend=backend, dir=dirn,
                     n_slices=2, tile_m=128, tile_n=128, n_cta=n_cta, timeout_ns=TMO)
            p = ao.Plan(ctx, d)
            A, B = si.ag_inputs(W, M, K, N, salt=11)
            Cg = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
            G = torch.empty(M, K, dtype=torch.bfloat16, device="cuda")
            ao.ag_gemm(p, A[rank].cuda(), B[rank].cuda(), Cg, G)
            torch.cuda.synchronize()
            ctx.check_async()
            check(Cg, on.ag_gemm([si.to_f64(a) for a in A], si.to_f64(B[rank])), "ag")
            assert torch.equal(G.cpu(), torch.cat(A, 0)), "gathered copy not bit-exact"
            for ep in range(5):  # back-to-back epochs, no host sync between them
                Ap, Bp = si.ag_provenance_inputs(W, M, 64 if K < 64 else K, N, epoch=ep + 1)
                outs = []
                Cp = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
                ao.ag_gemm(p, Ap[rank].cuda(), Bp[rank].cuda(), Cp)
                outs.append(Cp)
                torch.cuda.synchronize()
                c = Cp.float().cpu()
                rid = c[:, 0] + 32 * c[:, 1] + 1024 * c[:, 2]
                assert torch.equal(rid, torch.arange(M, dtype=torch.float32)), f"provenance rows epoch {ep}"
                assert torch.all(c[:, 3] == (ep + 1) % 32), f"provenance epoch {ep}"
            p.close()
        run(name, f)

    # ---- GEMM-RS: slots and atomic, random vs oracle, bitmask provenance, determinism (slots)
    for red in ("slots", "atomic"):
        name = f"rs_{red}"
        if not want("rs") and not want(name):
            continue

        def f(red=red):
            d = dict(op="gemm_rs", world_size=W, rank=rank, M=M, N=N, K=K, chunk_rows=C, tile_m=128, tile_n=128,
                     n_cta=n_cta, rs_reduce=red, timeout_ns=TMO)
            p = ao.Plan(ctx, d)
            A, B = si.rs_inputs(W, M, K, N, salt=12)
            D = torch.empty(M // W, N, dtype=torch.bfloat16, device="cuda")
            ao.gemm_rs(p, A[rank].cuda(), B[rank].cuda(), D)
            torch.cuda.synchronize()
            ctx.check_async()
            check(D, on.gemm_rs([si.to_f64(a) for a in A], [si.to_f64(b) for b in B], rank), "rs")
            if red == "slots":
                D2 = torch.empty_like(D)
                ao.gemm_rs(p, A[rank].cuda(), B[rank].cuda(), D2)
                torch.cuda.synchronize()
                assert torch.equal(D, D2), "slots RS must be bitwise deterministic"
            Ap, Bp = si.rs_provenance_inputs(W, M, K, N)
            for ep in range(5):
                ao.gemm_rs(p, Ap[rank].cuda(), Bp[rank].cuda(), D)
            torch.cuda.synchronize()
            assert torch.all(D.float().cpu() == 2 ** W - 1), "bitmask provenance"
            p.close()
        run(name, f)

    if want("sk"):
        # AG with the stream-K tail (Q28): W=2: 12 tiles on 5 workers -> 5 data-parallel, 7 split
        def f():
            d = dict(op="ag_gemm", world_size=W, rank=rank, M=M, N=N, K=K, chunk_rows=C, backend="ce", tile_m=128,
                     tile_n=128, n_cta=5, stream_k=1, timeout_ns=TMO)
            p = ao.Plan(ctx, d)
            T = (M // 128) * ((N + 127) // 128)
            assert json.loads(p.export_json()).get("sk_dp") == (T // 5 - 1) * 5
            A, B = si.ag_inputs(W, M, K, N, salt=15)
            Cg = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
            for _ in range(3):
                ao.ag_gemm(p, A[rank].cuda(), B[rank].cuda(), Cg)
            torch.cuda.synchronize()
            ctx.check_async()
            check(Cg, on.ag_gemm([si.to_f64(a) for a in A], si.to_f64(B[rank])), "ag stream-K")
            p.close()
        run("sk", f)

    if want("rs_bf16"):
        # the non-conforming bf16 RS wire (Q14): its own bound, exact bitmask
        def f():
            d = dict(op="gemm_rs", world_size=W, rank=rank, M=M, N=N, K=K, chunk_rows=C, tile_m=128, tile_n=128,
                     n_cta=n_cta, rs_reduce="atomic", rs_wire="bf16", timeout_ns=TMO)
            p = ao.Plan(ctx, d)
            A, B = si.rs_inputs(W, M, K, N, salt=16)
            D = torch.empty(M // W, N, dtype=torch.bfloat16, device="cuda")
            ao.gemm_rs(p, A[rank].cuda(), B[rank].cuda(), D)
            torch.cuda.synchronize()
            ctx.check_async()
            ok, e, fr = on.check_tolerance(D.float().cpu().numpy(),
                                           on.gemm_rs([si.to_f64(a) for a in A], [si.to_f64(b) for b in B], rank),
                                           elem_rel=1e-2 + W * 2.0 ** -8, frob_rel=2e-3 * W ** 0.5)
            assert ok, f"rs bf16 wire: {e:.3e} {fr:.3e}"
            Ap, Bp = si.rs_provenance_inputs(W, M, K, N)
            for ep in range(3):
                ao.gemm_rs(p, Ap[rank].cuda(), Bp[rank].cuda(), D)
            torch.cuda.synchronize()
            assert torch.all(D.float().cpu() == 2 ** W - 1), "bitmask provenance (bf16 wire)"
            p.close()
        run("rs_bf16", f)

    if want("ar"):
        def f():
            d = dict(op="gemm_ar", world_size=W, rank=rank, M=M, N=N, K=K, chunk_rows=C, tile_m=128, tile_n=128,
                     n_cta=n_cta, backend="ldst", n_slices=2, timeout_ns=TMO)
            p = ao.Plan(ctx, d)
            A, B = si.rs_inputs(W, M, K, N, salt=13)
            Cg = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
            for _ in range(3):
                ao.gemm_ar(p, A[rank].cuda(), B[rank].cuda(), Cg)
            torch.cuda.synchronize()
            ctx.check_async()
            check(Cg, on.gemm_ar([si.to_f64(a) for a in A], [si.to_f64(b) for b in B]), "ar")
            p.close()
        run("ar", f)

    if want("a2a"):
        def f():
            T, H, Na, k = 256, 128, 256, min(2, W)
            d = dict(op="a2a_gemm", world_size=W, rank=rank, M=T, N=Na, K=H, topk=k, chunk_rows=32, backend="ldst",
                     tile_m=128, tile_n=128, n_cta=n_cta, timeout_ns=TMO)
            p = ao.Plan(ctx, d)
            X, idx, B = si.moe_inputs(W, T, H, Na, topk=k, zipf=1.1, salt=14)
            Y = torch.zeros(W * T, Na, dtype=torch.bfloat16, device="cuda")
            rp = torch.zeros(T, k, dtype=torch.int32, device="cuda")
            rr = torch.zeros(1, dtype=torch.int32, device="cuda")
            for _ in range(3):
                ao.a2a_gemm(p, X[rank].cuda(), idx[rank].cuda(), B[rank].cuda(), Y, rp, rr)
            torch.cuda.synchronize()
            ctx.check_async()
            In = [i.numpy().astype(np.int64) for i in idx]
            ref = oa.a2a_gemm([si.to_f64(x) for x in X], In, [si.to_f64(b) for b in B])[rank]
            assert int(rr.item()) == ref.shape[0], "received rows"
            np.testing.assert_array_equal(rp.cpu().numpy(), oa.route_positions(In)[rank])
            if ref.shape[0]:
                check(Y[: ref.shape[0]], ref, "a2a")
            p.close()
        run("a2a", f)

    for causal in (0, 1):
        name = f"attn_causal{causal}"
        if not want("attn") and not want(name):
            continue

        def f(causal=causal):
            H, S = 2, 256
            d = dict(op="sp_attn", world_size=W, rank=rank, M=S, N=H, K=128, chunk_rows=256, backend="ce",
                     n_cta=n_cta, causal=causal, timeout_ns=TMO)
            p = ao.Plan(ctx, d)
            outs = []
            for ep in range(4):  # different K/V per epoch, no host sync in between
                Q, Kx, V = si.attn_inputs(W, H, S, 128, salt=400 + ep)
                O = torch.empty(H, S, 128, dtype=torch.bfloat16, device="cuda")
                ao.sp_attn(p, Q[rank].cuda(), Kx[rank].cuda(), V[rank].cuda(), O)
                outs.append((O, Q, Kx, V))
            torch.cuda.synchronize()
            ctx.check_async()
            for ep, (O, Q, Kx, V) in enumerate(outs):
                args = ([si.to_f64(t) for t in Q], [si.to_f64(t) for t in Kx], [si.to_f64(t) for t in V], rank,
                        128 ** -0.5)
                ref = oatt.sp_attention(*args, causal=bool(causal))
                # 2e-3, or 1.15x the bf16-P arithmetic's floor when higher (tests/test_gpu_attn.py)
                refb = oatt.round_bf16(oatt.sp_attention_p_bf16(*args, causal=bool(causal)))
                bound = max(2e-3, 1.15 * np.linalg.norm(refb - ref) / np.linalg.norm(ref))
                ok, e, fr = on.check_tolerance(O.float().cpu().numpy(), ref, frob_rel=bound)
                assert ok, f"attn epoch {ep}: {e:.3e} {fr:.3e}"
            p.close()
        run(name, f)

    for causal in (0, 1):
        name = f"hp_causal{causal}"
        if not want("hp") and not want(name):
            continue

        def f(causal=causal):
            # head-parallel attention: all-to-all of Q/K/V by head group in, output tiles
            # returned to their owners over IPC, 3 epochs without host sync
            H, S = 2 * W, 256
            d = dict(op="hp_attn", world_size=W, rank=rank, M=S, N=H, K=128, chunk_rows=256, backend="ce",
                     n_cta=n_cta, causal=causal, timeout_ns=TMO)
            p = ao.Plan(ctx, d)
            outs = []
            for ep in range(3):
                Q, Kx, V = si.attn_inputs(W, H, S, 128, salt=700 + ep)
                O = torch.empty(H, S, 128, dtype=torch.bfloat16, device="cuda")
                ao.hp_attn(p, Q[rank].cuda(), Kx[rank].cuda(), V[rank].cuda(), O)
                outs.append((O, Q, Kx, V))
            torch.cuda.synchronize()
            ctx.check_async()
            for ep, (O, Q, Kx, V) in enumerate(outs):
                args = ([si.to_f64(t) for t in Q], [si.to_f64(t) for t in Kx], [si.to_f64(t) for t in V], rank,
                        128 ** -0.5)
                ref = oatt.sp_attention(*args, causal=bool(causal))
                refb = oatt.round_bf16(oatt.sp_attention_p_bf16(*args, causal=bool(causal)))
                bound = max(2e-3, 1.15 * np.linalg.norm(refb - ref) / np.linalg.norm(ref))
                ok, e, fr = on.check_tolerance(O.float().cpu().numpy(), ref, frob_rel=bound)
                assert ok, f"hp epoch {ep}: {e:.3e} {fr:.3e}"
            p.close()
        run(name, f)

    if want("mismatch"):
        # collective semantics: rank 0 launches a plan whose desc differs (chunk_rows) ->
        # every rank's first launch reports AO_ERR_PEER instead of running a mixed schedule
        def f():
            d = dict(op="ag_gemm", world_size=W, rank=rank, M=M, N=N, K=K, chunk_rows=32 if rank == 0 else 64,
                     backend="ce", tile_m=128, tile_n=128, n_cta=n_cta, timeout_ns=TMO)
            p = ao.Plan(ctx, d)
            A, B = si.ag_inputs(W, M, K, N, salt=15)
            Cg = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
            try:
                ao.ag_gemm(p, A[rank].cuda(), B[rank].cuda(), Cg)
            except ao.AOError as e:
                assert e.status == "AO_ERR_PEER", e
                return {"status": e.status}
            raise AssertionError("plan mismatch across processes was not detected")
        run("mismatch", f)

    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
