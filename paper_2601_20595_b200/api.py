"""Python binding of the C ABI (include/autooverlap.h) -- same names, marshalling only.

PyTorch is used for device memory, streams and the process group (IPC-handle exchange);
it never computes any step of the hot path.  Tensors are passed to the library as raw
device pointers together with torch's current CUDA stream.

    ctx   = Context(device, rank, world_size, workspace_bytes)
    ctx.import_handles(all_blobs)                  # blobs from every rank
    plan  = Plan(ctx, desc)                        # desc: dict (oracle desc keys)
    ag_gemm(plan, A_shard, B, C)                   # AllGather -> GEMM
    gemm_rs(plan, A, B, C_shard)                   # GEMM -> ReduceScatter
"""
from __future__ import annotations

import ctypes

from . import _native as N
from ._native import AOError, check, lib, make_desc  # noqa: F401


def _ptr(t):
    return ctypes.c_void_p(0 if t is None else int(t.data_ptr()))


def _stream(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream))


def _require_bf16_cuda(*ts):
    import torch
    for t in ts:
        if t is None:
            continue
        if not t.is_cuda or t.dtype != torch.bfloat16 or not t.is_contiguous():
            raise ValueError("operands must be contiguous bf16 CUDA tensors")


def _expect(plan, **named):
    """Shape and device of every operand against the plan's desc (the kernels take their
    extents from the plan, so an undersized tensor would be read / written out of bounds)."""
    dev = plan.ctx.device if plan.ctx is not None else None
    for name, (t, shape) in named.items():
        if t is None:
            continue
        if tuple(t.shape) != tuple(int(x) for x in shape):
            raise AOError(1, f"{name}: shape {tuple(t.shape)} != {tuple(shape)} required by the plan")
        if dev is not None and t.device.index != dev:
            raise AOError(1, f"{name}: on cuda:{t.device.index}, the plan's ctx is on cuda:{dev}")


def _op_shapes(plan):
    d = plan.desc
    W, M, N, K = int(d.get("world_size", 1)), int(d["M"]), int(d["N"]), int(d["K"])
    return W, M, N, K


# ----------------------------------------------------------------------------- plans
def validate(desc: dict, sm_count: int = 148):
    d = make_desc(desc)
    buf = ctypes.create_string_buffer(4096)
    n = ctypes.c_int(0)
    lib().ao_plan_validate(ctypes.byref(d), sm_count, buf, len(buf), ctypes.byref(n))
    v = buf.value.decode()
    return [] if n.value == 0 else v.split(";")


def workspace_bytes(desc: dict) -> int:
    d = make_desc(desc)
    out = ctypes.c_size_t(0)
    check(lib().ao_plan_workspace_bytes(ctypes.byref(d), ctypes.byref(out)))
    return out.value


class Plan:
    """A chunk schedule.  Plan(None, desc, sm_count) is host-only (export / hash);
    Plan(ctx, desc) is bound to a ctx and can be launched."""

    def __init__(self, ctx, desc: dict, sm_count: int = 148):
        if desc.get("backend") == "auto":  # the tuned table's winner for this shape (tune.resolve)
            from .tune import resolve
            desc = resolve(desc)
        self.desc = dict(desc)
        self.ctx = ctx
        d = make_desc(desc)
        h = ctypes.c_void_p()
        if ctx is None:
            check(lib().ao_plan_create_host(ctypes.byref(d), sm_count, ctypes.byref(h)))
        else:
            check(lib().ao_plan_create(ctx.handle, ctypes.byref(d), ctypes.byref(h)))
        self.handle = h

    def export_json(self) -> str:
        need = ctypes.c_size_t(0)
        check(lib().ao_plan_export_json(self.handle, None, 0, ctypes.byref(need)))
        buf = ctypes.create_string_buffer(need.value)
        check(lib().ao_plan_export_json(self.handle, buf, need.value, ctypes.byref(need)))
        return buf.value.decode()

    def hash(self) -> int:
        out = ctypes.c_uint64(0)
        check(lib().ao_plan_hash(self.handle, ctypes.byref(out)))
        return out.value

    def info(self) -> dict:
        vals = [ctypes.c_int32(0) for _ in range(6)]
        check(lib().ao_plan_info(self.handle, *[ctypes.byref(v) for v in vals]))
        keys = ["tile_m", "tile_n", "cta_group", "n_cta", "n_tiles", "n_chunks"]
        return {k: v.value for k, v in zip(keys, vals)}

    def close(self):
        if self.handle:
            lib().ao_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def plan_json(desc: dict, sm_count: int = 148) -> str:
    p = Plan(None, desc, sm_count)
    try:
        return p.export_json()
    finally:
        p.close()


def group_schedule_json(plans, sm_count: int = 148) -> str:
    """ao_group_schedule_export: the launch-level (time-sliced / space-sliced) schedule of a
    group call over `plans` (host-only plans suffice)."""
    arr = (ctypes.c_void_p * len(plans))(*[p.handle.value for p in plans])
    op = N.OPS[plans[0].desc.get("op", "ag_gemm")]
    need = ctypes.c_size_t(0)
    check(lib().ao_group_schedule_export(len(plans), arr, op, sm_count, None, 0, ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    check(lib().ao_group_schedule_export(len(plans), arr, op, sm_count, buf, need.value, ctypes.byref(need)))
    return buf.value.decode()


# ------------------------------------------------------------------------- contexts
class Context:
    def __init__(self, device: int, rank: int, world_size: int, workspace: int):
        h = ctypes.c_void_p()
        check(lib().ao_ctx_create(int(device), int(rank), int(world_size), int(workspace), ctypes.byref(h)))
        self.handle = h
        self.device, self.rank, self.world_size = device, rank, world_size

    def export_handle(self) -> bytes:
        b = N.HandleBlob()
        check(lib().ao_ctx_export_handle(self.handle, ctypes.byref(b)))
        return bytes(b.bytes)

    def import_handles(self, blobs):
        arr = (N.HandleBlob * self.world_size)()
        for i, raw in enumerate(blobs):
            ctypes.memmove(arr[i].bytes, raw, N.AO_HANDLE_BYTES)
        check(lib().ao_ctx_import_handles(self.handle, arr))

    def trace_enable(self, capacity: int = 1 << 20):
        check(lib().ao_ctx_trace_enable(self.handle, int(capacity)))

    def trace_dump(self, path: str) -> int:
        n = ctypes.c_int64(0)
        check(lib().ao_ctx_trace_dump(self.handle, path.encode(), ctypes.byref(n)))
        return n.value

    def check_async(self):
        check(lib().ao_ctx_check_async(self.handle))

    def close(self):
        if self.handle:
            lib().ao_ctx_destroy(self.handle)
            self.handle = None


def loopback_world(device: int, world_size: int, workspace: int):
    """W ranks of one world inside this process on one GPU (SURVEY.md T4 loopback)."""
    ctxs = [Context(device, r, world_size, workspace) for r in range(world_size)]
    blobs = [c.export_handle() for c in ctxs]
    for c in ctxs:
        c.import_handles(blobs)
    return ctxs


def dist_world(device: int, workspace: int, group=None):
    """One rank per process: exchange IPC handles over torch.distributed (plumbing only)."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    ctx = Context(device, rank, world, workspace)
    blobs = [None] * world
    dist.all_gather_object(blobs, ctx.export_handle(), group=group)
    ctx.import_handles(blobs)
    dist.barrier(group)
    return ctx


# ------------------------------------------------------------------------------ ops
def ag_gemm(plan: Plan, A_shard, B, C, A_gathered_out=None, stream=None):
    """ao_ag_gemm: C[M, N] = concat_p(A_p) . B^T for this rank."""
    _require_bf16_cuda(A_shard, B, C, A_gathered_out)
    W, M, N, K = _op_shapes(plan)
    _expect(plan, A_shard=(A_shard, (M // W, K)), B=(B, (N, K)), C=(C, (M, N)), A_gathered_out=(A_gathered_out, (M, K)))
    check(lib().ao_ag_gemm(plan.handle, _ptr(A_shard), _ptr(B), _ptr(C), _ptr(A_gathered_out), _stream(stream)))


def gemm_rs(plan: Plan, A, B, C_shard, stream=None):
    """ao_gemm_rs: C_shard[S, N] = (sum_s A_s . B_s^T)[rank rows]."""
    _require_bf16_cuda(A, B, C_shard)
    W, M, N, K = _op_shapes(plan)
    _expect(plan, A=(A, (M, K)), B=(B, (N, K)), C_shard=(C_shard, (M // W, N)))
    check(lib().ao_gemm_rs(plan.handle, _ptr(A), _ptr(B), _ptr(C_shard), _stream(stream)))


def gemm_ar(plan: Plan, A, B, C, stream=None):
    """ao_gemm_ar (NEXT-1): C[M, N] = sum_s A_s . B_s^T on every rank (partition-based
    AllReduce fused with the GEMM)."""
    _require_bf16_cuda(A, B, C)
    W, M, N, K = _op_shapes(plan)
    _expect(plan, A=(A, (M, K)), B=(B, (N, K)), C=(C, (M, N)))
    check(lib().ao_gemm_ar(plan.handle, _ptr(A), _ptr(B), _ptr(C), _stream(stream)))


def _require_i32_cuda(*ts):
    import torch
    for t in ts:
        if t.dtype != torch.int32 or not t.is_cuda or not t.is_contiguous():
            raise AOError(1, "index arrays must be contiguous int32 CUDA tensors")


def _a2a_expect(plan, X, topk_idx, B, Y, route_pos, recv_rows):
    W, T, N, K = _op_shapes(plan)
    k = int(plan.desc.get("topk", 0))
    _expect(plan, X=(X, (T, K)), topk_idx=(topk_idx, (T, k)), B=(B, (N, K)), Y=(Y, (W * T, N)),
            route_pos=(route_pos, (T, k)), recv_rows=(recv_rows, (1,)))


def _attn_expect(plan, Q, K, V, O):
    _, S, H, D = _op_shapes(plan)
    _expect(plan, Q=(Q, (H, S, D)), K=(K, (H, S, D)), V=(V, (H, S, D)), O=(O, (H, S, D)))


def a2a_gemm(plan: Plan, X, topk_idx, B, Y, route_pos, recv_rows, stream=None):
    """ao_a2a_gemm (NEXT-3): MoE All-to-All dispatch fused with the expert GEMM.  X [T, K]
    bf16 tokens, topk_idx [T, k] int32 experts, B [N, K] this rank's expert; Y [W*T, N]
    (rows [0, recv_rows) valid), route_pos [T, k] int32, recv_rows [1] int32."""
    _require_bf16_cuda(X, B, Y)
    _require_i32_cuda(topk_idx, route_pos, recv_rows)
    _a2a_expect(plan, X, topk_idx, B, Y, route_pos, recv_rows)
    check(lib().ao_a2a_gemm(plan.handle, _ptr(X), _ptr(topk_idx), _ptr(B), _ptr(Y), _ptr(route_pos),
                            _ptr(recv_rows), _stream(stream)))


def a2a_gemm_group(plans, Xs, topk_idxs, Bs, Ys, route_pos, recv_rows, stream=None):
    """ao_a2a_gemm_group: one launch pair (prep + fused) for co-located ranks (loopback)."""
    _require_bf16_cuda(*Xs, *Bs, *Ys)
    _require_i32_cuda(*topk_idxs, *route_pos, *recv_rows)
    for i, p in enumerate(plans):
        _a2a_expect(p, Xs[i], topk_idxs[i], Bs[i], Ys[i], route_pos[i], recv_rows[i])
    check(lib().ao_a2a_gemm_group(len(plans), _plans(plans), _arr(Xs), _arr(topk_idxs), _arr(Bs), _arr(Ys),
                                  _arr(route_pos), _arr(recv_rows), _stream(stream)))


def sp_attn(plan: Plan, Q, K, V, O, stream=None):
    """ao_sp_attn (NEXT-4): O = softmax(Q K_all^T / sqrt(128)) V_all per head; Q/K/V/O
    [H, S_loc, 128] bf16, K/V gathered from all ranks in ring (arrival) order."""
    _require_bf16_cuda(Q, K, V, O)
    _attn_expect(plan, Q, K, V, O)
    check(lib().ao_sp_attn(plan.handle, _ptr(Q), _ptr(K), _ptr(V), _ptr(O), _stream(stream)))


def sp_attn_group(plans, Qs, Ks, Vs, Os, stream=None):
    """ao_sp_attn_group: one launch for co-located ranks (loopback)."""
    _require_bf16_cuda(*Qs, *Ks, *Vs, *Os)
    for i, p in enumerate(plans):
        _attn_expect(p, Qs[i], Ks[i], Vs[i], Os[i])
    check(lib().ao_sp_attn_group(len(plans), _plans(plans), _arr(Qs), _arr(Ks), _arr(Vs), _arr(Os),
                                 _stream(stream)))


def hp_attn(plan: Plan, Q, K, V, O, stream=None):
    """ao_hp_attn (NEXT-4, head-parallel / Ulysses): the result of sp_attn, computed by this
    rank for its head group over all ranks' queries and keys (all-to-all in and out)."""
    _require_bf16_cuda(Q, K, V, O)
    _attn_expect(plan, Q, K, V, O)
    check(lib().ao_hp_attn(plan.handle, _ptr(Q), _ptr(K), _ptr(V), _ptr(O), _stream(stream)))


def hp_attn_group(plans, Qs, Ks, Vs, Os, stream=None):
    """ao_hp_attn_group: one launch for co-located ranks (loopback)."""
    _require_bf16_cuda(*Qs, *Ks, *Vs, *Os)
    for i, p in enumerate(plans):
        _attn_expect(p, Qs[i], Ks[i], Vs[i], Os[i])
    check(lib().ao_hp_attn_group(len(plans), _plans(plans), _arr(Qs), _arr(Ks), _arr(Vs), _arr(Os),
                                 _stream(stream)))


def _arr(ts):
    return (ctypes.c_void_p * len(ts))(*[0 if t is None else int(t.data_ptr()) for t in ts])


def _plans(plans):
    return (ctypes.c_void_p * len(plans))(*[p.handle.value for p in plans])


def ag_gemm_group(plans, A_shards, Bs, Cs, A_gathered_outs=None, stream=None):
    """ao_ag_gemm_group: one fused launch for co-located ranks (loopback)."""
    _require_bf16_cuda(*A_shards, *Bs, *Cs)
    n = len(plans)
    gouts = A_gathered_outs if A_gathered_outs is not None else [None] * n
    for i, p in enumerate(plans):
        W, M, N, K = _op_shapes(p)
        _expect(p, A_shard=(A_shards[i], (M // W, K)), B=(Bs[i], (N, K)), C=(Cs[i], (M, N)),
                A_gathered_out=(gouts[i], (M, K)))
    check(lib().ao_ag_gemm_group(n, _plans(plans), _arr(A_shards), _arr(Bs), _arr(Cs), _arr(gouts), _stream(stream)))


def gemm_rs_group(plans, As, Bs, C_shards, stream=None):
    _require_bf16_cuda(*As, *Bs, *C_shards)
    for i, p in enumerate(plans):
        W, M, N, K = _op_shapes(p)
        _expect(p, A=(As[i], (M, K)), B=(Bs[i], (N, K)), C_shard=(C_shards[i], (M // W, N)))
    check(lib().ao_gemm_rs_group(len(plans), _plans(plans), _arr(As), _arr(Bs), _arr(C_shards), _stream(stream)))


def gemm_ar_group(plans, As, Bs, Cs, stream=None):
    _require_bf16_cuda(*As, *Bs, *Cs)
    for i, p in enumerate(plans):
        W, M, N, K = _op_shapes(p)
        _expect(p, A=(As[i], (M, K)), B=(Bs[i], (N, K)), C=(Cs[i], (M, N)))
    check(lib().ao_gemm_ar_group(len(plans), _plans(plans), _arr(As), _arr(Bs), _arr(Cs), _stream(stream)))


def gemm(A, B, C=None, tile_n: int = 0, tile_m: int = 0, stream=None):
    """ao_gemm: C = A . B^T through the same tcgen05 mainloop (no communication)."""
    import torch
    if C is None:
        C = torch.empty(A.shape[0], B.shape[0], dtype=torch.bfloat16, device=A.device)
    _require_bf16_cuda(A, B, C)
    if A.shape[1] != B.shape[1] or tuple(C.shape) != (A.shape[0], B.shape[0]) or not (A.device == B.device == C.device):
        raise AOError(1, f"gemm: A {tuple(A.shape)}, B {tuple(B.shape)}, C {tuple(C.shape)} (need A [M,K], B [N,K], "
                         "C [M,N] on one device)")
    check(lib().ao_gemm(A.device.index, _ptr(A), _ptr(B), _ptr(C), A.shape[0], B.shape[0], A.shape[1], tile_m,
                        tile_n, _stream(stream)))
    return C


def gemm_batched(As, Bs, Cs, tile_m: int = 0, tile_n: int = 0, group_m: int = 0, n_cta: int = 0, stream=None):
    """ao_gemm_batched: C_i = A_i . B_i^T for n same-shape problems in one persistent launch,
    n_cta CTAs each as in a plan desc (the GEMM-only leg of a loopback group)."""
    _require_bf16_cuda(*As, *Bs, *Cs)
    M, K = As[0].shape
    N = Bs[0].shape[0]
    for a, b, c in zip(As, Bs, Cs):
        if tuple(a.shape) != (M, K) or tuple(b.shape) != (N, K) or tuple(c.shape) != (M, N) or \
                not (a.device == b.device == c.device == As[0].device):
            raise AOError(1, "gemm_batched: every problem must be A [M,K], B [N,K], C [M,N] of one shape on one device")
    check(lib().ao_gemm_batched(As[0].device.index, len(As), _arr(As), _arr(Bs), _arr(Cs), M, N, K, tile_m, tile_n,
                                group_m, n_cta, _stream(stream)))
    return Cs


def transfer_bench(ctx, peer: int, backend: str, src, bytes_: int, chunk_bytes: int, n_ctas: int = 16,
                   n_streams: int = 1, iters: int = 10) -> float:
    """ao_transfer_bench (E4): mean ms to move bytes_ of `src` into rank `peer`'s symmetric
    buffer with one backend (CE: n_streams copy streams; TMA / LDST: n_ctas CTAs of 8 warps)."""
    out = ctypes.c_float(0)
    check(lib().ao_transfer_bench(ctx.handle, int(peer), N.BACKENDS[backend], _ptr(src), int(bytes_), int(chunk_bytes),
                                  int(n_ctas), int(n_streams), int(iters), ctypes.byref(out)))
    return out.value


def device_query(device: int, key: str) -> int:
    """ao_device_query: "sm_count", "cluster2_ctas", "cluster4_ctas"."""
    out = ctypes.c_int64(0)
    check(lib().ao_device_query(int(device), key.encode(), ctypes.byref(out)))
    return out.value


def debug_set(key: str, value: int):
    check(lib().ao_debug_set(key.encode(), int(value)))
