"""Multi-process (world_size 2, gloo, CPU) tests of the N > 1 host logic.

Each process plays one rank: it builds its plans through the C ABI (host-only calls),
exchanges hashes / canonical exports over torch.distributed, and checks the cross-rank
contract the fused kernels rely on (a schedule is the per-rank op lists; a
P2P op is recorded on exactly one side):
  * every rank built a plan with the same hash (collective semantics of the C ABI);
  * AG: every remote chunk arriving at rank r is delivered by exactly one op of its
    source's list, and r's arrival position is that op's index + 1;
  * RS: every non-own chunk of owner o is pushed to o by exactly one op of each other
    rank, and o waits for exactly W-1 contributions per own chunk.
Also runs bench.py's reference arm under torchrun (rank 0 prints one line, rank 1 exits).
"""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, descs, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2601_20595_b200.api as ao
        results = []
        for d in descs:
            p = ao.Plan(None, dict(d, rank=rank), sm_count=148)
            mine = (p.hash(), p.export_json())
            allv = [None] * world
            dist.all_gather_object(allv, mine)
            results.append(allv)
        if rank == 0:
            q.put(results)
    finally:
        dist.destroy_process_group()


def _run(descs, world=2):
    from paper_2601_20595_b200 import build
    build.build(verbose=False)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, descs, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    return res


DESCS = [
    dict(op="ag_gemm", world_size=2, M=1024, N=768, K=256, chunk_rows=128, backend="ce"),
    dict(op="ag_gemm", world_size=2, M=2048, N=512, K=128, chunk_rows=256, backend="tma", n_slices=2,
         chunk_order="chunk_major", intra="grouped", group_m=2),
    dict(op="gemm_rs", world_size=2, M=1024, N=512, K=256, chunk_rows=128),
    dict(op="gemm_rs", world_size=2, M=2048, N=1024, K=128, chunk_rows=256, chunk_order="chunk_major"),
]


def test_two_ranks_agree_and_schedules_are_consistent():
    res = _run(DESCS)
    for d, allv in zip(DESCS, res):
        hashes = {h for h, _ in allv}
        assert len(hashes) == 1, d
        plans = [json.loads(js) for _, js in allv]
        W = d["world_size"]
        for r in range(W):
            P = plans[r]
            assert P["rank"] == r
            assert P["plans"] == plans[0]["plans"]  # everyone exports the same global schedule
            for g, row0, rows, owner, pos in P["chunks"]:
                if d["op"] == "ag_gemm":
                    if owner == r:
                        assert pos == 0
                        continue
                    ops = [i for i, op in enumerate(P["plans"][owner])
                           if op["peer"] == r and op["src_chunk"] == [row0, rows]]
                    assert len(ops) == 1 and pos == ops[0] + 1
                else:
                    if owner == r:
                        assert P["contrib"][g] == W - 1
                    else:
                        assert P["contrib"][g] == 0
                    for s in range(W):
                        ops = [op for op in P["plans"][s] if op["src_chunk"] == [row0, rows]]
                        assert len(ops) == 1 and ops[0]["peer"] == owner and ops[0]["accumulate"] == 1


def test_bench_reference_arm_under_torchrun():
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl",
           "reference", "--steps", "1", "--warmup", "0", "--tokens", "512"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_two_ranks_agree_on_a2a_plans():
    """A2A-GEMM (NEXT-3): the static part of the schedule agrees across ranks (the ops are
    collective: same hash), and each rank's export names itself."""
    descs = [dict(op="a2a_gemm", world_size=2, M=512, N=512, K=256, topk=2, chunk_rows=64, backend="ldst"),
             dict(op="a2a_gemm", world_size=2, M=1024, N=768, K=128, topk=1, chunk_rows=128, backend="ldst",
                  intra="grouped", group_m=4, tile_m=128, tile_n=256)]
    res = _run(descs)
    for d, allv in zip(descs, res):
        assert len({h for h, _ in allv}) == 1, d
        for r, (_, js) in enumerate(allv):
            P = json.loads(js)
            assert P["rank"] == r and P["dynamic"] == 1 and P["topk"] == d["topk"]
            assert P["max_chunks_per_source"] == -(-d["M"] // d["chunk_rows"])
