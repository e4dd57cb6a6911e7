"""E4: transfer-backend bandwidth vs message size and #SMs / #streams,
measured through ao_transfer_bench -- the fused kernel's own TMA / LDST communication-warp
code and copy-engine memcpys (Fig.2c,d; Tab.2).

  python scripts/e4_microbench.py OUT.jsonl                  # loopback: into another rank's
                                                             # symmetric buffer in this process
  torchrun --nproc-per-node 2 scripts/e4_microbench.py OUT   # rank 0 -> rank 1 across processes
                                                             # (cudaIpc mapping; same GPU here)
One JSON line per point: mode, backend, ctas (TMA/LDST) or streams (CE), bytes, ms, GB/s
(bytes moved per second, one direction)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_20595_b200 as ao

SIZES = [4 << 10, 16 << 10, 64 << 10, 256 << 10, 1 << 20, 4 << 20, 16 << 20, 64 << 20, 256 << 20]
CTAS = [1, 2, 4, 8, 16, 32, 74, 148]


def sweep(ctx, peer, mode, out):
    src = torch.randint(-100, 100, (max(SIZES) // 2,), dtype=torch.int16, device="cuda").view(torch.bfloat16)
    for m in SIZES:
        iters = max(3, min(100, (256 << 20) // m))
        for streams in (1, 7):
            chunk = max(16, (m + streams - 1) // streams // 16 * 16) if streams > 1 else m
            ms = ao.transfer_bench(ctx, peer, "ce", src, m, chunk, n_streams=streams, iters=iters)
            rec = dict(mode=mode, backend="ce", streams=streams, bytes=m, ms=ms, GBps=m / (ms * 1e-3) / 1e9)
            out.write(json.dumps(rec) + "\n")
        for b in ("tma", "ldst"):
            for n in CTAS:
                warps = 8 * n
                chunk = max(16, -(-m // warps) // 16 * 16)
                ms = ao.transfer_bench(ctx, peer, b, src, m, chunk, n_ctas=n, iters=iters)
                rec = dict(mode=mode, backend=b, ctas=n, bytes=m, ms=ms, GBps=m / (ms * 1e-3) / 1e9)
                out.write(json.dumps(rec) + "\n")
        out.flush()
        print(mode, m, flush=True)


def main():
    path = sys.argv[1] if len(sys.argv) > 1 else "profiles/r02_e4.jsonl"
    ws = 2 * (max(SIZES) + (1 << 20))
    if "RANK" in os.environ:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        torch.cuda.set_device(0)
        ctx = ao.dist_world(0, ws)
        if dist.get_rank() == 0:
            with open(path, "a") as f:
                sweep(ctx, 1, "cross_process", f)
        dist.barrier()
        ctx.close()
        dist.destroy_process_group()
    else:
        ctxs = ao.loopback_world(0, 2, ws)
        with open(path, "a") as f:
            sweep(ctxs[0], 1, "loopback", f)
        for c in ctxs:
            c.close()


if __name__ == "__main__":
    main()
