"""Host<->device copy bandwidth on this box (pinned, 64 MB per direction, as the bench's e2e
leg copies per step): H2D alone, D2H alone, and both at once on two streams."""
import torch

n = 64 << 20
h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
up, down = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    for st in (up, down):
        torch.cuda.current_stream().wait_stream(st)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def h2d():
    up.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(up):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    down.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(down):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = timed(fn)
    print(f"{name}: {ms:.3f} ms per 64 MB{' each way' if name == 'both' else ''} = {n / ms / 1e6:.1f} GB/s per direction")
