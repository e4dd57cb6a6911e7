"""ONE RANK PER PROCESS on the one GPU of the test box: the production path (dist_world ->
cudaIpcOpenMemHandle -> per-rank ao_* calls with n_group = 1) that the loopback tests
never execute.  Each case runs tests/mp_worker.py under torch.distributed.run with W
processes; every process checks its own results against the fp64 oracle (provenance
bit-exact over back-to-back epochs) and a deliberate cross-process plan mismatch must
surface as AO_ERR_PEER.  Processes of one GPU time-slice (or share it under MPS)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _launch(W, cases, timeout=600, env_extra=None):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={W}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(ROOT, "tests", "mp_worker.py"),
           cases]
    env = dict(os.environ, OMP_NUM_THREADS="2", **(env_extra or {}))
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT, env=env)
    except subprocess.TimeoutExpired as e:
        out = (e.stdout or b"").decode(errors="replace") if isinstance(e.stdout, bytes) else (e.stdout or "")
        raise AssertionError(f"multi-process run timed out after {timeout} s; progress:\n{out[-3000:]}") from None
    recs = []
    dec = json.JSONDecoder()
    for line in r.stdout.splitlines():  # the processes' lines may interleave
        i = line.find("{")
        while i >= 0:
            try:
                rec, end = dec.raw_decode(line, i)
            except json.JSONDecodeError:
                break
            if isinstance(rec, dict) and "ok" in rec:
                recs.append(rec)
            i = line.find("{", end)
    return r, recs


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2601_20595_b200 import build
    build.build(verbose=False)


@pytest.fixture(scope="module")
def mps(tmp_path_factory):
    """A private MPS daemon (its own pipe directory, so only the workers launched with
    that environment connect): the W processes' persistent kernels then run concurrently
    instead of time-slicing.  None when MPS is not available on the box."""
    import shutil
    import time
    ctl = shutil.which("nvidia-cuda-mps-control")
    if ctl is None:
        yield None
        return
    d = tmp_path_factory.mktemp("mps")
    env = dict(CUDA_MPS_PIPE_DIRECTORY=str(d / "pipe"), CUDA_MPS_LOG_DIRECTORY=str(d / "log"))
    for v in env.values():
        os.makedirs(v, exist_ok=True)
    r = subprocess.run([ctl, "-d"], env=dict(os.environ, **env), capture_output=True, text=True)
    if r.returncode != 0:
        yield None
        return
    time.sleep(0.5)
    yield env
    subprocess.run([ctl], input="quit\n", env=dict(os.environ, **env), capture_output=True, text=True)


@pytest.mark.parametrize("W,cases,use_mps", [(2, "ag,rs,ar,a2a,attn,hp,sk,rs_bf16,mismatch", False),
                                             (4, "ag_ce_push,ag_tma_push,ag_ldst_pull,rs,ar,a2a,attn,hp,sk,rs_bf16,mismatch",
                                              True)])
def test_one_rank_per_process(W, cases, use_mps, mps):
    """W=2 time-sliced (no MPS: the ranks' kernels alternate on the GPU), W=4 concurrent
    under MPS when the box has it."""
    r, recs = _launch(W, cases, env_extra=mps if use_mps else None)
    bad = [x for x in recs if not x["ok"]]
    assert r.returncode == 0 and not bad, (r.returncode, bad[:4], r.stderr[-3000:])
    names = {x["case"] for x in recs}
    for c in cases.split(","):
        if c in ("ag", "rs", "attn", "hp"):
            assert any(n.startswith(c) for n in names), c
        else:
            assert c in names, c
    assert all(sum(1 for x in recs if x["case"] == n) == W for n in names)
