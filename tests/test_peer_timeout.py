"""A peer-exchange timeout can never let ranks decide differently.

Two processes share one B200 through CUDA IPC (the fused flag exchange of
K1, ma_stepper_check_xchg_async).  Step 0 runs normally.  At step 1 rank 1
arrives 4 s late while MA_PEER_TIMEOUT_S = 1: rank 0 gives up, posts the
poison value into every peer's slots and traps; rank 1, arriving later,
reads the poison and traps too.  Both processes must FAIL (a CUDA launch
failure on their next synchronisation) — neither may update while the
other skips, which is what the round-1 "timeout => local skip" allowed.
A third case: the late rank arrives INSIDE the timeout — both complete the
step with identical decisions.
"""
import os
import socket
import tempfile
import time

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, port, out_dir, late_s, timeout_s):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                      MA_PEER_TIMEOUT_S=str(timeout_s))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    res = "?"
    try:
        import paper_2505_23254_b200 as mab

        torch.cuda.set_device(0)
        n = 1 << 20
        g = torch.zeros(n, dtype=torch.bfloat16, device="cuda")
        p = torch.zeros(n, device="cuda")
        m = torch.zeros(n, device="cuda")
        v = torch.zeros(n, device="cuda")
        w = torch.zeros(n, dtype=torch.bfloat16, device="cuda")
        st = mab.Stepper(mab.AdamHyper(), 65536.0, 2000, "bf16", "bf16")
        x = mab.api.FlagExchange(2, rank, mab.api.torch_all_gather_bytes())
        groups = [(p, m, v, g, w)]
        st.check(g, xchg=x)
        st.apply(groups)
        st.finish()
        torch.cuda.synchronize()
        dist.barrier()
        if rank == 1:
            time.sleep(late_s)
        try:
            st.check(g, xchg=x)
            st.apply(groups)
            st.finish()
            torch.cuda.synchronize()
            res = f"done updates={st.state()['updates']}"
        except Exception as e:  # the trap surfaces as a CUDA error
            res = f"failed {type(e).__name__}: {str(e)[:200]}"
    finally:
        with open(os.path.join(out_dir, f"rank{rank}"), "w") as f:
            f.write(res)
        try:
            dist.destroy_process_group()
        except Exception:
            pass


def _run(late_s, timeout_s):
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(free_port(), d, late_s, timeout_s), nprocs=2, join=True)
        return [open(os.path.join(d, f"rank{r}")).read() for r in range(2)]


def test_late_peer_past_timeout_stops_every_rank():
    t0 = time.time()
    out = _run(late_s=4.0, timeout_s=1.0)
    assert all(r.startswith("failed") for r in out), out
    assert not any("done" in r for r in out)
    assert time.time() - t0 < 120


def test_late_peer_inside_timeout_completes_identically():
    out = _run(late_s=1.0, timeout_s=30.0)
    assert out == ["done updates=2", "done updates=2"], out
