"""The whole data-parallel ZeRO optimizer step over peer memory, no
collective call: every rank holds FULL-LENGTH gradients (a backward over its
own micro-batch) and the full working weights; per step

  K4  reduce-scatter of the gradients with the overflow check in its epilogue
      (peers read through CUDA IPC; the skip decision OR-ed across ranks by
      K4's last CTA)                         ma_stepper_reduce_scatter_async
  K2  unscale + AdamW + cast of this rank's partition, the new working
      weights stored into every rank's weight buffer      ma_stepper_apply_allgather_async
      (skipped on every rank when any rank overflowed)
  LossScaler                                              ma_stepper_finish_async

Checked against an oracle composition of the reference's pieces — rank-
ordered reduction (ora_reduce_check), adam_step_fp32 + cast, LossScaler —
bit for bit, with 2 and 4 processes sharing one B200, NaN/inf planted in
some steps on some ranks.
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch

from oracle import oracle as ora
from paper_2505_23254_b200.shard import shard_range

N_TOTAL, SUBGROUP, SEED = 300_007, 40_000, 5
STEPS = int(os.environ.get("MA_ZERO_SOAK_STEPS", "6"))  # soak runs: many steps
HYP = dict(lr=1e-3, weight_decay=0.01)
POISON = {(2, 1): 0x7FC0, (4, 0): 0xFF80}  # (step, rank) -> bf16 NaN / -inf
POISON.update({(s, s % 3): 0x7F80 for s in range(11, 100_000, 37)})  # soak: more skips
pytestmark = pytest.mark.gpu


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def rank_grads(rank, step, scale):
    """This rank's full-length scaled bf16 gradients (seeded)."""
    rng = np.random.default_rng(1000 * step + rank)
    g = ora.cast_from_f32((rng.standard_normal(N_TOTAL) * 0.01 * scale).astype(np.float32),
                          "bf16")
    if (step, rank) in POISON:
        g[(7919 * (rank + 1) + step) % N_TOTAL] = POISON[(step, rank)]
    return g


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist

    import paper_2505_23254_b200 as mab

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        run_rank(rank, world, out_dir, mab.api.torch_all_gather_bytes())
    finally:
        dist.destroy_process_group()


def run_rank(rank, world, out_dir, gather):
    """One rank's steps (also called in-process with world 1 and an identity
    gather, so the whole peer-memory protocol runs under compute-sanitizer in
    a single process)."""
    import paper_2505_23254_b200 as mab

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    G = torch.empty(N_TOTAL, dtype=torch.bfloat16, device=dev)   # full-length grads
    W = torch.empty(N_TOTAL, dtype=torch.bfloat16, device=dev)   # full working weights
    P0 = torch.empty(N_TOTAL, dtype=torch.float32, device=dev)
    mab.gen_seeded_weights(P0, W, seed=SEED)
    base, n = shard_range(N_TOTAL, world, rank, SUBGROUP)
    p = P0[base:base + n].clone()
    m = torch.zeros(n, dtype=torch.float32, device=dev)
    v = torch.zeros(n, dtype=torch.float32, device=dev)
    gp = torch.empty(n, dtype=torch.bfloat16, device=dev)        # reduced partition grads
    rs = mab.api.GradReduceScatter(world, rank, G, gather)
    ag = mab.api.GradReduceScatter(world, rank, W, gather)
    st = mab.Stepper(mab.AdamHyper(**HYP), 65536.0, 2000, "bf16", "bf16", device=dev)
    w = W[base:base + n]
    groups = [(p[o:o + SUBGROUP], m[o:o + SUBGROUP], v[o:o + SUBGROUP], gp[o:o + SUBGROUP],
               w[o:o + SUBGROUP]) for o in range(0, n, SUBGROUP)]
    for s in range(STEPS):
        scale = st.state()["scale"]
        G.copy_(torch.from_numpy(rank_grads(rank, s, scale).view(np.int16)).to(dev)
                .view(torch.bfloat16))
        st.reduce_scatter(rs, base, n, gp, post_scale=1.0 / world)
        st.apply_allgather(groups, ag)
        st.finish()
    torch.cuda.synchronize()
    assert not rs.timed_out() and not ag.timed_out()
    of, sc = st.history()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"),
             W=W.view(torch.int16).cpu().numpy().view(np.uint16), p=p.cpu().numpy(),
             m=m.cpu().numpy(), v=v.cpu().numpy(), overflow=of.astype(np.uint8), scale=sc,
             base=base, n=n)
    rs.close()
    ag.close()
    st.close()


def oracle_run(world):
    p, w = ora.fill_weights(N_TOTAL, seed=SEED, w_kind="bf16")
    m = np.zeros(N_TOTAL, np.float32)
    v = np.zeros(N_TOTAL, np.float32)
    scaler = ora.Scaler(65536.0, 2000, 0)
    h = ora.hyper(**HYP)
    updates, overflow, scales = 0, [], []
    parts = [shard_range(N_TOTAL, world, r, SUBGROUP) for r in range(world)]
    for s in range(STEPS):
        full = [rank_grads(r, s, scaler.scale) for r in range(world)]
        reduced, bad = [], False
        for b, n in parts:
            g, f = ora.reduce_check([x[b:b + n] for x in full], "bf16", 1.0 / world, "bf16")
            reduced.append(g)
            bad |= f
        if bad:
            ora.lib().ora_scaler_on_overflow(ora.C.byref(scaler))
        else:
            updates += 1
            for (b, n), g in zip(parts, reduced):
                for o in range(0, n, SUBGROUP):
                    k = min(SUBGROUP, n - o)
                    sl = slice(b + o, b + o + k)
                    pp, mm, vv = p[sl].copy(), m[sl].copy(), v[sl].copy()
                    w[sl] = ora.adam_step(pp, mm, vv, g[o:o + k], updates, h, scaler.scale,
                                          "bf16", "bf16")
                    p[sl], m[sl], v[sl] = pp, mm, vv
            ora.lib().ora_scaler_on_clean_step(ora.C.byref(scaler))
        overflow.append(bad)
        scales.append(scaler.scale)
    return dict(p=p, m=m, v=v, w=w, overflow=overflow, scale=scales)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_fused_zero_step_over_peer_memory(world):
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    import torch.multiprocessing as mp

    want = oracle_run(world)
    assert any(want["overflow"]) and not all(want["overflow"])
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, free_port(), d), nprocs=world, join=True)
        for r in range(world):
            res = np.load(os.path.join(d, f"rank{r}.npz"))
            assert res["overflow"].astype(bool).tolist() == want["overflow"], r
            assert res["scale"].tolist() == want["scale"], r
            assert np.array_equal(res["W"], want["w"]), r       # every partition, every rank
            b, n = int(res["base"]), int(res["n"])
            for k in "pmv":
                assert np.array_equal(res[k].view(np.uint32), want[k][b:b + n].view(np.uint32)), (r, k)


def test_fused_zero_step_single_process():
    """World 1 in this process: the entry barrier, K4 with its exit barrier /
    flag OR and K2's all-gather with both barriers all run (on one rank), so
    compute-sanitizer sees every peer-memory kernel (tools/sanitize.sh)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    want = oracle_run(1)
    assert any(want["overflow"]) and not all(want["overflow"])
    with tempfile.TemporaryDirectory() as d:
        run_rank(0, 1, d, lambda b: [b])
        res = np.load(os.path.join(d, "rank0.npz"))
        assert res["overflow"].astype(bool).tolist() == want["overflow"]
        assert res["scale"].tolist() == want["scale"]
        assert np.array_equal(res["W"], want["w"])
        for k in "pmv":
            assert np.array_equal(res[k].view(np.uint32), want[k].view(np.uint32)), k


def test_fused_zero_step_single_process_in_a_graph():
    """The same world-1 ZeRO step captured once as a CUDA graph (entry
    barrier, K4 + exit barrier / flag OR, K2 + all-gather barriers, scaler)
    and replayed every step: the exchange epochs live on the device, so the
    replays equal the eager run and the oracle."""
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    import paper_2505_23254_b200 as mab

    want = oracle_run(1)
    dev = torch.device("cuda", 0)
    G = torch.empty(N_TOTAL, dtype=torch.bfloat16, device=dev)
    W = torch.empty(N_TOTAL, dtype=torch.bfloat16, device=dev)
    p = torch.empty(N_TOTAL, dtype=torch.float32, device=dev)
    mab.gen_seeded_weights(p, W, seed=SEED)
    m = torch.zeros(N_TOTAL, dtype=torch.float32, device=dev)
    v = torch.zeros(N_TOTAL, dtype=torch.float32, device=dev)
    gp = torch.empty(N_TOTAL, dtype=torch.bfloat16, device=dev)
    one = lambda b: [b]  # noqa: E731
    rs = mab.api.GradReduceScatter(1, 0, G, one)
    ag = mab.api.GradReduceScatter(1, 0, W, one)
    st = mab.Stepper(mab.AdamHyper(**HYP), 65536.0, 2000, "bf16", "bf16", device=dev)
    groups = [(p[o:o + SUBGROUP], m[o:o + SUBGROUP], v[o:o + SUBGROUP], gp[o:o + SUBGROUP],
               W[o:o + SUBGROUP]) for o in range(0, N_TOTAL, SUBGROUP)]
    stream = torch.cuda.Stream()
    stream.wait_stream(torch.cuda.current_stream())

    def chain():
        st.reduce_scatter(rs, 0, N_TOTAL, gp, post_scale=1.0, stream=stream)
        st.apply_allgather(groups, ag, stream=stream)
        st.finish(stream=stream)

    graph = st.capture(chain, stream, reserve_steps=64)
    for s in range(STEPS):
        stream.synchronize()
        scale = st.state()["scale"]
        G.copy_(torch.from_numpy(rank_grads(0, s, scale).view(np.int16)).to(dev)
                .view(torch.bfloat16))
        torch.cuda.current_stream().synchronize()
        graph.launch(stream)
    stream.synchronize()
    of, sc = st.history()
    assert of.astype(bool).tolist() == want["overflow"]
    assert sc.tolist() == want["scale"]
    assert np.array_equal(W.view(torch.int16).cpu().numpy().view(np.uint16), want["w"])
    for k, t in zip("pmv", (p, m, v)):
        assert np.array_equal(t.cpu().numpy().view(np.uint32), want[k].view(np.uint32)), k
    graph.close()
    rs.close()
    ag.close()
    st.close()
