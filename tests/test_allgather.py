"""K2 fused with the weight all-gather (ma_stepper_apply_allgather_async):
the optimizer step of ZeRO data parallelism is followed by an all-gather of
the updated working weights; here K2 itself stores every rank's updated
partition into every peer's full-length weight buffer over peer memory
(CUDA IPC mappings), between an entry and an exit barrier.

2 and 4 processes on one B200 (the IPC mappings are same-device there; on an
NVSwitch box they are NVLink peers): after every step with configs[2]'s
seeded faults, EVERY rank's full weight buffer must equal the single-process
oracle's working weights over the whole partition, bit for bit.
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch

from oracle import oracle as ora
from paper_2505_23254_b200.shard import FaultPlan, shard_range

N_TOTAL, SUBGROUP, STEPS, SEED = 600_011, 50_000, 6, 1
HYP = dict(lr=1e-3, weight_decay=0.01)
pytestmark = pytest.mark.gpu


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist

    import paper_2505_23254_b200 as mab

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        W = torch.empty(N_TOTAL, dtype=torch.bfloat16, device=dev)   # full weights, shared
        mab.gen_seeded_weights(None, W, n=N_TOTAL, seed=SEED)
        base, n = shard_range(N_TOTAL, world, rank, SUBGROUP)
        p = torch.empty(n, dtype=torch.float32, device=dev)
        m = torch.zeros(n, dtype=torch.float32, device=dev)
        v = torch.zeros(n, dtype=torch.float32, device=dev)
        g = torch.empty(n, dtype=torch.bfloat16, device=dev)
        w = W[base:base + n]
        mab.gen_seeded_weights(p, w, base=base, seed=SEED)
        ag = mab.api.GradReduceScatter(world, rank, W, mab.api.torch_all_gather_bytes())
        st = mab.Stepper(mab.AdamHyper(**HYP), 65536.0, 2000, "bf16", "bf16", device=dev)
        groups = [(p[o:o + SUBGROUP], m[o:o + SUBGROUP], v[o:o + SUBGROUP], g[o:o + SUBGROUP],
                   w[o:o + SUBGROUP]) for o in range(0, n, SUBGROUP)]
        plan = FaultPlan(N_TOTAL, SUBGROUP, seed=7)
        for s in range(STEPS):
            mab.gen_pseudo_grads(g, w, step=s, base=base, seed=SEED, d_scale=st.scale_t)
            for f in plan.local(s, base, n):
                mab.plant_bits(g, f.index - base, f.bits)
            st.check(g)
            dist.all_reduce(st.flag, op=dist.ReduceOp.MAX)
            st.apply_allgather(groups, ag)
            st.finish()
        torch.cuda.synchronize()
        assert not ag.timed_out()
        of, sc = st.history()
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"),
                 W=W.view(torch.int16).cpu().numpy().view(np.uint16),
                 p=p.cpu().numpy(), overflow=of.astype(np.uint8), scale=sc, base=base, n=n)
        ag.close()
        st.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_update_fused_with_weight_allgather(world):
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    import torch.multiprocessing as mp

    plan = FaultPlan(N_TOTAL, SUBGROUP, seed=7)
    faults = [(f.step, f.index, f.bits) for s in range(STEPS) for f in plan.at(s)]
    want = ora.train(N_TOTAL, STEPS, SEED, g_kind="bf16", w_kind="bf16", hyp=ora.hyper(**HYP),
                     faults=faults)
    expected = [plan.expected_skip(s) for s in range(STEPS)]
    assert any(expected) and not all(expected)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, free_port(), d), nprocs=world, join=True)
        for r in range(world):
            res = np.load(os.path.join(d, f"rank{r}.npz"))
            assert res["overflow"].astype(bool).tolist() == expected, r
            assert res["scale"].tolist() == want["scale_after"].tolist(), r
            # every rank holds every partition's updated weights
            assert np.array_equal(res["W"], want["w"]), r
            b, n = int(res["base"]), int(res["n"])
            assert np.array_equal(res["p"].view(np.uint32), want["p"][b:b + n].view(np.uint32))


def test_allgather_rejects_foreign_weights():
    """groups' working weights must be views of the shared buffer."""
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    import paper_2505_23254_b200 as mab

    W = torch.zeros(4096, dtype=torch.bfloat16, device="cuda")
    ag = mab.api.GradReduceScatter(1, 0, W, lambda b: [b])
    st = mab.Stepper(mab.AdamHyper(), 65536.0, 2000, "bf16", "bf16")
    p, m, v = (torch.zeros(1024, device="cuda") for _ in range(3))
    g = torch.zeros(1024, dtype=torch.bfloat16, device="cuda")
    other = torch.zeros(1024, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(mab.MemAscendError) as ei:
        st.apply_allgather([(p, m, v, g, other)], ag)
    assert ei.value.code == "invalid-argument"
    st.apply_allgather([(p, m, v, g, W[1024:2048])], ag)   # world 1: local store only
    st.finish()
    torch.cuda.synchronize()
    ag.close()
    st.close()
