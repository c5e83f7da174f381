"""K4: gradient reduce-scatter with the overflow check in its epilogue
("the NCCL reduce-scatter epilogue").

Parity target: oracle ``ora_reduce_check`` (rank-ordered fp32 sum, optional
post-scale, canonical NaN, the reference's bit test of overflow.hpp:46-51 on
the stored values).  Single process: explicit source pointers
(ma_stepper_reduce_check_async) over every dtype pair, misaligned views,
planted non-finite values and sums that overflow only after the reduction.
Two processes on one B200: the IPC form (ma_rs_* +
ma_stepper_reduce_scatter_async) — peers read over peer mappings, entry and
exit barriers, the skip decision identical on both ranks without any
collective call.
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch

from oracle import oracle as ora

DEV = "cuda:0"
KINDS = ["f32", "bf16", "f16"]
TORCH = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}


def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a B200")


def rand_bits(rng, n, kind, scale=1.0):
    x = (rng.standard_normal(n) * scale).astype(np.float32)
    return x if kind == "f32" else ora.cast_from_f32(x, kind)


def to_dev(bits, kind, offset=0):
    """Device tensor holding `bits`, starting `offset` elements into its
    allocation (to exercise unaligned partitions)."""
    if kind == "f32":
        t = torch.from_numpy(np.ascontiguousarray(bits).view(np.int32))
    else:
        t = torch.from_numpy(np.ascontiguousarray(bits).view(np.int16))
    buf = torch.zeros(bits.size + offset, dtype=t.dtype, device=DEV)
    buf[offset:] = t.to(DEV)
    return buf[offset:].view(TORCH[kind])


def host_bits(t):
    if t.dtype == torch.float32:
        return t.view(torch.int32).cpu().numpy().view(np.float32)
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def same_bits(a, b):
    if a.dtype == np.float32:
        return np.array_equal(a.view(np.uint32), b.view(np.uint32))
    return np.array_equal(a, b)


def big_finite(kind):
    """Two of these sum past the fp32 / destination range."""
    return {"f32": np.float32(3.0e38), "bf16": np.uint16(0x7F70), "f16": np.uint16(0x7BFF)}[kind]


CASES = [
    # (nsrc, n, src offsets, dst offset, post_scale, plant)
    (1, 1, (0,), 0, 1.0, None),
    (2, 7, (0, 0), 0, 1.0, None),
    (2, 4096 * 3 + 5, (0, 0), 0, 0.5, None),
    (3, 100_003, (1, 1, 1), 1, 1.0, None),
    (3, 100_003, (1, 2, 3), 0, 1.0, None),           # no common alignment: scalar path
    (8, 1 << 20, (0,) * 8, 0, 0.125, None),
    (8, (1 << 20) + 3, (5,) * 8, 5, 0.3, None),
    (2, 65_537, (0, 0), 0, 1.0, ("inf", 1, 40_000)),
    (4, 65_537, (0,) * 4, 0, 0.25, ("nan", 3, 65_536)),
    (2, 65_537, (3, 3), 3, 1.0, ("nan", 0, 0)),
    (2, 65_537, (0, 0), 0, 1.0, ("sum_overflow", 0, 12_345)),
    (2, 65_537, (0, 0), 0, 1.0, ("max_finite", 0, 777)),
]


@pytest.mark.gpu
@pytest.mark.parametrize("sk", KINDS)
@pytest.mark.parametrize("dk", KINDS)
def test_reduce_check_vs_oracle(sk, dk):
    need_gpu()
    import paper_2505_23254_b200 as mab

    rng = np.random.default_rng(3 * KINDS.index(sk) + KINDS.index(dk))
    for nsrc, n, offs, doff, post, plant in CASES:
        srcs = [rand_bits(rng, n, sk) for _ in range(nsrc)]
        if plant:
            what, r, i = plant
            if what == "inf":
                srcs[r][i] = np.float32(np.inf) if sk == "f32" else (0x7F80 if sk == "bf16" else 0x7C00)
            elif what == "nan":
                srcs[r][i] = np.float32(np.nan) if sk == "f32" else (0x7FC1 if sk == "bf16" else 0x7E01)
            elif what == "sum_overflow":
                for s in srcs:
                    s[i] = big_finite(sk)
            elif what == "max_finite":
                srcs[r][i] = np.float32(3.0e38) if sk == "f32" else (0x7F7F if sk == "bf16" else 0x7BFF)
        want, want_flag = ora.reduce_check(srcs, sk, post, dk)
        st = mab.Stepper(mab.AdamHyper(), 65536.0, 2000, dk, "bf16")
        d_srcs = [to_dev(s, sk, o) for s, o in zip(srcs, offs)]
        dst = to_dev(np.zeros(n, np.float32 if dk == "f32" else np.uint16), dk, doff)
        st.reduce_check(d_srcs, dst, post_scale=post)
        torch.cuda.synchronize()
        got = host_bits(dst)
        case = (sk, dk, nsrc, n, offs, doff, post, plant)
        assert same_bits(got, want), case
        assert bool(st.flag.item()) == want_flag, case


# ------------------------------------------------------------ two processes
N_TOTAL, WORLD, STEPS = 1_000_003, 2, 4
SPLIT = 500_001  # rank 1's partition starts at an odd element (scalar head)


def partition(rank):
    return (0, SPLIT) if rank == 0 else (SPLIT, N_TOTAL - SPLIT)


def step_grads(rank, step):
    g = rand_bits(np.random.default_rng(1000 * rank + step), N_TOTAL, "bf16", scale=4.0)
    if step == 2 and rank == 1:
        g[7] = 0x7F80  # +inf in rank 0's partition: both ranks must skip
    if step == 3 and rank == 0:
        g[N_TOTAL - 1] = 0xFFC0  # NaN in rank 1's partition
    return g


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rs_worker(rank, port, out_dir):
    import torch.distributed as dist

    import paper_2505_23254_b200 as mab

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        torch.cuda.set_device(0)
        grads = torch.empty(N_TOTAL, dtype=torch.bfloat16, device=DEV)
        rs = mab.api.GradReduceScatter(WORLD, rank, grads, mab.api.torch_all_gather_bytes())
        st = mab.Stepper(mab.AdamHyper(), 65536.0, 2000, "bf16", "bf16")
        base, n = partition(rank)
        out = {}
        for s in range(STEPS):
            # the next backward overwrites the buffer in stream order after
            # the previous step's exit barrier
            grads.copy_(torch.from_numpy(step_grads(rank, s).view(np.int16)).to(DEV)
                        .view(torch.bfloat16))
            dst = torch.empty(n, dtype=torch.bfloat16, device=DEV)
            st.reduce_scatter(rs, base, n, dst, post_scale=0.5)
            out[f"flag{s}"] = np.array([st.flag.item()])
            st.finish()
            out[f"dst{s}"] = host_bits(dst)
        torch.cuda.synchronize()
        assert not rs.timed_out()
        of, _ = st.history()
        out["overflow"] = of.astype(np.uint8)
        rs.close()
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **out)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_two_ranks_reduce_scatter_over_peer_memory():
    need_gpu()
    import torch.multiprocessing as mp

    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_rs_worker, args=(free_port(), d), nprocs=WORLD, join=True)
        res = [np.load(os.path.join(d, f"rank{r}.npz")) for r in range(WORLD)]
    for s in range(STEPS):
        full = [step_grads(r, s) for r in range(WORLD)]
        want_any = False
        for r in range(WORLD):
            base, n = partition(r)
            want, flag = ora.reduce_check([g[base:base + n] for g in full], "bf16", 0.5, "bf16")
            want_any |= flag
            assert same_bits(res[r][f"dst{s}"], want), (s, r)
        for r in range(WORLD):
            assert bool(res[r][f"flag{s}"][0]) == want_any, (s, r)
    for r in range(WORLD):
        assert res[r]["overflow"].tolist() == [0, 0, 1, 1]
