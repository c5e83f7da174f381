"""Speculative update during the host-gradient transfer
(ma_stepper_check_host_spec_async / ma_stepper_apply_spec_async): every
sub-group whose gradients have landed is updated while the flag is still
clear, after a backup of its state; the step's final decision keeps or
restores it.  The result must equal the reference composition
(simulator.cpp:427-492, the oracle) bit for bit — faults in the first chunk
(nothing speculated), in the last chunk (everything speculated is rolled
back), in the middle — with the backup holding all, some or none of the
sub-groups, aligned and misaligned views."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a B200", allow_module_level=True)

import paper_2505_23254_b200 as mab  # noqa: E402
from oracle import oracle as ora  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


def bits(t):
    torch.cuda.synchronize()
    if t.element_size() == 4:
        return t.view(torch.int32).cpu().numpy().view(np.uint32)
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def run(n, cuts, steps, faults, seed, backup_groups, off, chunk, w_kind="bf16"):
    rs_bounds = list(zip([0] + cuts, cuts + [n]))
    p = torch.empty(n + off, dtype=torch.float32, device=DEV)[off:]
    m = torch.zeros(n + off, dtype=torch.float32, device=DEV)[off:]
    v = torch.zeros(n + off, dtype=torch.float32, device=DEV)[off:]
    w = torch.empty(n + off, dtype=torch.bfloat16 if w_kind == "bf16" else torch.float16,
                    device=DEV)[off:]
    g = torch.empty(n, dtype=torch.bfloat16, device=DEV)       # dev_g: the groups tile it
    tmp = torch.empty(n, dtype=torch.bfloat16, device=DEV)     # producer output
    host = torch.empty(n, dtype=torch.bfloat16).pin_memory()  # the step's host gradients
    mab.gen_seeded_weights(p, w, seed=seed)
    st = mab.Stepper(mab.AdamHyper(weight_decay=0.01), 65536.0, 2, "bf16", w_kind)
    groups = mab.Stepper.subgroups([(p[a:b], m[a:b], v[a:b], g[a:b], w[a:b])
                                    for a, b in rs_bounds], "bf16", w_kind)
    al = lambda x: (x + 255) // 256 * 256  # noqa: E731
    need = [3 * al(4 * (b - a)) + al(2 * (b - a)) for a, b in rs_bounds]
    nb = sum(need[:backup_groups])
    backup = torch.empty(max(nb, 1), dtype=torch.uint8, device=DEV) if nb else None
    for s in range(steps):
        mab.gen_pseudo_grads(tmp, w, step=s, seed=seed, d_scale=st.scale_t)
        for fs, idx, b in faults:
            if fs == s:
                mab.plant_bits(tmp, idx, b)
        torch.cuda.synchronize()
        host.copy_(tmp.cpu())
        st.check_from_host_spec(host, g, groups, backup, chunk_elems=chunk)
        st.apply_spec(groups)
        st.finish()
    torch.cuda.synchronize()
    of, sc = st.history()
    out = dict(p=bits(p), m=bits(m), v=bits(v), w=bits(w), of=of.tolist(), sc=sc.tolist())
    st.close()
    return out


N = 301_117
CUTS = [1, 40_000, 40_001, 97_003, 150_000, 222_222, 301_116]  # size-1 groups at both ends


@pytest.mark.parametrize("backup_groups", [8, 3, 0])
@pytest.mark.parametrize("off", [0, 1])
def test_spec_equals_reference(backup_groups, off):
    steps, seed = 7, 5
    faults = [(1, 17, 0x7FC0),          # first chunk: nothing speculated this step
              (3, N - 1, 0xFF80),       # last element: every speculated group rolled back
              (5, 160_000, 0x7F80)]     # middle: the groups before it stay speculative
    got = run(N, CUTS, steps, faults, seed, backup_groups, off, chunk=30_000)
    ref = ora.train(N, steps, seed, g_kind="bf16", w_kind="bf16",
                    hyp=ora.hyper(weight_decay=0.01), growth=2, faults=faults)
    assert got["of"] == ref["overflow"].astype(bool).tolist()
    assert got["sc"] == ref["scale_after"].tolist()
    for k in "pmv":
        assert np.array_equal(got[k], ref[k].view(np.uint32)), k
    assert np.array_equal(got["w"], ref["w"])


def test_spec_fp16_weights_and_one_chunk():
    steps, seed = 4, 9
    faults = [(2, 250_000, 0x7F81)]
    got = run(N, CUTS, steps, faults, seed, 8, 0, chunk=1 << 30, w_kind="f16")
    ref = ora.train(N, steps, seed, g_kind="bf16", w_kind="f16",
                    hyp=ora.hyper(weight_decay=0.01), growth=2, faults=faults)
    assert got["of"] == ref["overflow"].astype(bool).tolist()
    for k in "pmv":
        assert np.array_equal(got[k], ref[k].view(np.uint32)), k
    assert np.array_equal(got["w"], ref["w"])


@pytest.mark.parametrize("backup_groups", [8, 2])
def test_spec_pure_bf16_equals_reference(backup_groups):
    """The pure-bf16 form (K3 on bf16 weights / m / v) against the
    reference's pure-bf16 composition."""
    n, steps, seed = N, 6, 11
    faults = [(1, 40_000, 0x7FC0), (3, N - 1, 0x7F80)]
    bounds = list(zip([0] + CUTS, CUTS + [n]))
    w = torch.empty(n, dtype=torch.bfloat16, device=DEV)
    m = torch.zeros(n, dtype=torch.bfloat16, device=DEV)
    v = torch.zeros(n, dtype=torch.bfloat16, device=DEV)
    g = torch.empty(n, dtype=torch.bfloat16, device=DEV)
    tmp = torch.empty(n, dtype=torch.bfloat16, device=DEV)
    host = torch.empty(n, dtype=torch.bfloat16).pin_memory()
    mab.gen_seeded_weights(None, w, seed=seed)
    st = mab.Stepper(mab.AdamHyper(weight_decay=0.01), 65536.0, 2, "bf16", "bf16")
    groups = st.subgroups_bf16([(w[a:b], m[a:b], v[a:b], g[a:b]) for a, b in bounds])
    al = lambda x: (x + 255) // 256 * 256  # noqa: E731
    nb = sum(3 * al(2 * (b - a)) for a, b in bounds[:backup_groups])
    backup = torch.empty(nb, dtype=torch.uint8, device=DEV)
    for s in range(steps):
        mab.gen_pseudo_grads(tmp, w, step=s, seed=seed, d_scale=st.scale_t)
        for fs, idx, b in faults:
            if fs == s:
                mab.plant_bits(tmp, idx, b)
        torch.cuda.synchronize()
        host.copy_(tmp.cpu())
        st.check_from_host_spec_bf16(host, g, groups, backup, chunk_elems=30_000)
        st.apply_spec_bf16(groups)
        st.finish()
    torch.cuda.synchronize()
    of, sc = st.history()
    ref = ora.train(n, steps, seed, mixed=False, g_kind="bf16", w_kind="bf16",
                    hyp=ora.hyper(weight_decay=0.01), growth=2, faults=faults)
    assert of.tolist() == ref["overflow"].astype(bool).tolist()
    assert sc.tolist() == ref["scale_after"].tolist()
    assert np.array_equal(bits(w), ref["w"])
    assert np.array_equal(bits(m), ref["m16"])
    assert np.array_equal(bits(v), ref["v16"])
    st.close()


def test_spec_lifecycle():
    n = 4096
    p, m, v = (torch.zeros(n, device=DEV) for _ in range(3))
    w = torch.zeros(n, dtype=torch.bfloat16, device=DEV)
    g = torch.zeros(n, dtype=torch.bfloat16, device=DEV)
    host = torch.zeros(n, dtype=torch.bfloat16).pin_memory()
    st = mab.Stepper(mab.AdamHyper(), 1024.0, 2000, "bf16", "bf16")
    groups = mab.Stepper.subgroups([(p, m, v, g, w)], "bf16", "bf16")
    backup = torch.empty(1 << 20, dtype=torch.uint8, device=DEV)
    st.check_from_host_spec(host, g, groups, backup)
    with pytest.raises(mab.MemAscendError):      # the pending step must be completed first
        st.check_from_host_spec(host, g, groups, backup)
    other = mab.Stepper.subgroups([(p.clone(), m, v, g, w)], "bf16", "bf16")
    with pytest.raises(mab.MemAscendError):      # not the speculated sub-groups
        st.apply_spec(other)
    st.apply_spec(groups)
    st.finish()
    torch.cuda.synchronize()
    assert st.state()["updates"] == 1
    st.close()
