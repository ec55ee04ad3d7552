"""The multi-rank product path (N > 1: fused NVLink dispatch with arrival flags, arrival-
ordered and scattering GEMMs, device barriers, combine-backward stores into the owners'
buffers, the NCCL-exchange variant, owner-set expert-gradient sums) run forward AND
backward for N virtual ranks on ONE B200 (paper_2407_04656_b200/loopback.py), compared
with the torch-CPU fp32 oracle on the gathered global batch.

Reference contract: the padding-free all-to-all (flexep dispatch.py:247-283) and the
replica-group expert-gradient all-reduce; failure semantics PAPER.md:297.
Tolerances as tests/test_layer_gpu.py: per tensor ||got - ref|| <= 3e-2 ||ref|| and
max|got - ref| <= 6e-2 max|ref| (router grads 5e-2 / 1e-1).
"""

import math

import pytest
import torch

from oracle import moe_ref

pytestmark = pytest.mark.gpu


def _rel(got, ref, l2=3e-2, linf=6e-2, name=""):
    got, ref = got.detach().float().cpu(), ref.detach().float().cpu()
    e2 = (got - ref).norm() / ref.norm().clamp_min(1e-12)
    einf = (got - ref).abs().max() / ref.abs().max().clamp_min(1e-12)
    assert e2 <= l2 and einf <= linf, f"{name}: rel l2 {e2:.3e} rel linf {einf:.3e}"


def _world(N, E, k, d, dff, act, zipf, slot_factor=3, seed=3, **kw):
    from paper_2407_04656_b200.layer import zipf_router_bias
    from paper_2407_04656_b200.loopback import LoopbackWorld
    from paper_2407_04656_b200.placement import plan_for_loads, replica_matrix
    loads = [int(1000 / (e + 1) ** zipf) + 1 for e in range(E)]
    plan = plan_for_loads(loads, N, math.ceil(slot_factor * E / N), fault_threshold=min(2, N))
    R = replica_matrix(plan)
    world = LoopbackWorld(N)
    layers = world.make_layers(d, dff, E, k, R, seed=seed, init_std=0.05,
                               router_bias=zipf_router_bias(E, zipf, seed=1), activation=act,
                               **kw)
    return world, layers, R


def _full_weights(layers, E):
    """Every expert's weights (fp32, CPU) from whichever rank hosts it."""
    from paper_2407_04656_b200.layer import deinterleave_swiglu
    L0 = layers[0]
    act = L0.activation
    w1 = torch.zeros(E, L0.d_ff, L0.d)
    w3 = torch.zeros(E, L0.d_ff, L0.d) if act == "swiglu" else None
    w2 = torch.zeros(E, L0.d, L0.d_ff)
    for L in layers:
        for p, e in enumerate(L.local_ids):
            if act == "swiglu":
                a, b = deinterleave_swiglu(L.w1.detach()[p].float().cpu())
                w1[e], w3[e] = a, b
            else:
                w1[e] = L.w1.detach()[p].float().cpu()
            w2[e] = L.w2.detach()[p].float().cpu()
    return w1, w2, w3


def _check_against_oracle(world, layers, xs, douts, outs, grads):
    from paper_2407_04656_b200 import ops
    from paper_2407_04656_b200.layer import interleave_swiglu
    L0 = layers[0]
    E, k, Tn = L0.E, L0.k, xs[0].shape[0]
    idx = torch.cat([ops.router_gate(x, L0.wg.detach(), L0.bg.detach(), k, L0.renorm)[0].cpu()
                     for x in xs])
    w1, w2, w3 = _full_weights(layers, E)
    for t in (w1, w2, w3):
        if t is not None:
            t.requires_grad_(True)
    X = torch.cat([x.float().cpu() for x in xs]).requires_grad_(True)
    wg = L0.wg.detach().float().cpu().requires_grad_(True)
    bg = L0.bg.detach().float().cpu().requires_grad_(True)
    ref, _, _, _ = moe_ref.moe_forward_ref(X, wg, bg, w1, w2, k, L0.renorm, idx=idx, w3=w3)
    ref.backward(torch.cat([g.float().cpu() for g in douts]))
    for r, L in enumerate(layers):
        sl = slice(r * Tn, (r + 1) * Tn)
        dx, dwg, dbg, dW1, dW2 = grads[r]
        _rel(outs[r], ref[sl], name=f"rank {r} out")
        _rel(dx, X.grad[sl], name=f"rank {r} dx")
        _rel(dwg, wg.grad, l2=5e-2, linf=1e-1, name=f"rank {r} dwg")
        _rel(dbg, bg.grad, l2=5e-2, linf=1e-1, name=f"rank {r} dbg")
        for p, e in enumerate(L.local_ids):
            if float(w2.grad[e].abs().max()) == 0.0:
                assert float(dW2[p].float().abs().max()) == 0.0
                continue
            want1 = w1.grad[e] if w3 is None else interleave_swiglu(w1.grad[e], w3.grad[e])
            _rel(dW1[p], want1, name=f"rank {r} dW1[{e}] owners {L.R[e]}")
            _rel(dW2[p], w2.grad[e], name=f"rank {r} dW2[{e}]")


def _inputs(N, Tn, d, seed=11):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    xs = [torch.randn(Tn, d, generator=g, device="cuda").bfloat16() for _ in range(N)]
    douts = [torch.randn(Tn, d, generator=g, device="cuda").bfloat16() for _ in range(N)]
    return xs, douts


# tail: the N > 1 variant of the backward tail overlap (LZ_TAIL_OVERLAP_NX; None = the
# default "auto": on from N = 4); split: the last weight-gradient GEMM + all-reduce in two
# expert-id halves (LZ_SPLIT_WGRAD=1)
@pytest.mark.parametrize("N,E,k,act,zipf,exchange,scatter,tail,split", [
    (2, 16, 2, "gelu", 1.2, "p2p", True, None, False),      # the product default, N = 2
    (4, 16, 2, "swiglu", 1.2, "p2p", True, None, False),    # the product default, N = 4
    (8, 16, 2, "gelu", 1.2, "p2p", True, False, False),
    (8, 64, 1, "gelu", 1.5, "p2p", True, None, True),       # cfg4-like: 64 experts, top-1
    (4, 64, 2, "swiglu", 0.8, "p2p", True, False, False),
    (3, 8, 2, "gelu", 0.0, "p2p", True, True, True),        # side-stream backward tail at N = 3
    (4, 16, 2, "gelu", 1.2, "p2p", False, False, False),    # gathering P2P (LZ_P2P_SCATTER=0)
    (4, 16, 2, "gelu", 1.2, "nccl", True, False, False),    # LZ_EXCHANGE=nccl: a2a-v + regroup
    (2, 8, 2, "swiglu", 2.5, "nccl", True, False, False),
])
def test_loopback_fwd_bwd_matches_oracle(N, E, k, act, zipf, exchange, scatter, tail, split):
    d, dff, Tn = 512, 1024, 512
    world, layers, R = _world(N, E, k, d, dff, act, zipf, exchange=exchange)
    for L in layers:
        L.scatter, L.tail_overlap_nx, L.split_last_wgrad = scatter, tail, split
    xs, douts = _inputs(N, Tn, d)
    outs, grads = world.step(layers, xs, douts)
    torch.cuda.synchronize()
    for L in layers:
        L.check()
    assert world.requests > 0 and not world.lost
    _check_against_oracle(world, layers, xs, douts, outs, grads)


@pytest.mark.parametrize("N,act", [(4, "gelu"), (8, "swiglu")])
def test_loopback_bit_identical_to_single_rank(N, act):
    """Each rank's output and input gradient do not depend on where its rows were
    computed: the N-rank exchange (arrival GEMM, scattering epilogues, combine-backward
    stores into remote buffers, barriers) gives the same BITS as one rank running the
    same tokens locally (every row meets the same kernels in the same reduction order)."""
    from paper_2407_04656_b200.layer import MoELayer, zipf_router_bias
    E, k, d, dff, Tn = 16, 2, 512, 1024, 1024
    world, layers, R = _world(N, E, k, d, dff, act, 1.2)
    xs, douts = _inputs(N, Tn, d, seed=5)
    outs, grads = world.step(layers, xs, douts)
    single = MoELayer(d, dff, E, k, seed=3, init_std=0.05, router_bias=zipf_router_bias(E, 1.2, 1),
                      activation=act)
    for r in range(N):
        x = xs[r].clone().requires_grad_(True)
        single.zero_grad(set_to_none=True)
        out = single(x)
        out.backward(douts[r])
        assert torch.equal(outs[r], out), f"rank {r} out"
        assert torch.equal(grads[r][0], x.grad), f"rank {r} dx"


def test_loopback_full_size_cfg2_sampled():
    """BASELINE cfg2 at full size on 8 virtual ranks (65,536 tokens per rank, E16 top-2,
    d1024, d_ff4096, Zipf 1.2, c = ceil(6E/N)): sampled tokens' outputs and input grads
    against the oracle (each token's result depends only on its routing and the weights)."""
    from paper_2407_04656_b200 import ops
    from paper_2407_04656_b200.layer import zipf_router_bias
    from paper_2407_04656_b200.loopback import LoopbackWorld
    from paper_2407_04656_b200.placement import plan_for_loads, replica_matrix
    N, E, k, d, dff, Tn = 8, 16, 2, 1024, 4096, 65536
    bias = zipf_router_bias(E, 1.2, seed=0)
    world = LoopbackWorld(N)
    g = torch.Generator(device="cuda")
    g.manual_seed(1234)
    xs = [torch.randn(Tn, d, generator=g, device="cuda").bfloat16() for _ in range(N)]
    probe = world.make_layers(d, dff, E, k, None, seed=0, router_bias=bias,
                              router_std=1.28 / math.sqrt(d))[0]
    loads = sum(ops.router_gate(x, probe.wg.detach(), probe.bg.detach(), k)[3].long().cpu()
                for x in xs).tolist()
    R = replica_matrix(plan_for_loads(loads, N, math.ceil(6 * E / N), 2))
    layers = world.make_layers(d, dff, E, k, R, seed=0, router_bias=bias,
                               router_std=1.28 / math.sqrt(d))
    del probe
    ns = 24
    samples = [torch.randperm(Tn, generator=torch.Generator().manual_seed(r))[:ns].cuda()
               for r in range(N)]
    douts = []
    for s in samples:
        dd = torch.zeros(Tn, d, device="cuda").bfloat16()
        dd[s] = torch.randn(ns, d, generator=g, device="cuda").bfloat16()
        douts.append(dd)
    outs, grads = world.step(layers, xs, douts)
    torch.cuda.synchronize()
    for L in layers:
        L.check()
    w1, w2, _ = _full_weights(layers, E)
    L0 = layers[0]
    wg, bg = L0.wg.detach().float().cpu(), L0.bg.detach().float().cpu()
    for r in range(N):
        xsmp = xs[r][samples[r]]
        gidx = ops.router_gate(xsmp, L0.wg.detach(), L0.bg.detach(), k)[0].cpu()
        xr = xsmp.float().cpu().requires_grad_(True)
        ref, _, _, _ = moe_ref.moe_forward_ref(xr, wg, bg, w1, w2, k, False, idx=gidx)
        ref.backward(douts[r][samples[r]].float().cpu())
        _rel(outs[r][samples[r]], ref, name=f"rank {r} out")
        _rel(grads[r][0][samples[r]], xr.grad, name=f"rank {r} dx")
    imb = [L.imbalance() for L in layers]
    assert max(imb) < 1.5


def test_loopback_capacity_overflow_then_reserve():
    """Exchange buffers sized below the plan's need: every rank raises the same
    ExchangeCapacityError (nothing exchanged, no out-of-bounds write), reserve() grows the
    buffers, and the re-run step matches the oracle."""
    from paper_2407_04656_b200.dispatch import ExchangeCapacityError
    N, E, k, d, dff, Tn = 4, 8, 2, 256, 512, 4096
    world, layers, R = _world(N, E, k, d, dff, "gelu", 2.5, slot_factor=1)
    for L in layers:
        L.capacity_slack = 0.3     # 0.3 x 8192 rows + 8 x 255 padding < the hot rank's rows
    xs, douts = _inputs(N, Tn, d)
    world.step(layers, xs)
    torch.cuda.synchronize()
    needs = []
    for L in layers:
        with pytest.raises(ExchangeCapacityError) as ei:
            L.check()
        needs.append(ei.value.rows)
    assert len(set(needs)) == 1 and needs[0] > layers[0]._symm.rows
    for L in layers:
        L.reserve(needs[0])
    outs, grads = world.step(layers, xs, douts)
    torch.cuda.synchronize()
    for L in layers:
        L.check()
    _check_against_oracle(world, layers, xs, douts, outs, grads)


# the forward of a step after the first issues HIST, SYNC (after the dispatch + arrival
# signals), BARRIER (before the combine): lose after 1 = before the dispatch, after 2 =
# after the dispatch, before its expert GEMMs and the combine
@pytest.mark.parametrize("lose_after", [1, 2])
def test_loopback_lost_rank_aborts_then_shrinks(lose_after):
    """A rank lost mid-step (after its all-gather: before its dispatch -- the survivors'
    arrival GEMMs wait on its flag; or after its dispatch, before the combine -- the
    survivors' barrier waits on it): the device waits give up after the control block's
    timeout instead of hanging, every survivor's check() raises StepAbortedError, the
    step is discarded, the survivors re-plan (reference recipe) and move the lost rank's
    expert state from surviving owners, and the next step matches the oracle."""
    from paper_2407_04656_b200 import _lib
    from paper_2407_04656_b200.layer import StepAbortedError
    N, E, k, d, dff, Tn = 4, 16, 2, 512, 1024, 512
    world, layers, R = _world(N, E, k, d, dff, "gelu", 1.2, slot_factor=4)
    xs, douts = _inputs(N, Tn, d)
    _lib.control(timeout_s=0.25)
    _lib.control_reset()
    try:
        outs, grads = world.step(layers, xs, douts)          # healthy step (allocates)
        torch.cuda.synchronize()
        opts = []
        for L, gr in zip(layers, grads):
            L.check()
            L.w1.grad, L.w2.grad = gr[3], gr[4]
            opt = torch.optim.Adam([L.w1, L.w2], lr=1e-3)
            opt.step()
            opts.append(opt)
        # every owner of an expert holds the same weights and optimizer moments
        moments = {}
        for L, opt in zip(layers, opts):
            for p, e in enumerate(L.local_ids):
                m = (L.w1.data[p].clone(), opt.state[L.w1]["exp_avg"][p].clone(),
                     opt.state[L.w2]["exp_avg_sq"][p].clone())
                if e in moments:
                    assert all(torch.equal(a, b) for a, b in zip(m, moments[e]))
                moments[e] = m
        lost = 2
        world.step(layers, xs, lose={lost: lose_after})      # rank 2 dies mid-forward
        torch.cuda.synchronize()
        assert world.lost == {lost}
        for r, L in enumerate(layers):
            if r == lost:
                continue
            with pytest.raises(StepAbortedError) as ei:
                L.check()
            assert ei.value.status["timeout"]
        _lib.control_reset()
        loads = [int(1000 / (e + 1) ** 1.2) + 1 for e in range(E)]
        world2, survivors, report = world.shrink(layers, loads, slots=math.ceil(4 * E / 3),
                                                 optimizers=opts)
        assert report["live"] == [0, 1, 3] and world2.n == 3 and report["transfers"] > 0
        # migrated experts arrive with their weights AND optimizer moments
        for L, r in zip(survivors, report["live"]):
            opt = opts[r]
            assert opt.param_groups[0]["params"][0] is L.w1
            for p, e in enumerate(L.local_ids):
                w, m1, v2 = moments[e]
                assert torch.equal(L.w1.data[p], w), f"expert {e} weights on node {r}"
                assert torch.equal(opt.state[L.w1]["exp_avg"][p], m1), f"expert {e} exp_avg"
                assert torch.equal(opt.state[L.w2]["exp_avg_sq"][p], v2), f"expert {e} v"
        xs2 = [xs[r] for r in report["live"]]
        ds2 = [douts[r] for r in report["live"]]
        outs, grads = world2.step(survivors, xs2, ds2)
        torch.cuda.synchronize()
        for L in survivors:
            L.check()
        assert not report["checkpoint_fallback"]
        _check_against_oracle(world2, survivors, xs2, ds2, outs, grads)
    finally:
        _lib.control(timeout_s=10.0)
        _lib.control_reset()


def test_loopback_cfg3_shape_fwd_bwd():
    """BASELINE cfg3 expert shape (Mixtral: E8 top-2, d4096, d_ff14336 SwiGLU) on 2
    virtual ranks, full fwd + bwd incl. the replica-group gradient sums, against the
    oracle on the gathered batch (1024 tokens per rank: the CPU oracle's budget)."""
    N, E, k, d, dff, Tn = 2, 8, 2, 4096, 14336, 1024
    world, layers, R = _world(N, E, k, d, dff, "swiglu", 1.2, slot_factor=5)
    xs, douts = _inputs(N, Tn, d)
    outs, grads = world.step(layers, xs, douts)
    torch.cuda.synchronize()
    for L in layers:
        L.check()
    _check_against_oracle(world, layers, xs, douts, outs, grads)


def test_loopback_full_size_cfg3_sampled():
    """cfg3 at its full per-GPU size (16,384 tokens per rank) on 2 virtual ranks:
    sampled tokens' outputs and input gradients against the oracle."""
    from paper_2407_04656_b200 import ops
    from paper_2407_04656_b200.layer import interleave_swiglu  # noqa: F401
    N, E, k, d, dff, Tn = 2, 8, 2, 4096, 14336, 16384
    world, layers, R = _world(N, E, k, d, dff, "swiglu", 1.2, slot_factor=5)
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    xs = [torch.randn(Tn, d, generator=g, device="cuda").bfloat16() for _ in range(N)]
    ns = 16
    samples = [torch.randperm(Tn, generator=torch.Generator().manual_seed(r))[:ns].cuda()
               for r in range(N)]
    douts = []
    for smp in samples:
        dd = torch.zeros(Tn, d, device="cuda").bfloat16()
        dd[smp] = torch.randn(ns, d, generator=g, device="cuda").bfloat16()
        douts.append(dd)
    outs, grads = world.step(layers, xs, douts)
    torch.cuda.synchronize()
    for L in layers:
        L.check()
    w1, w2, w3 = _full_weights(layers, E)
    L0 = layers[0]
    wg, bg = L0.wg.detach().float().cpu(), L0.bg.detach().float().cpu()
    for r in range(N):
        xsmp = xs[r][samples[r]]
        gidx = ops.router_gate(xsmp, L0.wg.detach(), L0.bg.detach(), k)[0].cpu()
        xr = xsmp.float().cpu().requires_grad_(True)
        ref, _, _, _ = moe_ref.moe_forward_ref(xr, wg, bg, w1, w2, k, False, idx=gidx, w3=w3)
        ref.backward(douts[r][samples[r]].float().cpu())
        _rel(outs[r][samples[r]], ref, name=f"rank {r} out")
        _rel(grads[r][0][samples[r]], xr.grad, name=f"rank {r} dx")


def test_loopback_elastic_8_6_4():
    """BASELINE cfg5's 8 -> 6 -> 4 reconfiguration on one GPU: 8 virtual ranks, two ranks
    lost mid-step (after their dispatch), shrink to 6 with the reference re-plan recipe and
    expert-state moves, then two more lost, shrink to 4; after each shrink a full fwd + bwd
    step matches the oracle.  Slots per rank stay at the 8-rank value."""
    from paper_2407_04656_b200 import _lib
    from paper_2407_04656_b200.layer import StepAbortedError
    N, E, k, d, dff, Tn = 8, 16, 2, 512, 1024, 512
    slots = math.ceil(6 * E / 8)
    world, layers, R = _world(N, E, k, d, dff, "gelu", 1.2, slot_factor=6)
    xs, douts = _inputs(N, Tn, d)
    loads = [int(1000 / (e + 1) ** 1.2) + 1 for e in range(E)]
    _lib.control(timeout_s=0.25)
    _lib.control_reset()
    try:
        world.step(layers, xs, douts)
        torch.cuda.synchronize()
        for L in layers:
            L.check()
        for lost in ((3, 6), (1, 4)):
            world.step(layers, xs, lose={r: 2 for r in lost})   # after their dispatch
            torch.cuda.synchronize()
            assert world.lost == set(lost)
            for r, L in enumerate(layers):
                if r not in lost:
                    with pytest.raises(StepAbortedError):
                        L.check()
            _lib.control_reset()
            world, layers, report = world.shrink(layers, loads, slots=slots)
            keep = report["live"]
            xs, douts = [xs[r] for r in keep], [douts[r] for r in keep]
            outs, grads = world.step(layers, xs, douts)
            torch.cuda.synchronize()
            for L in layers:
                L.check()
            _check_against_oracle(world, layers, xs, douts, outs, grads)
        assert world.n == 4
    finally:
        _lib.control(timeout_s=10.0)
        _lib.control_reset()
