"""N virtual EP ranks on one GPU (VirtualEP): the N-rank plan, the fused P2P
dispatch/combine layouts and the per-rank grouped GEMMs must give, for every virtual
rank, bit-identically what the single-rank layer computes on that rank's tokens
(replicas of an expert share one weight copy, and every row is computed by the same
kernels in the same reduction order)."""

import pytest
import torch

from oracle import dispatch_ref

pytestmark = pytest.mark.gpu


def _setup(N, E, k, d, dff, Tn, act, zipf, seed=3, scatter=False):
    from paper_2407_04656_b200.layer import MoELayer, zipf_router_bias, default_slots
    from paper_2407_04656_b200.placement import plan_for_loads, replica_matrix
    from paper_2407_04656_b200.virtual import VirtualEP
    bias = zipf_router_bias(E, zipf) if zipf else None
    loads = [int(1000 / (e + 1) ** (zipf or 0.0)) + 1 for e in range(E)]
    plan = plan_for_loads(loads, N, default_slots(E, N), fault_threshold=min(2, N))
    R = replica_matrix(plan)
    vep = VirtualEP(d, dff, E, k, R, Tn, seed=seed, router_bias=bias, activation=act,
                    scatter=scatter)
    ref = MoELayer(d, dff, E, k, seed=seed, router_bias=bias, activation=act)
    torch.manual_seed(seed)
    xs = [torch.randn(Tn, d, device="cuda").bfloat16() for _ in range(N)]
    return vep, ref, xs, R


@pytest.mark.parametrize("N,E,k,act,zipf,scatter", [(4, 8, 2, "gelu", 1.2, False),
                                                     (8, 16, 2, "gelu", 0.8, False),
                                                     (8, 8, 1, "swiglu", 1.5, False),
                                                     (3, 8, 2, "gelu", 0.0, False),
                                                     (4, 8, 2, "gelu", 1.2, True),
                                                     (8, 16, 2, "swiglu", 0.8, True),
                                                     (3, 8, 1, "gelu", 0.0, True)])
def test_virtual_ranks_match_single_rank(N, E, k, act, zipf, scatter):
    """scatter=True: the second GEMM's epilogue returns rows to their source rank (the
    multi-GPU default) -- same bits as the gathered combine."""
    d, dff, Tn = 512, 1024, 1024
    vep, ref, xs, R = _setup(N, E, k, d, dff, Tn, act, zipf, scatter=scatter)
    with torch.no_grad():
        outs = vep(xs)
        torch.cuda.synchronize()
        vep.check()
        for r in range(N):
            want = ref(xs[r])
            assert torch.equal(outs[r], want), f"rank {r}: max diff " \
                f"{(outs[r].float() - want.float()).abs().max().item()}"


def test_virtual_plan_matches_oracle_schedule():
    """The device plans of all N virtual ranks reproduce the oracle's dispatch
    matrices (the all-gathered T is the stacked per-rank histograms)."""
    N, E, k = 8, 16, 2
    vep, _, xs, R = _setup(N, E, k, 512, 1024, 1024, "gelu", 1.0)
    with torch.no_grad():
        vep(xs)
    torch.cuda.synchronize()
    T = None
    for r, p in enumerate(vep.last_plans):
        D = p.D.cpu().numpy()
        if T is None:
            from paper_2407_04656_b200 import ops
            hists = [ops.router_gate(x, vep.wg, vep.bg, k)[3].cpu() for x in xs]
            T = torch.stack(hists, dim=1).numpy()
            Dref = dispatch_ref.full_dispatch_matrices(T.tolist(), R)
        for i in range(N):
            assert D[i].tolist() == Dref[i], f"sender {i} seen from rank {r}"
        sch = dispatch_ref.compute_dispatch_schedule(r, T.tolist(), R)
        assert p.recv_sizes.cpu().tolist() == sch["recv"]   # excludes self, as the reference
        assert p.send_sizes.cpu().tolist() == sch["s"]
