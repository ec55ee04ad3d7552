"""K1/K3/K7/K8 kernels vs the CPU oracle / torch fp32 references of the same op.

Tolerances (written per check): routed expert ids are exact for identical fp32
logits; fp32 softmax/weights 1e-5 abs; bf16 data movement is exact (pack) or one
bf16 rounding of an fp32 result (combine, backward): |err| <= 8e-3 * |ref| + 1e-3 * max|ref|.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import moe_ref  # noqa: E402
from paper_2407_04656_b200 import ops  # noqa: E402


def _close(got, ref, rtol=8e-3, atol_scale=1e-3):
    got, ref = got.float().cpu(), ref.float().cpu()
    tol = atol_scale * ref.abs().max().clamp_min(1e-6) + rtol * ref.abs()
    err = (got - ref).abs()
    assert (err <= tol).all(), f"max err {err.max().item():.4g} (ref max {ref.abs().max().item():.4g})"


def test_router_gate_histogram_slots():
    """The streaming router writes its histogram without a memset (per-CTA rows in a rolling
    per-launch workspace slot, summed by the last CTA, ticket self-reset): 600 launches of
    varying sizes wrap the 256-slot pool twice and every histogram stays exact, also when
    the same slot is replayed from a CUDA graph."""
    g = torch.Generator().manual_seed(3)
    E, k, d = 16, 2, 256
    wg = (torch.randn(E, d, generator=g) * 0.05).bfloat16().cuda()
    bias = torch.zeros(E).cuda()
    xs = [torch.randn(n, d, generator=g).bfloat16().cuda() for n in (1, 17, 700, 5000)]
    for i in range(600):
        x = xs[i % len(xs)]
        idx, _, _, hist = ops.router_gate(x, wg, bias, k)
        ref = torch.bincount(idx.reshape(-1).long(), minlength=E).int()
        assert torch.equal(hist, ref), i
    x = xs[-1]
    graph = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(graph, stream=s):
        out = ops.router_gate(x, wg, bias, k)
    for _ in range(5):
        out[3].fill_(-1)
        graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(out[3], torch.bincount(out[0].reshape(-1).long(), minlength=E).int())


@pytest.mark.parametrize("Tn,E,k,renorm", [(1000, 16, 2, False), (4096, 8, 2, True),
                                           (333, 64, 1, False), (64, 5, 3, True),
                                           (100000, 64, 2, False), (5000, 1024, 2, True),
                                           (777, 33, 1, False), (256, 16, 2, True),
                                           (300, 64, 4, False)])
def test_gate_topk_exact_ids(Tn, E, k, renorm):
    g = torch.Generator().manual_seed(Tn + E)
    logits = torch.randn(Tn, E, generator=g)
    logits[::7, 1] = logits[::7, 0]  # exact ties -> lower id must win
    idx, w, probs, hist = ops.gate_topk(logits.cuda(), k, renorm)
    ridx, rw, rprobs = moe_ref.gate_ref(logits, k, renorm)
    assert torch.equal(idx.cpu(), ridx)
    assert torch.allclose(w.cpu(), rw, atol=1e-5)
    assert torch.allclose(probs.cpu(), rprobs, atol=1e-5)
    assert torch.equal(hist.cpu(), torch.bincount(ridx.reshape(-1).long(), minlength=E).int())


@pytest.mark.parametrize("Tn,d,E,k", [(4096, 1024, 16, 2), (1000, 512, 8, 2), (257, 2048, 64, 1),
                                      (100, 4096, 8, 2), (70000, 1024, 16, 2), (300, 96, 5, 1),
                                      (513, 256, 40, 3), (2405, 512, 8, 1), (40000, 256, 16, 2),
                                      (5003, 1024, 3, 1), (3000, 128, 12, 4), (5, 512, 16, 2),
                                      (2368, 1024, 16, 2), (9472, 1024, 16, 2)])
def test_router_gate(Tn, d, E, k):
    g = torch.Generator().manual_seed(d)
    x = torch.randn(Tn, d, generator=g).bfloat16()
    wg = (torch.randn(E, d, generator=g) * 0.02).bfloat16()
    bias = torch.randn(E, generator=g) * 0.5
    idx, w, probs, hist = ops.router_gate(x.cuda(), wg.cuda(), bias.cuda(), k)
    logits = x.float() @ wg.float().t() + bias
    ridx, rw, rprobs = moe_ref.gate_ref(logits, k)
    # fp32 accumulate in a different order: probabilities within 1e-4; ids equal except
    # where the k-th / (k+1)-th logit margin is below 1e-3
    assert torch.allclose(probs.cpu(), rprobs, atol=1e-4)
    srt = logits.sort(dim=1, descending=True).values
    margin = (srt[:, :k] - srt[:, 1:k + 1]).abs().min(dim=1).values
    safe = margin > 1e-3
    assert safe.float().mean() > 0.9
    assert torch.equal(idx.cpu()[safe], ridx[safe])
    assert int(hist.sum()) == Tn * k
    assert torch.equal(hist.cpu(), torch.bincount(idx.cpu().reshape(-1).long(), minlength=E).int())
    # a token's logits do not depend on its position in the batch (the streaming kernel
    # splits the batch into per-SM ranges): any row subset routes identically
    sub = torch.arange(Tn - 1, -1, -3)
    idx2, w2, probs2, _ = ops.router_gate(x[sub].cuda(), wg.cuda(), bias.cuda(), k)
    assert torch.equal(idx2.cpu(), idx.cpu()[sub])
    assert torch.equal(probs2.cpu(), probs.cpu()[sub])


def _rows(Tn, k, n_rows, gen):
    return torch.randperm(n_rows, generator=gen)[:Tn * k].int()


@pytest.mark.parametrize("d", [1024, 2048])   # cfg2 / cfg4 model widths
@pytest.mark.parametrize("m,off", [([2500, 0, 3500], [0, 2560, 2560, 6144]),      # 128-aligned
                                   ([2049, 0, 3951], [0, 2304, 2304, 6400])])     # pads up to 255
def test_pack_exact_and_pad_zero(m, off, d):
    gen = torch.Generator().manual_seed(5)
    Tn, k = 3000, 2
    x = torch.randn(Tn, d, generator=gen).bfloat16()
    mt = torch.tensor(m, dtype=torch.int32)
    ot = torch.tensor(off, dtype=torch.int32)
    perm = torch.randperm(6000, generator=gen)
    real_rows = torch.cat([torch.arange(off[e], off[e] + m[e]) for e in range(3)])
    row = real_rows[perm].int()
    out = torch.full((off[-1], d), 7.0).bfloat16().cuda()
    ops.pack(x.cuda(), row.cuda(), k, out, mt.cuda(), ot.cuda())
    ref = torch.zeros(off[-1], d).bfloat16()
    ref[row.long()] = x.repeat_interleave(k, dim=0)
    assert torch.equal(out.cpu(), ref)


@pytest.mark.parametrize("d,k", [(1024, 2), (2048, 1), (2048, 2)])
def test_combine_and_backward(d, k):
    gen = torch.Generator().manual_seed(6)
    Tn, E = 2048, 16
    n_rows = Tn * k + 512
    y = torch.randn(n_rows, d, generator=gen).bfloat16()
    row = _rows(Tn, k, n_rows, gen)
    w = torch.rand(Tn, k, generator=gen)
    out = ops.combine(y.cuda(), row.cuda(), w.cuda(), k)
    yr = y.float()[row.long()].view(Tn, k, d)
    ref = (yr * w.unsqueeze(-1)).sum(1)
    _close(out, ref)
    # backward: dy rows and dw
    dout = torch.randn(Tn, d, generator=gen).bfloat16()
    dy = torch.full((n_rows, d), 3.0).bfloat16().cuda()
    dw = ops.combine_bwd(dout.cuda(), y.cuda(), row.cuda(), w.cuda(), k, dy)
    ref_dy = (dout.float().unsqueeze(1) * w.unsqueeze(-1)).reshape(Tn * k, d)
    _close(dy.cpu()[row.long()], ref_dy)
    ref_dw = (dout.float().unsqueeze(1) * yr).sum(-1)
    _close(dw, ref_dw, rtol=1e-4, atol_scale=1e-4)
    del E


@pytest.mark.parametrize("renorm,Tn,d,E,k", [(False, 1024, 512, 16, 2), (True, 1024, 512, 16, 2),
                                              (False, 5003, 1024, 8, 1), (True, 3001, 256, 12, 2),
                                              (False, 700, 2048, 16, 2), (True, 257, 512, 32, 3)])
def test_dispatch_bwd_and_router_grads(renorm, Tn, d, E, k):
    """dx = sum_s dxe[row] + dlogits . wg and dlogits from the softmax/top-k backward,
    against torch autograd on the same fp32 math (streaming kernel: E <= 16, k <= 2,
    d % 256 == 0, d <= 1024; the register-prefetch kernel otherwise)."""
    gen = torch.Generator().manual_seed(7)
    x = torch.randn(Tn, d, generator=gen).bfloat16()
    wg = (torch.randn(E, d, generator=gen) * 0.05).bfloat16()
    logits = (x.float() @ wg.float().t()).requires_grad_(True)
    idx, _, _ = moe_ref.gate_ref(logits, k, renorm)
    probs = torch.softmax(logits, 1)
    wsel = torch.gather(probs, 1, idx.long())
    if renorm:
        wsel = wsel / wsel.sum(1, keepdim=True)
    dw = torch.randn(Tn, k, generator=gen)
    (wsel * dw).sum().backward()
    ref_dlog = logits.grad
    n_rows = Tn * k
    row = _rows(Tn, k, n_rows, gen)
    dxe = torch.randn(n_rows, d, generator=gen).bfloat16()
    dx, dlog = ops.dispatch_bwd(dxe.cuda(), row.cuda(), probs.detach().cuda(), idx.cuda(),
                                dw.cuda(), wg.cuda(), renorm, Tn)
    _close(dlog, ref_dlog, rtol=1e-4, atol_scale=1e-5)
    # the gate backward alone (router weight gradient off the critical path) gives the
    # same bits as the fused dispatch backward
    dlog2 = ops.gate_bwd(probs.detach().cuda(), idx.cuda(), dw.cuda(), renorm)
    assert torch.equal(dlog2, dlog)
    ref_dx = dxe.float()[row.long()].view(Tn, k, d).sum(1) + ref_dlog @ wg.float()
    _close(dx, ref_dx)
    dwg, db = ops.router_wgrad(dlog, x.cuda())
    _close(dwg, dlog.cpu().t() @ x.float(), rtol=1e-4, atol_scale=1e-4)
    _close(db, dlog.cpu().sum(0), rtol=1e-4, atol_scale=1e-4)


@pytest.mark.parametrize("Tn,d,E", [(1000, 1024, 16), (333, 2048, 8), (4099, 4096, 40),
                                     (100, 96, 5), (17, 256, 64)])
def test_router_wgrad_shapes(Tn, d, E):
    """dWg = dlogits^T x and dbias = sum_t dlogits: tensor-core path (d % 256 == 0, any
    E, ragged token counts) and the FMA path, against fp32 torch."""
    gen = torch.Generator().manual_seed(11)
    x = torch.randn(Tn, d, generator=gen).bfloat16()
    dlog = torch.randn(Tn, E, generator=gen) * 1e-2
    dwg, db = ops.router_wgrad(dlog.cuda(), x.cuda())
    _close(dwg, dlog.t() @ x.float(), rtol=1e-4, atol_scale=1e-4)
    _close(db, dlog.sum(0), rtol=1e-4, atol_scale=1e-4)


def test_copy_segments():
    gen = torch.Generator().manual_seed(8)
    d = 256
    src = torch.randn(1000, d, generator=gen).bfloat16().cuda()
    dst = torch.zeros(1200, d).bfloat16().cuda()
    s = torch.tensor([0, 100, 600], dtype=torch.int32)
    t = torch.tensor([500, 0, 900], dtype=torch.int32)
    c = torch.tensor([100, 500, 250], dtype=torch.int32)
    ops.copy_segments(src, dst, s.cuda(), t.cuda(), c.cuda(), 500)
    for a, b, n in zip(s.tolist(), t.tolist(), c.tolist()):
        assert torch.equal(dst[b:b + n].cpu(), src[a:a + n].cpu())
    assert np.count_nonzero(dst[850:900].float().cpu().numpy()) == 0
