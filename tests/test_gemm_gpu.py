"""tcgen05 grouped GEMM (K4-K6) vs a torch fp32 reference of the same op.

Tolerance: inputs are bf16, accumulation fp32, output rounded to bf16, so the
error bound is ~2^-8 relative per element plus accumulation-order noise:
|got - ref| <= 1e-2 * max|ref| + 1e-2 * |ref| elementwise.
"""

import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2407_04656_b200 import _lib, ops  # noqa: E402


@pytest.fixture(params=[1, 2], ids=["cta1", "cta2"], autouse=True)
def cg(request):
    """Run every GEMM test on the single-CTA and on the CTA-pair (cta_group::2) kernel;
    mode-0 segment sizes are scaled to the variant's row alignment."""
    prev = ops.set_gemm_cta_group(request.param)
    yield request.param
    ops.set_gemm_cta_group(2)
    del prev


def _close(got, ref, rtol=1e-2, atol_scale=1e-2):
    got = got.float()
    ref = ref.float()
    if ref.numel() == 0:
        return
    tol = atol_scale * ref.abs().max().clamp_min(1e-6) + rtol * ref.abs()
    bad = (got - ref).abs() > tol
    assert not bad.any(), f"{int(bad.sum())} / {bad.numel()} mismatches, max err " \
                          f"{(got - ref).abs().max().item():.4g}, max ref {ref.abs().max().item():.4g}"


def _offsets(sizes):
    off = [0]
    for s in sizes:
        off.append(off[-1] + s)
    return torch.tensor(off, dtype=torch.int32, device="cuda"), off


@pytest.mark.parametrize("sizes,K,N", [([128], 64, 256), ([128, 256, 0, 384], 128, 256),
                                       ([512, 128], 1024, 512), ([1024], 1024, 4096)])
def test_rows_kmajor(sizes, K, N, cg):
    torch.manual_seed(0)
    off_t, off = _offsets([v * cg for v in sizes])
    rows, G = off[-1], len(sizes)
    A = torch.randn(rows, K, device="cuda").bfloat16()
    B = (torch.randn(G, N, K, device="cuda") / K ** 0.5).bfloat16()
    C = torch.full((rows, N), float("nan"), device="cuda").bfloat16()
    ops.grouped_gemm_rows(A, B, off_t, C)
    torch.cuda.synchronize()
    for g in range(G):
        a = A[off[g]:off[g + 1]].float()
        _close(C[off[g]:off[g + 1]], a @ B[g].float().t())


@pytest.mark.parametrize("sizes,K,N", [([128, 256], 128, 256), ([384, 0, 128], 512, 512)])
def test_rows_mnmajor_b(sizes, K, N, cg):
    torch.manual_seed(1)
    off_t, off = _offsets([v * cg for v in sizes])
    rows, G = off[-1], len(sizes)
    A = torch.randn(rows, K, device="cuda").bfloat16()
    B = (torch.randn(G, K, N, device="cuda") / K ** 0.5).bfloat16()  # [K, N] per group
    C = torch.empty((rows, N), device="cuda").bfloat16()
    ops.grouped_gemm_rows(A, B, off_t, C, b_major=_lib.LZ_MN_MAJOR)
    torch.cuda.synchronize()
    for g in range(G):
        _close(C[off[g]:off[g + 1]], A[off[g]:off[g + 1]].float() @ B[g].float())


def test_gelu_and_dgelu_epilogues(cg):
    """GELU epilogue: C = gelu(acc) and AUX = gelu'(acc) (the backward factor);
    dGELU epilogue: C = acc * AUX."""
    torch.manual_seed(2)
    sizes, K, N = [256, 128], 256, 512
    off_t, off = _offsets([v * cg for v in sizes])
    rows, G = off[-1], len(sizes)
    A = torch.randn(rows, K, device="cuda").bfloat16()
    B = (torch.randn(G, N, K, device="cuda") / K ** 0.5).bfloat16()
    D = torch.empty((rows, N), device="cuda").bfloat16()
    Act = torch.empty((rows, N), device="cuda").bfloat16()
    ops.grouped_gemm_rows(A, B, off_t, Act, epilogue=_lib.LZ_EPI_GELU, aux=D)
    B2 = (torch.randn(G, K, N, device="cuda") / K ** 0.5).bfloat16()
    dH = torch.empty((rows, N), device="cuda").bfloat16()
    ops.grouped_gemm_rows(A, B2, off_t, dH, b_major=_lib.LZ_MN_MAJOR,
                          epilogue=_lib.LZ_EPI_DGELU, aux=D)
    torch.cuda.synchronize()
    Drows = ops.aux_rows(D)   # the aux stream is in the private blocked layout
    for g in range(G):
        sl = slice(off[g], off[g + 1])
        pre = (A[sl].float() @ B[g].float().t()).requires_grad_(True)
        act = torch.nn.functional.gelu(pre, approximate="tanh")
        act.backward(torch.ones_like(act))
        _close(Act[sl], act.detach(), rtol=2e-2)
        _close(Drows[sl], pre.grad, rtol=2e-2)
        _close(dH[sl], (A[sl].float() @ B2[g].float()) * Drows[sl].float(), rtol=2e-2)


def test_gelu_aux_layout_roundtrip():
    x = torch.arange(64 * 96, dtype=torch.float32).view(64, 96)
    from paper_2407_04656_b200 import ops as O
    assert torch.equal(O.aux_rows(O.aux_blocked(x)), x)


@pytest.mark.parametrize("sizes,M,N", [([128], 256, 256), ([64, 0, 192, 128], 256, 512),
                                       ([1024, 512], 1024, 256), ([2048, 0, 4352, 256], 512, 1536),
                                       ([8192, 3072], 1024, 4096)])
def test_wgrad_variable_k(sizes, M, N):
    """Variable-K weight gradients; N % 512 == 0 runs the 256 x 512 tiles (NS = 2)."""
    torch.manual_seed(3)
    off_t, off = _offsets(sizes)
    rows, G = off[-1], len(sizes)
    A = torch.randn(rows, M, device="cuda").bfloat16()
    B = torch.randn(rows, N, device="cuda").bfloat16()
    C = torch.full((G, M, N), float("nan"), device="cuda").bfloat16()
    ops.grouped_gemm_wgrad(A, B, off_t, C)
    torch.cuda.synchronize()
    for g in range(G):
        sl = slice(off[g], off[g + 1])
        ref = A[sl].float().t() @ B[sl].float()
        if off[g + 1] == off[g]:
            assert (C[g] == 0).all()
        else:
            _close(C[g], ref)


def test_persistent_grid_smaller_than_tiles(cg):
    torch.manual_seed(4)
    off_t, off = _offsets([640 * cg, 384 * cg])
    K, N = 192, 768
    A = torch.randn(off[-1], K, device="cuda").bfloat16()
    B = (torch.randn(2, N, K, device="cuda") / K ** 0.5).bfloat16()
    C = torch.empty((off[-1], N), device="cuda").bfloat16()
    ops.grouped_gemm_rows(A, B, off_t, C, num_sms=4)  # 4 CTAs loop over 24 tiles
    torch.cuda.synchronize()
    for g in range(2):
        _close(C[off[g]:off[g + 1]], A[off[g]:off[g + 1]].float() @ B[g].float().t())


def test_wgrad_interleaved_output():
    """c_group_rows / c_row_offset place C_g inside a flat per-expert buffer."""
    torch.manual_seed(5)
    off_t, off = _offsets([128, 256])
    M, N = 256, 512
    A = torch.randn(off[-1], M, device="cuda").bfloat16()
    B = torch.randn(off[-1], N, device="cuda").bfloat16()
    buf = torch.zeros(2, 3 * M, N, device="cuda").bfloat16()   # per group: [pad M | C_g | pad M]
    ops.grouped_gemm_wgrad(A, B, off_t, buf, c_group_rows=3 * M, c_row_offset=M)
    torch.cuda.synchronize()
    for g in range(2):
        sl = slice(off[g], off[g + 1])
        _close(buf[g, M:2 * M], A[sl].float().t() @ B[sl].float())
        assert (buf[g, :M] == 0).all() and (buf[g, 2 * M:] == 0).all()


def _interleave(w1, w3):
    """[G, F, K] x2 -> [G, 2F, K] with 128-row blocks alternating gate / up."""
    G, F, K = w1.shape
    return torch.stack([w1.view(G, F // 128, 128, K), w3.view(G, F // 128, 128, K)],
                       dim=2).reshape(G, 2 * F, K)


def test_swiglu_epilogues(cg):
    """SwiGLU: C = silu(g) u, AUX = [silu(g) | u silu'(g)] (interleaved like W1|W3);
    dSwiGLU: C = [dA * u silu'(g) | dA * silu(g)] = [dgate | dup]."""
    torch.manual_seed(6)
    sizes, K, F = [256, 512], 256, 512
    off_t, off = _offsets([v * cg for v in sizes])
    rows, G = off[-1], len(sizes)
    X = torch.randn(rows, K, device="cuda").bfloat16()
    w1 = (torch.randn(G, F, K, device="cuda") / K ** 0.5).bfloat16()
    w3 = (torch.randn(G, F, K, device="cuda") / K ** 0.5).bfloat16()
    W13 = _interleave(w1, w3).contiguous()
    H = torch.empty(rows, 2 * F, device="cuda").bfloat16()
    Act = torch.empty(rows, F, device="cuda").bfloat16()
    ops.grouped_gemm_rows(X, W13, off_t, Act, epilogue=_lib.LZ_EPI_SWIGLU, aux=H)
    B2 = (torch.randn(G, K, F, device="cuda") / K ** 0.5).bfloat16()
    dH = torch.empty(rows, 2 * F, device="cuda").bfloat16()
    ops.grouped_gemm_rows(X, B2, off_t, dH, b_major=_lib.LZ_MN_MAJOR,
                          epilogue=_lib.LZ_EPI_DSWIGLU, aux=H)
    torch.cuda.synchronize()
    Hrows = ops.aux_rows(H)   # private blocked layout -> row-major view
    for g in range(G):
        sl = slice(off[g], off[g + 1])
        xg = X[sl].float()
        gate = (xg @ w1[g].float().t()).requires_grad_(True)
        up = (xg @ w3[g].float().t()).requires_grad_(True)
        act = torch.nn.functional.silu(gate) * up
        dA = xg @ B2[g].float()
        act.backward(dA)
        Hi = Hrows[sl].view(-1, F // 128, 2, 128)
        S, Q = Hi[:, :, 0].reshape(-1, F), Hi[:, :, 1].reshape(-1, F)
        sg = torch.sigmoid(gate.detach())
        _close(Act[sl], act.detach(), rtol=2e-2)
        _close(S, torch.nn.functional.silu(gate.detach()), rtol=2e-2)
        _close(Q, up.detach() * sg * (1 + gate.detach() * (1 - sg)), rtol=2e-2)
        dHi = dH[sl].view(-1, F // 128, 2, 128)
        _close(dHi[:, :, 0].reshape(-1, F), gate.grad, rtol=3e-2)
        _close(dHi[:, :, 1].reshape(-1, F), up.grad, rtol=3e-2)
