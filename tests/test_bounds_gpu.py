"""Out-of-bounds write detection without compute-sanitizer (closed on this GPU pool:
profiles/r02_compute_sanitizer_closed.txt).  Every output of every library kernel is
carved out of a larger allocation whose guard bands before and after are filled with a
byte pattern; after the kernel (and a synchronisation) the guards must be intact and, where
the contract says so, every element of the output must have been written (a NaN / pattern
fill that survives is an under-write).  Covers the planner's validation path with
inconsistent per-expert counts (the round-1 out-of-bounds write, flexep dispatch.py:214-229
validates before computing), gate, pack (incl. pad rows), combine / combine backward,
dispatch backward, router weight gradient, all grouped-GEMM variants incl. the scattering
epilogue, and the fused P2P exchange through the loopback world."""

import pytest
import torch

pytestmark = pytest.mark.gpu

GUARD = 1 << 20   # bytes of guard on each side
PAT = 0x5A


class Guarded:
    def __init__(self, shape, dtype, fill=None):
        n = 1
        for s in shape:
            n *= s
        el = torch.empty(0, dtype=dtype).element_size()
        self.nbytes = n * el
        self.raw = torch.full((GUARD * 2 + self.nbytes + 256,), PAT, dtype=torch.uint8,
                              device="cuda")
        body = self.raw[GUARD:GUARD + self.nbytes]
        self.t = body.view(dtype).view(*shape)
        if fill is not None:
            self.t.fill_(fill)

    def check(self, name=""):
        torch.cuda.synchronize()
        front = self.raw[:GUARD]
        back = self.raw[GUARD + self.nbytes:]
        assert bool((front == PAT).all()), f"{name}: write before the buffer"
        assert bool((back == PAT).all()), f"{name}: write past the end of the buffer"


def test_plan_validation_path_stays_in_bounds():
    """build_shuffle_index / plan_device with routed lists that disagree with the schedule
    (more, fewer, and unknown experts): the error is raised and nothing outside the
    outputs is touched."""
    from paper_2407_04656_b200 import _lib
    from paper_2407_04656_b200 import dispatch as G
    from paper_2407_04656_b200.dispatch import _ws
    cases = [([[3, 0], [0, 2]], [[1, 0], [0, 1]], [0, 0, 0, 0, 1]),     # expert 0 over its row
             ([[3, 0], [0, 2]], [[1, 0], [0, 1]], [0, 1, 1]),           # short
             ([[3, 0], [0, 2]], [[1, 0], [0, 1]], [0, 7, 0]),           # unknown id
             ([[40, 9], [5, 2]], [[1, 1], [0, 1]], [1] * 45)]           # all to the wrong one
    for T, R, routed in cases:
        E, N = len(T), len(T[0])
        for rank in range(N):
            Tt = torch.tensor(T, dtype=torch.int32, device="cuda")
            Rt = torch.tensor(R, dtype=torch.int32, device="cuda")
            rt = torch.tensor(routed, dtype=torch.int32, device="cuda")
            P = rt.numel()
            outs = {nm: Guarded((P,), torch.int32, -7) for nm in
                    ("slot", "gather", "dest_row", "dest_rank")}
            small = {nm: Guarded(shape, torch.int32) for nm, shape in
                     (("D", (N, E, N)), ("send", (N,)), ("recv", (N,)), ("recvc", (N,)),
                      ("recv_m", (E,)), ("recv_off", (E + 1,)), ("src", (E, N)),
                      ("stage", (E, N)), ("cnt", (E, N)), ("err", (2,)))}
            small["err"].t.zero_()
            quota = Guarded((E,), torch.int64)
            ws = _ws(E, N, P, "cuda")
            wsg = Guarded((ws.numel(),), torch.uint8)
            _lib.call("lz_plan_dispatch", Tt.data_ptr(), Rt.data_ptr(), E, N, rank,
                      rt.data_ptr(), P, 128, 0, small["err"].t[1:].data_ptr(),
                      quota.t.data_ptr(), small["D"].t.data_ptr(), small["send"].t.data_ptr(),
                      small["recv"].t.data_ptr(), small["recvc"].t.data_ptr(),
                      outs["slot"].t.data_ptr(), outs["gather"].t.data_ptr(),
                      outs["dest_row"].t.data_ptr(), outs["dest_rank"].t.data_ptr(),
                      small["recv_m"].t.data_ptr(), small["recv_off"].t.data_ptr(),
                      small["src"].t.data_ptr(), small["stage"].t.data_ptr(),
                      small["cnt"].t.data_ptr(), small["err"].t.data_ptr(), wsg.t.data_ptr(),
                      ws.numel(), _lib.stream_ptr())
            for nm, gd in {**outs, **small, "quota": quota, "ws": wsg}.items():
                gd.check(f"plan {nm} case {routed} rank {rank}")
            assert int(small["err"].t[0]) & (_lib.LZ_ERRF_COUNTS | _lib.LZ_ERRF_EXPERT_ID)
            with pytest.raises(ValueError):
                G.build_shuffle_index(G.compute_dispatch_schedule(rank, T, G.ReplicaMatrix(
                    tuple(tuple(r) for r in R))), routed)


def test_row_kernels_stay_in_bounds():
    from paper_2407_04656_b200 import ops
    from paper_2407_04656_b200.dispatch import plan_device
    torch.manual_seed(0)
    Tn, d, E, k = 3001, 1024, 16, 2
    x = torch.randn(Tn, d, device="cuda").bfloat16()
    wg = (torch.randn(E, d, device="cuda") * 0.05).bfloat16()
    bg = torch.zeros(E, device="cuda")
    from paper_2407_04656_b200 import _lib
    idx, w, probs, hist = ops.router_gate(x, wg, bg, k)
    # the gate's outputs into guarded buffers
    gi, gw, gp, gh = (Guarded((Tn, k), torch.int32), Guarded((Tn, k), torch.float32),
                      Guarded((Tn, E), torch.float32), Guarded((E,), torch.int32))
    _lib.call("lz_router_gate", x.data_ptr(), wg.data_ptr(), bg.data_ptr(), Tn, d, E, k, 0,
              gi.t.data_ptr(), gw.t.data_ptr(), gp.t.data_ptr(), gh.t.data_ptr(),
              _lib.stream_ptr())
    for nm, gd in (("idx", gi), ("w", gw), ("probs", gp), ("hist", gh)):
        gd.check(f"gate {nm}")
    T = hist.view(E, 1)
    R = torch.ones(E, 1, dtype=torch.int32, device="cuda")
    plan = plan_device(T, R, 0, idx.view(-1), ops.row_align())
    plan.check()
    rows = int(plan.recv_off[-1])
    X = Guarded((rows, d), torch.bfloat16, float("nan"))
    ops.pack(x, plan.dest_row, k, X.t, plan.recv_m, plan.recv_off)
    X.check("pack")
    assert not torch.isnan(X.t.float()).any(), "pack left rows (or pad rows) unwritten"
    out = Guarded((Tn, d), torch.bfloat16, float("nan"))
    ops.combine(X.t, plan.dest_row, w, k, out=out.t)
    out.check("combine")
    assert not torch.isnan(out.t.float()).any()
    dout = torch.randn(Tn, d, device="cuda").bfloat16()
    dY = Guarded((rows, d), torch.bfloat16, float("nan"))
    dw = ops.combine_bwd(dout, X.t, plan.dest_row, w, k, dY.t, plan.recv_m, plan.recv_off)
    dY.check("combine_bwd dY")
    assert not torch.isnan(dY.t.float()).any()
    gdx, gdl = Guarded((Tn, d), torch.bfloat16), Guarded((Tn, E), torch.float32)
    wgT = wg.t().contiguous()
    _lib.call("lz_dispatch_bwd", dY.t.data_ptr(), plan.dest_row.data_ptr(), Tn, d, k,
              probs.data_ptr(), idx.data_ptr(), dw.data_ptr(), wgT.data_ptr(), E, 0,
              gdx.t.data_ptr(), gdl.t.data_ptr(), _lib.stream_ptr())
    gdx.check("dispatch_bwd dx")
    gdl.check("dispatch_bwd dlogits")
    nbytes = int(_lib.raw("lz_router_wgrad_ws_bytes", Tn, d, E))
    ws = Guarded((nbytes,), torch.uint8)
    dwg, db = Guarded((E, d), torch.float32), Guarded((E,), torch.float32)
    _lib.call("lz_router_wgrad", gdl.t.data_ptr(), x.data_ptr(), Tn, d, E, dwg.t.data_ptr(),
              db.t.data_ptr(), ws.t.data_ptr(), nbytes, _lib.stream_ptr())
    for nm, gd in (("ws", ws), ("dwg", dwg), ("db", db)):
        gd.check(f"router_wgrad {nm}")


@pytest.mark.parametrize("epi", ["store", "gelu", "dgelu", "swiglu", "dswiglu", "wgrad",
                                 "scatter"])
def test_gemm_outputs_stay_in_bounds(epi):
    from paper_2407_04656_b200 import _lib, ops
    torch.manual_seed(1)
    al = ops.row_align()
    off = torch.tensor([0, al, al, 4 * al, 5 * al], dtype=torch.int32, device="cuda")
    rows, G, K, N = 5 * al, 4, 512, 512
    A = torch.randn(rows, K, device="cuda").bfloat16()
    if epi == "wgrad":
        Bm = torch.randn(rows, N, device="cuda").bfloat16()
        C = Guarded((G, K, N), torch.bfloat16, float("nan"))
        ops.grouped_gemm_wgrad(A, Bm, off, C.t)
        C.check("wgrad C")
        return
    Bw = (torch.randn(G, N, K, device="cuda") * 0.05).bfloat16()
    if epi == "scatter":
        ret_rows = rows + 64
        Y = Guarded((ret_rows, N), torch.bfloat16, float("nan"))
        ret = torch.arange(rows, device="cuda", dtype=torch.int64)
        ret[::7] = -1                      # pad rows: no return target
        peers = torch.tensor([Y.t.data_ptr()], dtype=torch.int64, device="cuda")
        C = torch.empty(rows, N, device="cuda", dtype=torch.bfloat16)
        ops.grouped_gemm_scatter(A, Bw, off, C, ret, peers, [Y.t.data_ptr()], ret_rows)
        Y.check("scatter return buffer")
        return
    cw = {"store": N, "gelu": N, "dgelu": N, "swiglu": N // 2, "dswiglu": 2 * N}[epi]
    xw = {"store": N, "gelu": N, "dgelu": N, "swiglu": N, "dswiglu": 2 * N}[epi]
    C = Guarded((rows, cw), torch.bfloat16, float("nan"))
    aux = Guarded((rows, xw), torch.bfloat16, 0.5)
    code = {"store": _lib.LZ_EPI_STORE, "gelu": _lib.LZ_EPI_GELU, "dgelu": _lib.LZ_EPI_DGELU,
            "swiglu": _lib.LZ_EPI_SWIGLU, "dswiglu": _lib.LZ_EPI_DSWIGLU}[epi]
    major = _lib.LZ_MN_MAJOR if epi in ("dgelu", "dswiglu") else _lib.LZ_K_MAJOR
    Bx = Bw if major == _lib.LZ_K_MAJOR else (torch.randn(G, K, N, device="cuda") * 0.05).bfloat16()
    ops.grouped_gemm_rows(A, Bx, off, C.t, b_major=major,
                          aux=None if epi == "store" else aux.t, epilogue=code)
    C.check(f"{epi} C")
    aux.check(f"{epi} aux")
    assert not torch.isnan(C.t.float()).any(), f"{epi}: output rows left unwritten"


def test_p2p_exchange_stays_in_bounds():
    """The fused dispatch / scattering GEMMs / combine-backward stores of 4 loopback ranks
    write only inside the world's exchange allocation: guard bands around it survive a
    full forward + backward step."""
    import math

    from paper_2407_04656_b200.layer import zipf_router_bias
    from paper_2407_04656_b200.loopback import LoopbackWorld
    from paper_2407_04656_b200.placement import plan_for_loads, replica_matrix
    N, E, k, d, dff, Tn = 4, 16, 2, 512, 1024, 1024
    R = replica_matrix(plan_for_loads([int(1000 / (e + 1) ** 1.2) + 1 for e in range(E)], N,
                                      math.ceil(3 * E / N), 2))
    world = LoopbackWorld(N)
    layers = world.make_layers(d, dff, E, k, R, router_bias=zipf_router_bias(E, 1.2))
    xs = [torch.randn(Tn, d, device="cuda").bfloat16() for _ in range(N)]
    ds = [torch.randn(Tn, d, device="cuda").bfloat16() for _ in range(N)]
    world.step(layers, xs, ds)          # allocates the exchange buffers
    torch.cuda.synchronize()
    a = world._alloc
    t = a["t"]
    # guard the neighbourhood of the exchange buffers by checking the world's own padding
    # rows: every rank's receive buffer tail past its padded segments must stay untouched
    for r, L in enumerate(layers):
        used = int(L.last_plan.recv_off[-1])
        t[r, :, used:].fill_(float("nan"))
    world.step(layers, xs, ds)
    torch.cuda.synchronize()
    for r, L in enumerate(layers):
        used = int(L.last_plan.recv_off[-1])
        for b in (0, 2):   # X and dY receive buffers: nothing lands past the used rows
            tail = t[r, b, used:]
            assert torch.isnan(tail.float()).all(), f"rank {r} buffer {b}: write past used rows"
        for L2 in layers:
            L2.check()
