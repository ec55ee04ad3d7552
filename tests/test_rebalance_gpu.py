"""Device routing-history window (lz_load_record) and the periodic rebalance at N = 1."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def test_load_window_ring():
    from paper_2407_04656_b200.rebalance import LoadWindow
    E, N, W = 8, 3, 4
    win = LoadWindow(E, W)
    assert win.loads() is None
    g = torch.Generator().manual_seed(0)
    hist = []
    for step in range(7):
        T = torch.randint(0, 1000, (E, N), generator=g, dtype=torch.int32)
        win.record(T.cuda())
        hist.append(T.sum(1).tolist())
        n = min(step + 1, W)
        want = [sum(h[e] for h in hist[-n:]) // n for e in range(E)]
        assert win.loads() == tuple(want)
    assert win.steps() == 7


def test_load_window_graph_replay():
    """The record is device-only (position advanced on the GPU): replays of a captured
    forward keep filling the ring."""
    from paper_2407_04656_b200.rebalance import LoadWindow
    E, N = 16, 1
    win = LoadWindow(E, 8)
    T = torch.arange(E, dtype=torch.int32, device="cuda").view(E, N).contiguous()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        win.record(T)
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        win.record(T)
    for _ in range(5):
        graph.replay()
    torch.cuda.synchronize()
    assert win.steps() == 6
    assert win.loads() == tuple(range(E))


def test_rebalance_layer_n1():
    from paper_2407_04656_b200.layer import MoELayer, zipf_router_bias
    from paper_2407_04656_b200.rebalance import Rebalancer
    E, d, dff, k, Tn = 8, 512, 1024, 2, 2048
    layer = MoELayer(d, dff, E, k, seed=4, router_bias=zipf_router_bias(E, 0.0))
    rb = Rebalancer([layer], slots=3 * E, interval=3)
    layer.bg.data.copy_(zipf_router_bias(E, 2.0, seed=3).cuda())
    torch.manual_seed(0)
    x = torch.randn(Tn, d, device="cuda").bfloat16()
    hists = []
    with torch.no_grad():
        before = layer(x)
        hists.append(layer.last_plan.D.sum(dim=(0, 2)))
        assert rb.step() is None
        layer(x)
        assert rb.step() is None
        layer(x)
        rep = rb.step()
        after = layer(x)
    assert rep is not None and rep["changed"], rep
    # loads = the integer mean of the three recorded steps (identical batches here)
    assert list(rep["loads"][0]) == hists[0].tolist()
    hot = max(range(E), key=lambda e: rep["loads"][0][e])
    assert layer.R[hot][0] == max(r[0] for r in layer.R) and layer.R[hot][0] > 1
    # replicas share one weight copy: the new plan changes nothing numerically
    assert torch.equal(before, after)
