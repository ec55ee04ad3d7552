"""Row a12: the reference's cost model of this path (simulator.py:198-266).  The oracle
restatement is pinned to golden values the reference produced
(tests/golden/make_cost_golden.py); the device version (cost.py: bit-exact device plan +
two reductions) must reproduce them exactly."""

import json
import os

import pytest

from oracle import dispatch_ref as O

HERE = os.path.dirname(os.path.abspath(__file__))


def _cases():
    with open(os.path.join(HERE, "golden", "cost_golden.json")) as f:
        return json.load(f)["cases"]


def test_oracle_cost_matches_reference_golden():
    for c in _cases():
        assert O.adaptive_layer_cost(c["R"], c["tokens"], c["n"]) == (c["max_node"], c["cross"])
        a, b, o = c["cost_model"]
        st = O.step_time_adaptive({0: c["R"], 1: c["R"]}, {0: c["tokens"], 1: c["tokens"][::-1]},
                                  c["n"], a, b, o)
        assert st == pytest.approx(c["step_time"], rel=1e-12)


@pytest.mark.gpu
def test_device_cost_matches_reference_golden():
    from types import SimpleNamespace

    from paper_2407_04656_b200 import cost
    from paper_2407_04656_b200.dispatch import ReplicaMatrix
    for c in _cases():
        R = ReplicaMatrix(tuple(tuple(r) for r in c["R"]))
        assert cost.adaptive_layer_cost(R, c["tokens"], c["n"]) == (c["max_node"], c["cross"])
        a, b, o = c["cost_model"]
        cm = SimpleNamespace(per_token_compute_s=a, per_token_comm_s=b, step_overhead_s=o)
        st = cost.step_time_model({0: R, 1: R}, {0: c["tokens"], 1: c["tokens"][::-1]}, cm,
                                  c["n"])
        assert st == pytest.approx(c["step_time"], rel=1e-12)


@pytest.mark.gpu
def test_layer_cost_of_live_plan_matches_oracle():
    """The cost terms of a layer's real (non-uniform) plan equal the oracle's on the
    all-gathered T of that step."""
    import torch

    from paper_2407_04656_b200.layer import zipf_router_bias
    from paper_2407_04656_b200.loopback import LoopbackWorld
    from paper_2407_04656_b200.placement import plan_for_loads, replica_matrix
    N, E, k, d, dff, Tn = 4, 16, 2, 256, 256, 2048
    R = replica_matrix(plan_for_loads([int(1000 / (e + 1) ** 1.2) for e in range(E)], N, 12, 2))
    world = LoopbackWorld(N)
    layers = world.make_layers(d, dff, E, k, R, router_bias=zipf_router_bias(E, 1.2))
    xs = [torch.randn(Tn, d, device="cuda").bfloat16() for _ in range(N)]
    world.step(layers, xs)
    D = layers[0].last_plan.D.cpu().numpy()
    T = D.sum(axis=2).T                      # T[e][i] = sum_j D[i][e][j]
    Dref = O.full_dispatch_matrices(T.tolist(), R)
    node = [sum(Dref[i][e][j] for i in range(N) for e in range(E)) for j in range(N)]
    cross = sum(Dref[i][e][j] for i in range(N) for e in range(E) for j in range(N) if i != j)
    for L in layers:
        assert L.layer_cost() == (max(node), cross)
