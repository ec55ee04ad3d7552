"""Host plan producer vs the reference's own outputs (tests/golden/placement_golden.json)."""

import pytest

from paper_2407_04656_b200 import placement as P


def test_plans_match_reference(golden):
    for case in golden["placement"]["plans"]:
        spec = P.ClusterSpec(case["n"], case["c"], case["f"])
        alloc = P.allocate_replicas(case["loads"], spec)
        assert list(alloc.replicas) == case["replicas"]
        assert list(alloc.sorted_order) == case["sorted_order"]
        assert alloc.f_used == case["f_used"]
        plan = P.build_mro_plan(alloc, spec)
        assert [list(r) for r in plan.slots] == case["slots"]
        assert P.replica_matrix(plan) == case["R"]


def test_from_plan_kat(golden):
    k = golden["placement"]["from_plan_kat"]
    alloc = P.AllocationPlan((2, 4), (0, 1), 2)
    plan = P.build_mro_plan(alloc, P.ClusterSpec(k["n"], k["c"]))
    assert P.replica_matrix(plan) == k["R"] == [[1, 1, 0], [1, 1, 2]]


def test_node_mapping_matches_reference(golden):
    for case in golden["placement"]["node_mapping"]:
        old_cols = list(zip(*case["old_slots"]))
        holdings = {v: set(old_cols[v]) for v in case["live"]}
        new_cols = [set(c) for c in zip(*case["new_slots"])]
        got = P.greedy_node_mapping(holdings, new_cols, case["live"])
        assert [list(a) for a in got] == case["assignment"]


def test_infeasible():
    with pytest.raises(P.InfeasibleError):
        P.allocate_replicas([1] * 10, P.ClusterSpec(2, 4))


def test_replica_matrix_rank_order():
    spec = P.ClusterSpec(3, 2, 1)
    plan = P.build_mro_plan(P.AllocationPlan((2, 4), (0, 1), 1), spec)
    # columns mapped to nodes 7, 2, 5 -> communicator ranks 2, 0, 1
    R = P.replica_matrix(plan, order=[7, 2, 5])
    base = P.replica_matrix(plan)
    for e in range(2):
        assert R[e] == [base[e][1], base[e][2], base[e][0]]
