"""Recovery probability (reference reliability.py) -- host parts on CPU, the GPU
enumeration (lz_recovery_count) against the reference's exact Fractions."""

from fractions import Fraction
from itertools import combinations

import pytest

from paper_2407_04656_b200 import placement as P
from paper_2407_04656_b200 import reliability as R


def _plan(case):
    spec = P.ClusterSpec(case["n"], case["c"], case["f"])
    alloc = P.allocate_replicas(case["loads"], spec)
    plan = P.build_mro_plan(alloc, spec)
    assert [list(r) for r in plan.slots] == case["slots"]
    return spec, alloc, plan


def test_closed_form_matches_reference(golden):
    for case in golden["placement"]["recovery"]:
        spec, alloc, _ = _plan(case)
        for r, (num, den) in case["closed_form"].items():
            assert R.recovery_probability_closed_form(alloc, spec, int(r)) == Fraction(num, den)


def test_is_recoverable_and_argument_errors(golden):
    case = golden["placement"]["recovery"][0]
    _, _, plan = _plan(case)
    n = plan.n_nodes
    assert R.is_recoverable(plan, range(n))
    assert not R.is_recoverable(plan, [])
    with pytest.raises(ValueError):
        R.is_recoverable(plan, [n])
    with pytest.raises(ValueError):
        R.recovery_probability_exact(plan, n + 1)
    with pytest.raises(R.EnumerationCapError):
        R.recovery_probability_exact(plan, n // 2, enumeration_cap=1)


@pytest.mark.gpu
def test_exact_matches_reference(golden):
    for case in golden["placement"]["recovery"]:
        _, _, plan = _plan(case)
        for k, (num, den) in case["exact"].items():
            assert R.recovery_probability_exact(plan, int(k)) == Fraction(num, den), (case, k)


@pytest.mark.gpu
def test_exact_beyond_reference_cap():
    """N = 40 nodes, k = 10 failures: C(40, 10) = 847,660,528 failed sets (the reference
    refuses above 10^6); cross-checked against an independent host count over the
    failed sets that hit every holder of some expert (inclusion-exclusion)."""
    spec = P.ClusterSpec(40, 2, 2)
    alloc = P.allocate_replicas([1] * 16 + [9, 7, 5, 3], spec)
    plan = P.build_mro_plan(alloc, spec)
    k = 10
    got = R.recovery_probability_exact(plan, k, enumeration_cap=10**12)
    holders = [frozenset(j for j, cs in enumerate(plan.col_sets) if e in cs)
               for e in range(plan.n_experts)]
    import math
    bad = 0
    # inclusion-exclusion over sets of experts whose holders all fail
    hs = sorted(set(holders), key=len)
    for m in range(1, len(hs) + 1):
        for sub in combinations(hs, m):
            u = frozenset().union(*sub)
            if len(u) <= k:
                bad += (-1) ** (m + 1) * math.comb(40 - len(u), k - len(u))
    total = math.comb(40, k)
    assert got == Fraction(total - bad, total)
