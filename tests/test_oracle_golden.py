"""Pin the CPU oracle (oracle/dispatch_ref.py) against vectors produced by the
reference itself (tests/golden/make_golden.py).  CPU only."""

import hashlib
import json
import random

import numpy as np
import pytest

from oracle import dispatch_ref as O
from tests.golden.make_golden import gen_fuzz, gen_owner_only


def _digest(obj):
    return hashlib.sha256(json.dumps(obj, sort_keys=True, separators=(",", ":")).encode()).hexdigest()


def test_split_proportionally_vectors(golden):
    for total, w, want in golden["dispatch"]["split"]:
        assert O.split_proportionally(total, w) == want
    with pytest.raises(ValueError):
        O.split_proportionally(3, [0, 0])
    for total, n, want in golden["dispatch"]["split_evenly"]:
        assert O.split_proportionally(total, [1] * n) == want


def test_dispatch_kats(golden):
    for case in golden["dispatch"]["kat"]:
        for i, want in enumerate(case["schedules"]):
            assert O.compute_dispatch_schedule(i, case["T"], case["R"]) == want
    u = golden["dispatch"]["unroutable"]
    with pytest.raises(O.UnroutableTokenError):
        O.compute_dispatch_schedule(0, u["T"], u["R"])


def test_c12_schedule(golden):
    c = golden["dispatch"]["c12"]
    for i, want in enumerate(c["schedules"]):
        assert O.compute_dispatch_schedule(i, c["T"], c["R"]) == want
    assert c["schedules"][0]["D"] == [[3, 0, 0, 0, 0, 0], [3, 0, 0, 0, 0, 0], [0, 0, 1, 2, 0, 0],
                                     [3, 0, 0, 0, 0, 0], [0, 0, 1, 1, 1, 0], [3, 0, 0, 0, 0, 0]]


@pytest.mark.parametrize("name", ["c07", "fa57", "loca1", "d15"])
def test_fuzz_sets_digest(golden, name):
    spec = golden["dispatch"]["fuzz"][name]
    rng = random.Random(spec["seed"])
    res = []
    for _ in range(spec["count"]):
        t, r = gen_fuzz(rng, spec["tmax"]) if spec["gen"] == "fuzz" else gen_owner_only(rng)
        try:
            mats = O.full_dispatch_matrices(t, r)
            scheds = [O.compute_dispatch_schedule(i, t, r) for i in range(len(t[0]))]
            O.simulate_all_to_all(scheds)
            res.append({"T": t, "R": r, "D": mats, "schedules": scheds})
        except O.UnroutableTokenError:
            res.append({"T": t, "R": r, "error": "unroutable"})
    assert res[:len(spec["head"])] == spec["head"]
    assert _digest(res) == spec["digest"]


def test_shuffle_vectors(golden):
    for case in golden["dispatch"]["shuffle_kat"]:
        assert O.build_shuffle_index(case["D"], case["routed"]).tolist() == case["index"]
    for case in golden["dispatch"]["shuffle"]:
        sch = O.compute_dispatch_schedule(case["rank"], case["T"], case["R"])
        idx = O.build_shuffle_index(sch["D"], case["routed"])
        assert idx.tolist() == case["index"]
        inv = O.invert_permutation(idx)
        assert np.array_equal(idx[inv], np.arange(idx.size))


def test_shuffle_validation():
    D = [[3, 0], [0, 2]]
    with pytest.raises(ValueError):
        O.build_shuffle_index(D, [0, 0, 0])
    with pytest.raises(ValueError):
        O.build_shuffle_index(D, [0, 0, 0, 0, 1])
    with pytest.raises(ValueError):
        O.build_shuffle_index(D, [0, 0, 0, 1, 7])


def test_simulate_all_to_all_mismatch():
    s0 = O.compute_dispatch_schedule(0, [[5, 5]], [[1, 0]])
    bad = O.compute_dispatch_schedule(1, [[5, 9]], [[1, 0]])
    with pytest.raises(O.DispatchConsistencyError):
        O.simulate_all_to_all([s0, bad])
    ok = O.simulate_all_to_all([s0, O.compute_dispatch_schedule(1, [[5, 5]], [[1, 0]])])
    assert ok[0][0] == [5, 5] and ok[1][0] == [0, 0]


def test_gather_load_matrix():
    assert O.gather_load_matrix([[3, 1], [0, 4]]) == ((3, 0), (1, 4))
    with pytest.raises(ValueError):
        O.gather_load_matrix([[1, 2], [3]])
