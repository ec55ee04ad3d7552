"""Golden vectors for the reference's cost model of this path:
``adaptive_layer_cost`` (simulator.py:198-219) and the adaptive ``step_time_model``
(simulator.py:248-266), produced by running the REFERENCE itself on placement plans the
reference builds (allocate_replicas + build_mro_plan).  Build container only:

    python tests/golden/make_cost_golden.py      -> tests/golden/cost_golden.json
"""

from __future__ import annotations

import json
import os
import random
import sys

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    sys.path.insert(0, REF)
    from flexep.allocation import allocate_replicas
    from flexep.core import ClusterSpec, CostModel
    from flexep.dispatch import ReplicaMatrix
    from flexep.placement import build_mro_plan
    from flexep.simulator import adaptive_layer_cost, step_time_model

    rng = random.Random(0xC057)
    cases = []
    shapes = [(6, 3, 4, 2), (8, 4, 4, 2), (16, 8, 6, 2), (16, 4, 12, 2), (64, 8, 32, 2),
              (8, 2, 12, 2), (16, 6, 8, 2), (32, 8, 12, 1), (64, 4, 64, 2)]
    for E, n, c, f in shapes:
        for rep in range(6):
            s = rng.choice([0.0, 0.8, 1.2, 2.5])
            total = rng.choice([4096, 65536 * n * 2, 1_000_003])
            w = [int(1e6 / (e + 1) ** s) + 1 for e in range(E)]
            rng.shuffle(w)
            wsum = sum(w)
            tokens = [total * x // wsum for x in w]
            tokens[0] += total - sum(tokens)
            spec = ClusterSpec(n, c, f)
            plan = build_mro_plan(allocate_replicas(tokens, spec), spec)
            R = [list(r) for r in ReplicaMatrix.from_plan(plan).counts]
            mx, cross = adaptive_layer_cost(plan, tokens, n)
            cm = CostModel()
            st = step_time_model("adaptive", {0: plan, 1: plan}, {0: tokens, 1: tokens[::-1]},
                                 cm, n)
            cases.append({"E": E, "n": n, "c": c, "f": f, "tokens": tokens, "R": R,
                          "max_node": mx, "cross": cross, "step_time": st,
                          "cost_model": [cm.per_token_compute_s, cm.per_token_comm_s,
                                         cm.step_overhead_s]})
    with open(os.path.join(HERE, "cost_golden.json"), "w") as f:
        json.dump({"cases": cases}, f, separators=(",", ":"))
    print(len(cases), "cost cases")


if __name__ == "__main__":
    main()
