"""B200-native (sm_100a) Lazarus MoE-layer hot path (arXiv 2407.04656).

gating -> replica-split planning -> pack -> [all-to-all] -> grouped expert FFN
-> [all-to-all] -> combine, fwd + bwd + replica-group gradient sync, driven by the
host-side placement plans of the reference package.  See DESIGN.md.

Modules: ``dispatch`` (drop-in for flexep.dispatch), ``placement`` (host plan
producer), ``cost`` (the reference's cost model on the device plan), ``ops`` (thin
wrappers over the C-ABI kernels), ``layer`` (MoELayer), ``comm`` (NCCL plumbing and the
process fabric), ``loopback`` (N ranks on one GPU), ``elastic`` (re-plan after rank
failure), ``rebalance`` (periodic load-driven re-placement), ``reliability``.
"""

__version__ = "0.1.0"
