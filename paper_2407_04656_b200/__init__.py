"""B200-native (sm_100a) Lazarus MoE-layer hot path (arXiv 2407.04656).

gating -> replica-split planning -> pack -> [all-to-all] -> grouped expert FFN
-> [all-to-all] -> combine, fwd + bwd + replica-group gradient sync, driven by the
host-side placement plans of the reference package.  See DESIGN.md.

Modules: ``dispatch`` (drop-in for flexep.dispatch), ``placement`` (host plan
producer), ``ops`` (thin wrappers over the C-ABI kernels), ``layer`` (MoELayer),
``comm`` (NCCL plumbing), ``elastic`` (re-plan after rank failure).
"""

__version__ = "0.1.0"
