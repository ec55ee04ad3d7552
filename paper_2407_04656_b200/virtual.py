"""N virtual EP ranks on ONE GPU, exchanging through device memory (SURVEY.md 4.4
"single-GPU multi-rank loopback"; BASELINE config 1: "4 simulated EP ranks").

Every virtual rank owns its token batch and its plan column exactly like a real rank;
the all-gather of the histograms is a device-side stack, and the dispatch / combine use
the same fused P2P kernels as the multi-GPU path (``lz_pack_p2p`` / ``lz_combine_p2p``)
with the per-rank receive buffers as the "peers" -- so the N-rank layouts, destination
rows and kernels are exercised at any N (e.g. 8) on a single device.  Forward only
(config 1 is a forward benchmark); the experts of ALL virtual ranks run through one
grouped tcgen05 GEMM launch per layer GEMM (the ranks' receive regions are laid out back
to back in one buffer).
"""

from __future__ import annotations

import os

import torch

from . import _lib, ops
from .dispatch import plan_device
from .layer import init_expert


class VirtualEP:
    def __init__(self, d_model: int, d_ff: int, n_experts: int, top_k: int, replicas,
                 tokens_per_rank: int, *, seed: int = 0, init_std: float = 0.02,
                 router_bias=None, router_std: float | None = None, device=None,
                 activation: str = "gelu", scatter: bool = False):
        self.d, self.d_ff, self.E, self.k = d_model, d_ff, n_experts, top_k
        self.R = [list(r) for r in replicas]
        self.N = len(self.R[0])
        self.Tn = tokens_per_rank
        self.activation = activation
        dev = torch.device(device) if device is not None else torch.device("cuda")
        self.device = dev
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        self.wg = (torch.randn(n_experts, d_model, generator=g, device=dev) *
                   (init_std if router_std is None else router_std)).bfloat16()
        self.bg = (torch.zeros(n_experts, device=dev) if router_bias is None
                   else torch.as_tensor(router_bias, dtype=torch.float32, device=dev).clone())
        self.R_dev = torch.tensor(self.R, dtype=torch.int32, device=dev)
        # hosted experts per virtual rank, one weight copy per (expert, rank) -- all ranks'
        # copies concatenated so ONE grouped GEMM launch serves every virtual rank
        self.local = [[e for e in range(self.E) if self.R[e][r] > 0] for r in range(self.N)]
        w1, w2, flat = [], [], []
        for r in range(self.N):
            for e in self.local[r]:
                a, b = init_expert(seed, e, d_model, d_ff, init_std, dev, activation)
                w1.append(a)
                w2.append(b)
                flat.append(r * (self.E + 1) + e)
        flat.append((self.N - 1) * (self.E + 1) + self.E)
        self.w1 = torch.stack(w1).contiguous()
        self.w2 = torch.stack(w2).contiguous()
        self.flat = torch.tensor(flat, dtype=torch.long, device=dev)
        # every rank's receive region is packed right after the previous rank's (bases
        # computed on the device from the plans), so the concatenated group offsets are
        # monotonic with no gap rows between ranks
        align = 256
        self.cap = (self.N * tokens_per_rank * top_k + self.N * self.E * (align - 1) + align - 1
                    ) // align * align
        self.X = torch.empty((self.cap, d_model), dtype=torch.bfloat16, device=dev)
        self.Y = torch.empty_like(self.X)
        self._none = torch.empty(0, dtype=torch.int32, device=dev)
        self.last_plans = None
        # the per-rank stages (gate, plan, pack, combine) are a few CTAs each: run the N
        # virtual ranks' chains concurrently on N streams (fork / join; under graph capture
        # they become parallel branches of the graph)
        self.streams = ([torch.cuda.Stream(device=dev) for _ in range(self.N)]
                        if os.environ.get("LZ_VIRTUAL_STREAMS", "1") != "0" else None)
        # scatter mode (the multi-GPU default): the second GEMM's epilogue writes every
        # output row straight back to its source rank's return buffer (row = assignment),
        # through the owner-side return map the dispatch records
        self.scatter = scatter
        if scatter:
            P = tokens_per_rank * top_k
            self.RET = torch.empty(self.cap, dtype=torch.int64, device=dev)
            self.YR = torch.empty((self.N, P, d_model), dtype=torch.bfloat16, device=dev)
            self.ret_host = [self.YR[r].data_ptr() for r in range(self.N)]
            self.peers_ret = torch.tensor(self.ret_host, dtype=torch.int64, device=dev)

    def _per_rank(self, fn):
        """[fn(r) for r in ranks], rank r's launches on stream r (joined before return)."""
        if self.streams is None:
            return [fn(r) for r in range(self.N)]
        main = torch.cuda.current_stream(self.device)
        out = []
        for r, st in enumerate(self.streams):
            st.wait_stream(main)
            with torch.cuda.stream(st):
                out.append(fn(r))
        for st in self.streams:
            main.wait_stream(st)
        return out

    @torch.no_grad()
    def forward(self, xs):
        """xs: list of N [tokens_per_rank, d] bf16 tensors -> list of N outputs."""
        N, E, k, d, d_ff = self.N, self.E, self.k, self.d, self.d_ff
        gates = self._per_rank(lambda r: ops.router_gate(xs[r], self.wg, self.bg, k, probs=False))
        T = torch.stack([gt[3] for gt in gates], dim=1).contiguous()   # all-gather analog
        align = ops.row_align()
        plans = self._per_rank(lambda r: plan_device(T, self.R_dev, r, gates[r][0].view(-1),
                                                     align))
        self.last_plans = plans
        offs = torch.stack([p.recv_off for p in plans]).to(torch.int64)          # [N, E+1]
        base = torch.cumsum(offs[:, E], 0) - offs[:, E]                         # [N]
        row_b = 2 * d
        peers_x = base * row_b + self.X.data_ptr()
        peers_y = base * row_b + self.Y.data_ptr()
        off = (offs + base[:, None]).view(-1).index_select(0, self.flat).to(torch.int32)
        if self.scatter:
            ret_peers = base * 8 + self.RET.data_ptr()
            self.RET.fill_(-1)   # pad rows of every region
        def pack(r):   # every rank scatters its rows into the owners' regions (disjoint)
            # forward only: pad rows are never read back, so they are not zeroed (E = 0)
            if self.scatter:
                ops.pack_p2p_ret(xs[r], plans[r].dest_rank, plans[r].dest_row, k, peers_x, self.X,
                                 self._none, self._none, ret_peers, self.RET, r, plans[r].slot)
            else:
                ops.pack_p2p(xs[r], plans[r].dest_rank, plans[r].dest_row, k, peers_x, self.X,
                             self._none, self._none)
        self._per_rank(pack)
        swi = self.activation == "swiglu"
        H = torch.empty((self.cap, 2 * d_ff if swi else d_ff), dtype=torch.bfloat16,
                        device=self.device)
        A = torch.empty((self.cap, d_ff), dtype=torch.bfloat16, device=self.device)
        ops.grouped_gemm_rows(self.X, self.w1, off, A, aux=H,
                              epilogue=_lib.LZ_EPI_SWIGLU if swi else _lib.LZ_EPI_GELU)
        if self.scatter:
            ops.grouped_gemm_scatter(A, self.w2, off, self.Y, self.RET, self.peers_ret,
                                     self.ret_host, self.YR.shape[1])
            return self._per_rank(lambda r: ops.combine(self.YR[r], plans[r].slot, gates[r][1],
                                                        k))
        ops.grouped_gemm_rows(A, self.w2, off, self.Y)
        return self._per_rank(lambda r: ops.combine_p2p(peers_y, plans[r].dest_rank,
                                                        plans[r].dest_row, gates[r][1], k, d))

    __call__ = forward

    def check(self) -> None:
        for p in self.last_plans or []:
            p.check()
