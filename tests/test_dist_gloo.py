"""Multi-rank host logic on CPU (gloo, world_size 2 and 3): the load all-gather, the
padding-free all-to-all-v in the reference's send order, the regroup into the padded
expert-major receive layout, and the in-place replica-group gradient all-reduce.
Device kernels are replaced by the oracle (the layout contract is what is tested)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import dispatch_ref as O
from paper_2407_04656_b200 import comm
from paper_2407_04656_b200.elastic import replan, transfer_schedule
from paper_2407_04656_b200.placement import plan_for_loads, replica_matrix


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, n, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=n)
    try:
        E, k, d, P_tok = 6, 2, 8, 40  # noqa: F841
        rng = np.random.default_rng(100 + rank)
        routed = rng.choice(E, size=P_tok * k, p=np.array([.4, .2, .15, .1, .1, .05])).astype(np.int32)
        hist = torch.from_numpy(np.bincount(routed, minlength=E).astype(np.int32))
        # (1) load all-gather -> T [E, N]
        T = comm.allgather_hist(hist)
        allh = [torch.empty_like(hist) for _ in range(n)]
        dist.all_gather(allh, hist)
        assert torch.equal(T, torch.stack(allh, 1))
        T_list = T.tolist()
        R = replica_matrix(plan_for_loads(T.sum(1).tolist(), n, 4, 2))
        sch = O.compute_dispatch_schedule(rank, T_list, R)
        D_all = np.array(O.full_dispatch_matrices(T_list, R))
        # (2) pack in the reference send order, all-to-all-v
        x = torch.arange(P_tok, dtype=torch.float32).repeat_interleave(d).view(P_tok, d) + 1000 * rank
        index = O.build_shuffle_index(sch["D"], routed)          # send slot -> assignment
        send = x[torch.from_numpy(index // k)]
        recv_counts = [int(D_all[j, :, rank].sum()) for j in range(n)]
        stage = torch.empty(sum(recv_counts), d)
        comm.all_to_all_rows(stage, send, recv_counts, sch["s"])
        # (3) regroup into the expert-major, 4-row padded layout; check every row landed at
        # the destination row the sender computed for it (source order kept)
        m, pad_off, src_off = O.recv_layout(D_all, rank, align=4)
        X = torch.full((int(pad_off[-1]), d), -1.0)
        st = 0
        for i in range(n):
            for e in range(E):
                c = int(D_all[i, e, rank])
                X[src_off[e][i]:src_off[e][i] + c] = stage[st:st + c]
                st += c
        # every sender's rows: the tokens it routed to e that the plan gave to this rank
        for i in range(n):
            rng_i = np.random.default_rng(100 + i)
            r_i = rng_i.choice(E, size=P_tok * k, p=np.array([.4, .2, .15, .1, .1, .05]))
            idx_i = O.build_shuffle_index(O.compute_dispatch_schedule(i, T_list, R)["D"], r_i)
            base = sum(int(D_all[i, :, j].sum()) for j in range(rank))
            for e in range(E):
                pre = sum(int(D_all[i, ee, rank]) for ee in range(e))
                c = int(D_all[i, e, rank])
                toks = idx_i[base + pre: base + pre + c] // k
                want = torch.from_numpy(toks).float().repeat_interleave(d).view(c, d) + 1000 * i
                assert torch.equal(X[src_off[e][i]:src_off[e][i] + c], want)
        # (4) replica-group all-reduce in place (experts sharing an owner set share a group);
        # a hand-made R where the same owner set maps to different local positions per rank
        if n == 3:
            R = [[1, 1, 0], [0, 1, 1], [1, 1, 0], [1, 0, 1], [1, 1, 0], [0, 1, 1]]
        groups = comm.ReplicaGroups(R)
        local = [e for e in range(E) if R[e][rank] > 0]
        g1 = torch.stack([torch.full((3, 2), float(rank + 1) * (e + 1)) for e in local])
        g2 = torch.stack([torch.full((2,), float(rank + 1)) for e in local])
        groups.allreduce([g1, g2], local)
        for p, e in enumerate(local):
            owners = [j for j in range(n) if R[e][j] > 0]
            want = sum(j + 1 for j in owners)
            assert torch.allclose(g1[p], torch.full((3, 2), float(want * (e + 1))))
            assert torch.allclose(g2[p], torch.full((2,), float(want)))
        # the same sums issued as two expert-id ranges (the split last weight-gradient
        # all-reduce of the backward tail): every owner set's members issue the same sequence
        h1 = torch.stack([torch.full((3, 2), float(rank + 1) * (e + 1)) for e in local])
        works = groups.allreduce_async([h1], local, (0, E // 2))
        works += groups.allreduce_async([h1], local, (E // 2, E))
        for w in works:
            w.wait()
        assert torch.equal(h1, g1)
        q.put((rank, "ok"))
    except Exception as exc:  # surface to the parent
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [2, 3])
def test_multirank_host_path_gloo(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, n, port, q)) for r in range(n)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(n)]
    for p in procs:
        p.join(timeout=60)
    for rank, msg in res:
        assert msg == "ok", f"rank {rank}:\n{msg}"


def test_elastic_replan_and_transfers():
    """8 -> 6 -> 4 host re-plan (reference recipe) and the state-transfer schedule."""
    E, c = 16, 6
    loads = [int(1000 * (1 + e) ** -1.2) + 10 for e in range(E)]
    plan8 = plan_for_loads(loads, 8, c, 2)
    holdings = {v: set(plan8.column(v)) for v in range(8)}
    for live in ([0, 1, 2, 4, 5, 7], [0, 2, 4, 7]):
        held = {v: holdings[v] for v in live}
        plan, order, R = replan(loads, live, held, c, 2)
        assert sorted(order) == sorted(live)
        assert all(sum(row) > 0 for row in R)                       # every expert hosted
        transfers, orphans = transfer_schedule(R, sorted(live), held)
        for e, src, dst in transfers:
            assert e in held[src] and e not in held[dst] and src != dst
        newly = {(e, v) for r, v in enumerate(sorted(live)) for e in range(E)
                 if R[e][r] > 0 and e not in held[v]}
        assert newly == {(e, dst) for e, _, dst in transfers} | {(e, v) for e, v in orphans}
        holdings = {v: {e for e in range(E) if R[e][r] > 0} for r, v in enumerate(sorted(live))}


def _migrate_worker(rank, n, port, q):
    """Two CPU ranks with MoELayer objects (no kernels run: construction and set_plan are
    host/tensor work): rank 1 newly hosts expert 0, whose weights and Adam moments must
    arrive from rank 0 over gloo send/recv, and the optimizer must follow the new
    Parameters (elastic.exchange_expert_state + remap_optimizer)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=n)
    try:
        from paper_2407_04656_b200.elastic import exchange_expert_state, remap_optimizer
        from paper_2407_04656_b200.layer import MoELayer
        E, d, dff = 4, 256, 256
        R0 = [[1, 0], [1, 1], [0, 1], [0, 1]]       # expert 0 only on rank 0
        layer = MoELayer(d, dff, E, 2, replicas=R0, group=dist.group.WORLD, device="cpu",
                         seed=7, activation="swiglu")
        opt = torch.optim.Adam([layer.w1, layer.w2], lr=1e-2)
        layer.w1.grad = torch.full_like(layer.w1, 0.5 + rank)
        layer.w2.grad = torch.full_like(layer.w2, -0.25)
        opt.step()
        before = {e: [t.clone() for t in ts] for e, ts in
                  __import__("paper_2407_04656_b200.elastic", fromlist=["x"])
                  .expert_slices(layer, opt).items()}
        R1 = [[1, 1], [1, 1], [0, 1], [0, 1]]       # rank 1 now also hosts expert 0
        slices = exchange_expert_state([layer], [((0, 0), 0, 1)], rank, {0: 0, 1: 1},
                                       dist.group.WORLD, [opt])[0]
        info = layer.set_plan(R1, weights={e: (v[0], v[1]) for e, v in slices.items()})
        remap_optimizer(opt, layer, info, slices)
        assert opt.param_groups[0]["params"][0] is layer.w1
        got = {e: [layer.w1.data[p], layer.w2.data[p],
                   opt.state[layer.w1]["exp_avg"][p], opt.state[layer.w1]["exp_avg_sq"][p],
                   opt.state[layer.w2]["exp_avg"][p], opt.state[layer.w2]["exp_avg_sq"][p]]
               for p, e in enumerate(layer.local_ids)}
        # send rank 0's expert-0 state to the test for comparison with rank 1's copy
        q.put((rank, {e: [t.tolist() for t in v] for e, v in got.items() if e == 0},
               {e: [t.tolist() for t in v] for e, v in before.items() if e == 0},
               layer.local_ids, int(opt.state[layer.w1]["step"])))
        opt.step()   # the optimizer keeps stepping the live parameters
    except Exception as exc:  # pragma: no cover - surfaced by the parent
        q.put((rank, repr(exc), None, None, None))
        raise
    finally:
        dist.destroy_process_group()


def test_expert_state_migration_moves_optimizer_state():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_migrate_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, got, before, ids, step = q.get(timeout=300)
        assert not isinstance(got, str), got
        res[r] = (got, before, ids, step)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[1][2] == [0, 1, 2, 3] and res[0][2] == [0, 1]
    src = res[0][1][0]     # rank 0's expert 0 before the move: w1, w2, 4 moments
    dst = res[1][0][0]     # rank 1's expert 0 after the move
    assert len(src) == 6 and src == dst
    assert res[1][3] == 1


def _fabric_worker(rank, n, port, q):
    """comm.ProcessFabric serving the layer's exchange requests over gloo (CPU tensors):
    HIST (all-gather), A2A (row all-to-all-v), ALLREDUCE, EXPERT_AR (replica groups), WAIT,
    SYNC -- the same request stream the MoE layer's per-rank step yields."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=n)
    try:
        fab = comm.ProcessFabric(None)
        assert (fab.rank, fab.world) == (rank, n)
        hist = torch.tensor([rank, 10 + rank, 20 + rank], dtype=torch.int32)
        T = fab.serve((comm.HIST, hist))
        assert T.tolist() == [[j + 10 * e for j in range(n)] for e in range(3)]   # T[e][j]
        # A2A: rank i sends (j + 1) rows to rank j, row value 100 i + j
        send_sizes = [j + 1 for j in range(n)]
        recv_counts = [rank + 1] * n
        inp = torch.cat([torch.full((j + 1, 4), float(100 * rank + j)) for j in range(n)])
        out = torch.empty(sum(recv_counts), 4)
        fab.serve((comm.A2A, out, inp, recv_counts, send_sizes))
        want = torch.cat([torch.full((rank + 1, 4), float(100 * i + rank)) for i in range(n)])
        assert torch.equal(out, want)
        flat = torch.full((5,), float(rank + 1))
        fab.serve((comm.ALLREDUCE, flat))
        assert torch.equal(flat, torch.full((5,), float(sum(range(1, n + 1)))))

        class L:   # the two attributes EXPERT_AR reads from the layer
            pass
        R = [[1] * n, [1 if j == 0 else 0 for j in range(n)], [1] * n]
        lay = L()
        lay.local_ids = [e for e in range(3) if R[e][rank] > 0]
        lay.replica_groups = fab.replica_groups(R)
        g = torch.stack([torch.full((2, 2), float(rank + 1)) for _ in lay.local_ids])
        works = fab.serve((comm.EXPERT_AR, lay, [g]))
        fab.serve((comm.WAIT, works))
        for p, e in enumerate(lay.local_ids):
            owners = [j for j in range(n) if R[e][j] > 0]
            assert torch.equal(g[p], torch.full((2, 2), float(sum(j + 1 for j in owners))))
        assert fab.serve((comm.SYNC,)) is None
        q.put((rank, "ok"))
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [2, 3])
def test_process_fabric_serves_layer_requests(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_fabric_worker, args=(r, n, port, q)) for r in range(n)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(n)]
    for p in procs:
        p.join(timeout=60)
    for rank, msg in res:
        assert msg == "ok", f"rank {rank}:\n{msg}"


def test_loopback_world_serves_requests_on_cpu_tensors():
    """LoopbackWorld's request serving (HIST stack, A2A copies, ALLREDUCE, EXPERT_AR owner-
    set sums, lockstep divergence detection, lost-rank collectives) on CPU tensors."""
    from paper_2407_04656_b200 import loopback as LB
    world = LB.LoopbackWorld.__new__(LB.LoopbackWorld)   # no CUDA streams needed here
    world.n, world.lost, world.requests, world._alloc = 3, set(), 0, None
    hs = {r: torch.tensor([r, r + 5], dtype=torch.int32) for r in range(3)}
    T = world.serve(comm.HIST, {r: (comm.HIST, hs[r]) for r in range(3)})[0]
    assert T.tolist() == [[0, 1, 2], [5, 6, 7]]
    outs = {r: torch.empty(3 * (r + 1), 2) for r in range(3)}
    inps = {r: torch.cat([torch.full((j + 1, 2), float(10 * r + j)) for j in range(3)])
            for r in range(3)}
    world.serve(comm.A2A, {r: (comm.A2A, outs[r], inps[r], [r + 1] * 3, [1, 2, 3])
                           for r in range(3)})
    for r in range(3):
        want = torch.cat([torch.full((r + 1, 2), float(10 * i + r)) for i in range(3)])
        assert torch.equal(outs[r], want)
    flats = {r: torch.full((3,), float(r)) for r in range(3)}
    world.serve(comm.ALLREDUCE, {r: (comm.ALLREDUCE, flats[r]) for r in range(3)})
    assert all(torch.equal(f, torch.full((3,), 3.0)) for f in flats.values())

    class L:
        E = 2
    layers = {}
    for r in range(3):
        layers[r] = L()
        layers[r].local_ids = [0, 1] if r < 2 else [1]
    grads = {r: torch.stack([torch.full((2,), float(r + 1))] * len(layers[r].local_ids))
             for r in range(3)}
    world.serve(comm.EXPERT_AR, {r: (comm.EXPERT_AR, layers[r], [grads[r]]) for r in range(3)})
    assert grads[0][0].tolist() == [3.0, 3.0] and grads[1][0].tolist() == [3.0, 3.0]   # e0: 0,1
    assert grads[0][1].tolist() == [6.0, 6.0] and grads[2][0].tolist() == [6.0, 6.0]   # e1: all

    def gen(kinds):
        for kd in kinds:
            yield (kd,)
        return "done"
    assert world.run([gen([comm.SYNC, comm.SYNC]) for _ in range(3)]) == ["done"] * 3
    with pytest.raises(RuntimeError, match="diverged"):
        world.run([gen([comm.SYNC]), gen([comm.WAIT]), gen([comm.SYNC])])
    world.lost = {2}
    with pytest.raises(LB.PeerLostError):
        world.serve(comm.HIST, {r: (comm.HIST, hs[r]) for r in range(2)})
