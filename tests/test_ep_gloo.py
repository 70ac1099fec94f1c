"""The expert-parallel protocol (paper_2510_19366_b200/ep.py) with world size 2
over gloo on CPU: route -> plan -> pack -> all-to-all -> local experts ->
all-to-all back -> combine.  The data-path steps are played by the oracle
(test infrastructure), so this pins the multi-process exchange logic (counts,
splits, ordering, dedup, deterministic combine) against the single-process
oracle layer on the same tokens."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

U32 = 0xFFFFFFFF
S, D, FF, K_MAX = 4, 32, 64, 8


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _data(oracle, E):
    experts = []
    for e in range(E):
        wg, wu, wd = oracle.random_expert(D, FF, 300 + e)
        experts.append((wg / math.sqrt(D), wu / math.sqrt(D), wd / math.sqrt(FF)))
    experts = [tuple(np.ascontiguousarray(a, np.float32) for a in ex) for ex in experts]
    parts = [oracle.random_balanced_partition(FF, S, 400 + e) for e in range(E)]
    wr = oracle.uniform_pm1(7, D * E * S, 1.0 / math.sqrt(D))
    return experts, parts, wr


class OracleEpOps:
    """The ops interface of ep.CudaEpOps, played by the CPU oracle."""

    def __init__(self, oracle, experts, parts, wr, rank, world):
        self.o, self.rank, self.world = oracle, rank, world
        self.ex, self.parts, self.wr = experts, parts, wr
        self.E = len(experts)
        # contiguous sub-expert ranges (ep.py / ep.cu): whole experts or sub-expert granularity
        self.per_rank = self.E * S // world
        self.first_e = self.per_rank * rank // S
        self.last_e = (self.per_rank * (rank + 1) - 1) // S

    def route(self, x, k, kpt):
        xn = x.numpy()
        logits = self.o.router_logits(xn, self.wr, xn.shape[0], D, self.E * S)
        sel, w, _ = self.o.route(logits, k, K_MAX, 1, k_per_token=None if kpt is None else kpt.numpy())
        return torch.from_numpy(sel.view(np.int32).copy()), torch.from_numpy(w)

    def plan(self, sel):
        s = sel.numpy().view(np.uint32)
        self.dest = [sorted({int(g) // self.per_rank for g in row if g != U32}) for row in s]
        counts = [0] * self.world
        for dl in self.dest:
            for r in dl:
                counts[r] += 1
        self.counts = counts
        return counts

    def pack(self, x, sel, w, n_send):
        s = sel.numpy().view(np.uint32)
        wn = w.numpy()
        rows, ssel, sw, self.pos = [], [], [], {}
        for r in range(self.world):  # grouped by rank, tokens ascending
            for t, dl in enumerate(self.dest):
                if r not in dl:
                    continue
                self.pos[(t, r)] = len(rows)
                base = (r * self.per_rank // S) * S  # local ids on rank r
                ids = [(int(g) - base, wn[t, j]) for j, g in enumerate(s[t])
                       if g != U32 and int(g) // self.per_rank == r]
                rows.append(x[t].numpy())
                ssel.append([i for i, _ in ids] + [U32] * (K_MAX - len(ids)))
                sw.append([v for _, v in ids] + [0.0] * (K_MAX - len(ids)))
        assert len(rows) == n_send
        return (torch.from_numpy(np.array(rows, np.float32).reshape(n_send, D)),
                torch.from_numpy(np.array(ssel, np.uint32).reshape(n_send, K_MAX).view(np.int32)),
                torch.from_numpy(np.array(sw, np.float32).reshape(n_send, K_MAX)))

    def experts(self, recv_x, recv_sel, recv_w):
        if recv_x.shape[0] == 0:
            return recv_x.new_empty((0, D))
        lo, hi = self.first_e, self.last_e + 1
        y = self.o.layer_forward(self.ex[lo:hi], self.parts[lo:hi], S,
                                 recv_x.numpy(), recv_sel.numpy().view(np.uint32), recv_w.numpy(), 1)
        return torch.from_numpy(y)

    def combine(self, back, T):
        b = back.numpy()
        y = np.zeros((T, D), np.float32)
        for t, dl in enumerate(self.dest):
            acc = np.zeros(D, np.float32)
            for r in dl:  # ascending rank order
                acc += b[self.pos[(t, r)]]
            y[t] = acc
        return torch.from_numpy(y)


def _worker(rank, world, port, out_dir, E):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    from oracle_lib import Oracle
    from paper_2510_19366_b200.ep import ExpertParallelLayer
    o = Oracle()
    experts, parts, wr = _data(o, E)
    T = 20 + 7 * rank  # ragged: ranks hold different token counts
    x = torch.from_numpy(o.uniform_pm1(50 + rank, T * D).reshape(T, D))
    kpt = torch.from_numpy(np.random.default_rng(rank).choice([1, 2, 4, 8], size=T).astype(np.int32))
    layer = ExpertParallelLayer(OracleEpOps(o, experts, parts, wr, rank, world))
    y, sel, w, counts, recv_counts = layer.forward(x, k_per_token=kpt, return_routing=True)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), x=x.numpy(), y=y.numpy(), sel=sel.numpy(), w=w.numpy(),
             kpt=kpt.numpy(), counts=np.array(counts), recv_counts=np.array(recv_counts))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,E", [(2, 4), (2, 3)])  # E=3: sub-expert granularity (6 of 12 per rank)
def test_expert_parallel_gloo_matches_single_process(oracle, tmp_path, world, E):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), E), nprocs=world, join=True)
    experts, parts, wr = _data(oracle, E)
    res = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    # the counts each rank sends are what the peers receive
    for r in range(world):
        for q in range(world):
            assert res[r]["counts"][q] == res[q]["recv_counts"][r]
    for r in range(world):
        x, y = res[r]["x"], res[r]["y"]
        sel = res[r]["sel"].view(np.uint32)
        logits = oracle.router_logits(x, wr, x.shape[0], D, E * S)
        osel, ow, _ = oracle.route(logits, 0, K_MAX, 1, k_per_token=res[r]["kpt"].astype(np.uint32))
        assert np.array_equal(sel, osel)
        want = oracle.layer_forward(experts, parts, S, x, osel, ow, 1)
        rms = np.sqrt((want.astype(np.float64) ** 2).mean(axis=1, keepdims=True))
        # partials are rounded to fp32 per rank before the combine: fp32-level agreement
        assert np.all(np.abs(y - want) <= 1e-5 * (rms + np.abs(want)))
