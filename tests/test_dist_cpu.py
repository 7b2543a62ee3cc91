"""N>1 host logic on CPU with the gloo backend (world 2, 3 and 8 -- 8 is the
bench's M2 launch: Qwen2.5-7B FSDP-8 -> TP-2 x DP-4, AUTO rank map, 2 GiB
buckets, link-weight balancing): the NCCL-id
bootstrap broadcast, plan determinism across ranks (every rank builds the same
plan from the same request, PAPER.md:555/576 plans must agree for the
collective sync), and ledger symmetry (what r sends g is what g receives)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_20863_b200.state import Plan, bootstrap_nccl_id, plan_digest
        from plexgen import MODELS, manifest
        nid = bootstrap_nccl_id(rank)
        ids = [None] * world
        dist.all_gather_object(ids, nid)
        from paper_2605_20863_b200 import _lib as L
        big = world in (2, 8)
        model = "qwen2.5-7b" if big else "mid-moe"
        tp = 2 if big else 1
        ep = 1
        plan = Plan(manifest(model), head_dim=MODELS[model].head_dim, world=world, tp=tp, dp=world // tp, ep=ep,
                    rank_map=L.RANKMAP_AUTO if world == 8 else L.RANKMAP_TP_FAST)
        dig = [plan_digest(plan, g) for g in range(world)]
        digs = [None] * world
        dist.all_gather_object(digs, dig)
        info = plan.rank_info(rank)
        sr = [None] * world
        dist.all_gather_object(sr, (info.send_bytes, info.recv_bytes))
        L = plan.ledger()
        # NEXT-1 balancing: every rank contributes its own link rate, all-gathered
        # (as bench.py does); every rank must derive the same carried buckets
        import torch
        w = torch.tensor([10.0 + 5.0 * rank])
        ws = [torch.zeros(1) for _ in range(world)]
        dist.all_gather(ws, w)
        cp = Plan(manifest(model), world=world, bucket_bytes={2: 1 << 30, 8: 2 << 30}.get(world, 1 << 14),
                  link_weights=[float(x) for x in ws])
        carry = [(c.owner, c.bucket, c.carrier, c.slab_offset, c.bytes, c.carry_offset) for c in cp.carry()]
        carries = [None] * world
        dist.all_gather_object(carries, carry)
        # NEXT-2 replica plans: the all-gather ledger is symmetric
        rp = Plan(manifest(model), world=world, replica_param=True)
        gi = rp.rank_info(rank)
        gs = [None] * world
        dist.all_gather_object(gs, (gi.gather_send_bytes, gi.gather_recv_bytes))
        ok = (all(i == ids[0] for i in ids) and len(ids[0]) == 128 and any(ids[0])
              and all(d == digs[0] for d in digs)
              and sr[rank][0] == int(L[rank].sum() - L[rank, rank])
              and sum(s for s, _ in sr) == sum(r for _, r in sr)
              and all(c == carries[0] for c in carries) and len(carries[0]) > 0
              and sum(a for a, _ in gs) == sum(b for _, b in gs) > 0)
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 8])
def test_gloo_multi_rank_host_logic(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    assert all(res[r] for r in range(world)), res
