"""Multi-rank host logic on CPU (gloo, world size 2): every rank computes the
same LPT shard plan (pe_shard_plan) and exchange buckets (pe_shard_buckets),
owns a disjoint subset, and the torch-level all-gather, a replay of
pe_polar_sharded's per-bucket owner broadcasts and a replay of its zero-copy
per-bucket all-gather over the pe_shard_layout buffer each leave every rank
with every matrix's bytes."""
import os
import socket

import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["PE_SHARD_BUCKETS"] = "3"       # several buckets on a small set (plan, layout, call agree)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import pe_synth as syn
        from paper_2505_16932_b200 import dist as pdist
        shapes = syn.layer_set_shapes("gpt2-small", layers=2) + [(5, 7), (9, 3)]
        idx, owner = pdist.owned(shapes, rank, world)
        # stand-in for pe_polar results: a value pattern unique per matrix
        local = {}
        for i in idx:
            r, c = shapes[i]
            t = (torch.arange(r * c, dtype=torch.float32) % 251 + i).to(torch.bfloat16)
            local[i] = t.view(torch.int16).view(torch.uint8)
        out = pdist.gather_outputs(local, shapes, owner, world, 2,
                                   lambda nb: torch.zeros(nb, dtype=torch.uint8))
        ok = len(out) == len(shapes)
        for i, (r, c) in enumerate(shapes):
            exp = (torch.arange(r * c, dtype=torch.float32) % 251 + i).to(torch.bfloat16)
            got = out[i].view(torch.int16).view(torch.bfloat16)
            ok = ok and torch.equal(got, exp)
        # zero-copy plan: results written into the send buffer, one all-gather
        gp = pdist.GatherPlan(shapes, owner, world, rank, 2, torch.bfloat16, "cpu")
        for i, v in zip(gp.local_index, gp.local_views):
            r, c = shapes[i]
            v.copy_((torch.arange(r * c, dtype=torch.float32) % 251 + i).to(torch.bfloat16).view(r, c))
        views = gp.gather()
        for i, (r, c) in enumerate(shapes):
            exp = (torch.arange(r * c, dtype=torch.float32) % 251 + i).to(torch.bfloat16).view(r, c)
            ok = ok and torch.equal(views[i], exp) and (views[i].data_ptr() - gp.recv.data_ptr()) % 256 == 0
        plans = [None] * world
        dist.all_gather_object(plans, owner)
        # pe_polar_sharded's exchange schedule (pe_dist.cpp), replayed with
        # gloo: buckets from pe_shard_buckets (identical on every rank), each
        # matrix broadcast from its pe_shard_plan owner into every rank's output
        from paper_2505_16932_b200 import pe_shard_buckets
        beg = pe_shard_buckets(shapes, 4)
        begs = [None] * world
        dist.all_gather_object(begs, beg)
        outs = [torch.zeros(r * c, dtype=torch.bfloat16) for r, c in shapes]
        for i in idx:
            r, c = shapes[i]
            outs[i].copy_((torch.arange(r * c, dtype=torch.float32) % 251 + i).to(torch.bfloat16))
        for b in range(4):
            for i in range(beg[b], beg[b + 1]):
                dist.broadcast(outs[i], src=owner[i])
        for i, (r, c) in enumerate(shapes):
            ok = ok and torch.equal(outs[i], (torch.arange(r * c, dtype=torch.float32) % 251 + i).to(torch.bfloat16))
        # the zero-copy layout (pe_shard_layout, dist.sharded_outputs): every
        # rank writes its owned results into its chunk of each bucket, one
        # all-gather per bucket over the chunks completes every output
        from paper_2505_16932_b200 import pe_shard_layout
        offs, chunks, total = pe_shard_layout(shapes, world, chunks=True)
        flat, views = pdist.sharded_outputs(shapes, world, torch.bfloat16, "cpu")
        ok = ok and len(chunks) == 3 and flat.numel() == total == world * sum(chunks)
        flat.zero_()
        for i in idx:
            r, c = shapes[i]
            views[i].copy_((torch.arange(r * c, dtype=torch.float32) % 251 + i).to(torch.bfloat16).view(r, c))
        base = 0
        for ch in chunks:
            parts = [flat[base + k * ch:base + (k + 1) * ch] for k in range(world)]
            dist.all_gather(parts, parts[rank].clone())
            base += world * ch
        for i, (r, c) in enumerate(shapes):
            exp = (torch.arange(r * c, dtype=torch.float32) % 251 + i).to(torch.bfloat16).view(r, c)
            ok = ok and torch.equal(views[i], exp) and offs[i] % 256 == 0
        layouts = [None] * world
        dist.all_gather_object(layouts, (offs, chunks))
        same = all(p == owner for p in plans) and all(bb == beg for bb in begs)
        same = same and all(lay == (offs, chunks) for lay in layouts)
        q.put((rank, ok, same, sorted(idx)))
    finally:
        dist.destroy_process_group()


def test_shard_and_allgather_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    owned = []
    for rank, ok, same_plan, idx in res:
        assert ok and same_plan
        owned += idx
    assert sorted(owned) == list(range(len(owned)))
