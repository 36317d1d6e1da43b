"""Data-parallel Muon sharding of a layer set.

Every rank holds every momentum matrix; rank r orthogonalises the matrices
``pe_shard_plan`` assigns to it (deterministic LPT, identical on all ranks, no
communication), then every rank receives every result (each rank needs all
of polar(M) for its weight update W <- W - lr * polar(M)).

The product path is ``attach`` + ``sharded_outputs`` + ``polar_sharded``:
libpe's own NCCL communicator (pe_attach_comm) and pe_polar_sharded, whose
outputs live in one flat buffer laid out by pe_shard_layout, so every rank's
last update epilogue writes its own chunk and one in-place all-gather per
bucket fills the rest while later buckets compute;
torch.distributed only hands the NCCL unique id around.  ``polar_split``
runs one matrix split by columns over the ranks.  ``GatherPlan`` and
``gather_outputs`` are the torch-level alternative (one all-gather of
per-rank packed results; NCCL or gloo), kept for users without libpe's
communicator and exercised by the gloo tests.
"""
from __future__ import annotations

from . import PE_BF16, PE_FP32, pe_nccl_unique_id, pe_shard_layout, pe_shard_plan


def owned(shapes, rank, world):
    """Indices of the matrices rank `rank` computes (ascending)."""
    owner = pe_shard_plan(shapes, world)
    return [i for i, o in enumerate(owner) if o == rank], owner


def _nbytes(shape, elem_size):
    return int(shape[0]) * int(shape[1]) * elem_size


def gather_outputs(local, shapes, owner, world, elem_size, make_buffer, group=None):
    """All-gather per-rank results.

    local       dict {matrix index -> flat uint8 tensor of that matrix's bytes}
                for the indices this rank owns (all on one device).
    owner       pe_shard_plan output (list, len = len(shapes)).
    make_buffer callable(nbytes) -> zero uint8 tensor on the transport device.
    Returns {matrix index -> flat uint8 tensor} for every matrix.
    """
    import torch
    import torch.distributed as dist

    per_rank = [[i for i, o in enumerate(owner) if o == r] for r in range(world)]
    sizes = [sum(_nbytes(shapes[i], elem_size) for i in idx) for idx in per_rank]
    cap = max(max(sizes), 1)
    rank = dist.get_rank(group)
    send = make_buffer(cap)
    off = 0
    for i in per_rank[rank]:
        nb = _nbytes(shapes[i], elem_size)
        send[off:off + nb].copy_(local[i].view(torch.uint8).reshape(-1))
        off += nb
    recv = [make_buffer(cap) for _ in range(world)]
    dist.all_gather(recv, send, group=group)
    out = {}
    for r in range(world):
        off = 0
        for i in per_rank[r]:
            nb = _nbytes(shapes[i], elem_size)
            out[i] = recv[r][off:off + nb]
            off += nb
    return out


class GatherPlan:
    """Preallocated all-gather of one layer set's results with no packing
    copy: pe_polar writes this rank's results straight into the send buffer
    (``local_views``), one ``all_gather_into_tensor`` fills ``recv`` (world x
    cap bytes), and ``views`` are every matrix's result inside ``recv``.
    Matrix slots are 256-byte aligned (the library wants 16-byte-aligned
    buffers).  Built once per layer set; reuse it every step."""

    def __init__(self, shapes, owner, world, rank, elem_size, dtype, device):
        import torch
        self.world, self.rank = world, rank
        per_rank = [[i for i, o in enumerate(owner) if o == r] for r in range(world)]
        offs, caps = {}, []
        for r in range(world):
            off = 0
            for i in per_rank[r]:
                offs[i] = (r, off)
                off += (_nbytes(shapes[i], elem_size) + 255) // 256 * 256
            caps.append(off)
        self.cap = max(max(caps), 256)
        self.recv = torch.zeros(world * self.cap, dtype=torch.uint8, device=device)
        self.send = torch.zeros(self.cap, dtype=torch.uint8, device=device)

        def view(buf, off, shape):
            nb = _nbytes(shape, elem_size)
            return buf[off:off + nb].view(dtype).view(int(shape[0]), int(shape[1]))

        self.local_index = per_rank[rank]
        self.local_views = [view(self.send, offs[i][1], shapes[i]) for i in self.local_index]
        self.views = [view(self.recv, offs[i][0] * self.cap + offs[i][1], shapes[i]) for i in range(len(shapes))]

    def gather(self, group=None):
        import torch.distributed as dist
        dist.all_gather_into_tensor(self.recv, self.send, group=group)
        return self.views


def attach(ctx, group=None):
    """pe_attach_comm over the ranks of a torch.distributed group: rank 0 makes
    the ncclUniqueId (pe_nccl_unique_id), torch.distributed hands it to the
    others (plumbing only), and every rank binds a libpe NCCL communicator to
    its context.  Returns (rank, world)."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    box = [pe_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    ctx.attach_comm(box[0], rank, world)
    return rank, world


def sharded_outputs(shapes, world, dtype, device):
    """One flat output buffer in pe_shard_layout order (identical on every
    rank) and the per-matrix views into it.  Passing the views as
    pe_polar_sharded's outputs turns its exchange into one in-place
    all-gather per bucket with no packing copy.  Returns (flat, views)."""
    import torch
    code = PE_BF16 if dtype == torch.bfloat16 else PE_FP32
    es = 2 if code == PE_BF16 else 4
    offs, total = pe_shard_layout(shapes, world, code)
    flat = torch.empty(total, dtype=torch.uint8, device=device)
    views = [flat[o:o + int(r) * int(c) * es].view(dtype).view(int(r), int(c)) for o, (r, c) in zip(offs, shapes)]
    return flat, views


def polar_sharded(ctx, inputs, outputs, iters=5, stream=None):
    """pe_polar_sharded: the layer set is split over the
    ranks by pe_shard_plan, each rank computes its share and libpe exchanges
    the results over NCCL bucket by bucket, overlapping the remaining
    compute: one in-place all-gather per bucket when ``outputs`` are the views
    of ``sharded_outputs``, else per-matrix broadcasts.  Needs ``attach``."""
    return ctx.polar_sharded(inputs, outputs, iters=iters, stream=stream)


def polar_split(ctx, shard, iters=5, group=None, out=None):
    """Intra-matrix sharding: this rank's column block
    of one wide matrix, orthogonalised jointly with the other ranks' blocks;
    the fp32 partial Grams and the squared norm are summed with
    torch.distributed.all_reduce (NCCL on GPUs).  Returns this rank's
    columns of polar(M)."""
    import torch.distributed as dist
    return ctx.polar_split(shard, lambda t: dist.all_reduce(t, group=group), out=out, iters=iters)
