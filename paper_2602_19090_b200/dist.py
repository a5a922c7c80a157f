"""Multi-GPU plumbing for the block-column partition: torch.distributed supplies the
process group; libozr creates its own NCCL communicator from a unique id that rank 0 broadcasts over it.
Marshalling only — every collective of the sweep is issued inside libozr on the context's stream."""
from ._ozr import ozr_comm_create_nccl, ozr_comm_nccl_id


def partition(n, world_size, rank):
    """Columns [col0, col0 + nl) owned by `rank`: the equal block partition libozr uses (n % P == 0)."""
    if n % world_size:
        raise ValueError(f"n = {n} is not a multiple of the {world_size} ranks")
    nl = n // world_size
    return rank * nl, nl


def broadcast_id(uid, group=None):
    """Rank 0's 128-byte id to every rank over the torch.distributed group (any backend)."""
    import torch.distributed as dist
    obj = [uid if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def comm_from_process_group(device, group=None):
    """An ozr NCCL communicator spanning the torch.distributed group (one rank per GPU)."""
    import torch.distributed as dist
    rank, ws = dist.get_rank(group), dist.get_world_size(group)
    uid = broadcast_id(ozr_comm_nccl_id() if rank == 0 else None, group)
    return ozr_comm_create_nccl(uid, ws, rank, device)


def broadcast_tensor(t, src=0, group=None):
    """torch.distributed.broadcast of a vector or a COLUMN-MAJOR matrix (stride (1, ld), the library's
    layout): collectives need contiguous tensors, and the transpose of a column-major matrix is a
    contiguous row-major view of the same memory."""
    import torch.distributed as dist
    if t.dim() == 2 and not t.is_contiguous():
        v = t.t()
        if not v.is_contiguous():
            raise ValueError("expected a contiguous column-major matrix")
        dist.broadcast(v, src=src, group=group)
    else:
        dist.broadcast(t, src=src, group=group)
    return t
