"""torch plumbing around libsagips: device memory (the caller-owned
workspace), the current CUDA stream, and process groups for the multi-rank
rendezvous (IPC handles of the exchange windows, the NCCL unique id).
No arithmetic of the method lives here."""
import torch

from . import _lib


def current_stream_ptr(device=None):
    return ctypes_void(torch.cuda.current_stream(device).cuda_stream)


def ctypes_void(x):
    import ctypes
    return ctypes.c_void_p(x)


def make_context(cfg, device=None):
    """Allocate the workspace with torch and create the rank context on the
    current stream of `device`."""
    if not torch.cuda.is_available():
        raise RuntimeError("sagips needs a CUDA device (sm_100a); there is no CPU fallback")
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    nbytes = _lib.workspace_size(cfg)
    ws = torch.empty(nbytes, dtype=torch.uint8, device=device)
    with torch.cuda.device(device):
        ctx = _lib.Context(cfg, ws.data_ptr(), nbytes, current_stream_ptr(device), keepalive=ws)
    return ctx


def connect(ctx, group=None):
    """Multi-rank wiring through torch.distributed (rendezvous only)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if world == 1:
        return
    handles = [None] * world
    dist.all_gather_object(handles, ctx.ipc_handle(), group=group)
    ctx.connect_peers(handles)
    uid = [_lib.nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(uid, src=0, group=group)
    ctx.connect_nccl(uid[0])


def close(ctx, group=None):
    """Quiesce, then destroy (include/sagips.h sagips_destroy): every rank
    synchronises its device and passes a barrier before any rank frees the
    exchange window its peers map."""
    torch.cuda.synchronize()
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.barrier(group=group)
    except Exception:
        pass
    ctx.close()
