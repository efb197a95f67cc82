"""Multi-GPU xmap: library-row sharding over one process per GPU.

North-star row (e) of SURVEY.md section 8: the dataset X[N][T] is replicated
once from rank 0 with an NCCL broadcast over NVLink, rank g computes the rho
columns of libraries [g N / G, (g+1) N / G) for every target with the
single-device kernels (``cmb_xmap_dev``), and the slabs are gathered to
rank 0.  There is no other collective: pairs are independent and every rank
processes the same distinct-E set, so per-rank work is uniform and rho is
bitwise identical for any G (per-pair arithmetic does not depend on G).

Two implementations of the same plan:

* ``init_native_comm`` + ``xmap_native_rank`` -- the product path: libcmb200's
  own NCCL communicator (``cmb_nccl_init_rank``; the 128-byte id travels over
  torch.distributed's CPU group, which is only plumbing) and
  ``cmb_xmap_rank``, which broadcasts X, computes the rank's library block and
  gathers the library-major rows to rank 0 with grouped ncclSend/ncclRecv --
  no torch collective on the data path, rank 0 holds rho plus one shard.
* ``xmap_sharded`` -- the same plan over torch.distributed collectives, kept
  for gloo runs (ranks sharing one GPU, CPU tests with an oracle ``compute``).

All arithmetic runs in libcmb200.
"""

from __future__ import annotations

from typing import Callable

import numpy as np

from . import _native as nat


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous library block of ``rank`` (sizes differ by at most one)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def slab_width(n: int, world: int) -> int:
    """Common (padded) column count of every rank's rho slab, a multiple of 4."""
    w = -(-n // world)
    return (w + 3) // 4 * 4


def native_shard(X, estar: np.ndarray, tau: int, lo: int, hi: int, slab, stats: np.ndarray | None,
                 device: int, stream_handle: int | None) -> None:
    """rho_T[:, 0:hi-lo] of libraries [lo, hi) into ``slab`` (torch, [N][ldr]) on the device."""
    N, T = X.shape
    est = np.ascontiguousarray(estar, dtype=np.int32)
    nat.call("cmb_xmap_dev", device, X.data_ptr(), N, T, X.stride(0), nat.ptr(est), tau, lo, hi,
             slab.data_ptr(), slab.stride(0), stream_handle, nat.ptr(stats))


def _host_staged(group) -> bool:
    """gloo moves CUDA tensors through host copies (functional multi-rank runs that
    share one GPU, CMB_DIST_BACKEND=gloo); NCCL moves them device to device."""
    import torch.distributed as dist
    return dist.is_initialized() and dist.get_backend(group) == "gloo"


def broadcast_(t, src: int = 0, group=None) -> None:
    """In-place broadcast of a device tensor from ``src``."""
    import torch.distributed as dist
    if _host_staged(group) and t.is_cuda:
        h = t.cpu()
        dist.broadcast(h, src=src, group=group)
        t.copy_(h)
    else:
        dist.broadcast(t, src=src, group=group)


def all_gather_rows(part, n_total: int, group=None):
    """Concatenate every rank's ``part`` (contiguous shards of a length-``n_total``
    vector, shard_bounds order; sizes may differ by one) on every rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    w = -(-n_total // world)
    buf = torch.zeros(w, dtype=part.dtype, device=part.device)
    buf[: part.numel()] = part
    staged = _host_staged(group) and buf.is_cuda
    src = buf.cpu() if staged else buf
    outs = [torch.empty_like(src) for _ in range(world)]
    dist.all_gather(outs, src, group=group)
    pieces = []
    for g in range(world):
        lo, hi = shard_bounds(n_total, world, g)
        pieces.append(outs[g][: hi - lo])
    res = torch.cat(pieces)
    return res.to(part.device) if staged else res


def xmap_sharded(X, estar: np.ndarray, tau: int = 1, group=None, compute: Callable | None = None,
                 stats: np.ndarray | None = None, broadcast: bool = True, gather: bool = True):
    """Sharded all-to-all cross map.

    ``X``: torch tensor [N][T] float32 on this rank's device (meaningful on
    rank 0 when ``broadcast``).  Returns on rank 0 a torch tensor
    rho_T[N][G * slab] (target-major; column c of rank g's slab is library
    shard_bounds(N, G, g)[0] + c; padding columns are NaN), None elsewhere.
    ``compute`` replaces the device kernel (tests run the same plumbing on
    CPU with gloo and an oracle-backed compute).  ``gather=False`` skips the
    gather and returns every rank its own slab (callers that copy each rank's
    slab to host memory directly).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    N = X.shape[0]
    if world > 1 and broadcast:
        broadcast_(X, src=0, group=group)
    lo, hi = shard_bounds(N, world, rank)
    w = slab_width(N, world)
    slab = torch.full((N, w), float("nan"), dtype=torch.float32, device=X.device)
    if compute is None:
        dev = X.device.index or 0
        handle = torch.cuda.current_stream(X.device).cuda_stream
        native_shard(X, estar, tau, lo, hi, slab, stats, dev, handle)
    else:
        compute(X, estar, tau, lo, hi, slab)
    if world == 1 or not gather:
        return slab
    staged = _host_staged(group) and slab.is_cuda
    src = slab.cpu() if staged else slab
    gathered = [torch.empty_like(src) for _ in range(world)] if rank == 0 else None
    dist.gather(src, gathered, dst=0, group=group)
    if rank != 0:
        return None
    out = torch.cat(gathered, dim=1)
    return out.to(slab.device) if staged else out


def assemble(rhoT_slabs, n: int, world: int) -> np.ndarray:
    """rho[lib, tgt] (numpy, float32) from the gathered target-major slabs."""
    rt = rhoT_slabs.cpu().numpy() if hasattr(rhoT_slabs, "cpu") else np.asarray(rhoT_slabs)
    w = slab_width(n, world)
    cols = []
    for g in range(world):
        lo, hi = shard_bounds(n, world, g)
        cols.append(rt[:, g * w: g * w + (hi - lo)])
    return np.concatenate(cols, axis=1).T


# ---------------------------------------------------------------- native NCCL path
def init_native_comm(device: int, group=None) -> dict:
    """Create this process's libcmb200 NCCL communicator (rank and size of the
    torch.distributed group; one process per GPU).  Returns {"nranks", "rank",
    "nccl_version"} as reported by the communicator itself."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    uid = np.zeros(128, dtype=np.uint8)
    if rank == 0:
        nat.call("cmb_nccl_unique_id", nat.ptr(uid))
    box = [uid.tobytes() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0, group=group)
    uid = np.frombuffer(box[0], dtype=np.uint8).copy()
    nat.call("cmb_nccl_init_rank", device, nat.ptr(uid), world, rank)
    n, r, v = (np.zeros(1, dtype=np.int32) for _ in range(3))
    nat.call("cmb_nccl_info", device, nat.ptr(n), nat.ptr(r), nat.ptr(v))
    return {"nranks": int(n[0]), "rank": int(r[0]), "nccl_version": int(v[0])}


def xmap_native_rank(X, estar: np.ndarray, tau: int, rho=None, stats: np.ndarray | None = None,
                     device: int | None = None, stream_handle: int | None = None) -> None:
    """One rank of the sharded cross map through libcmb200 (cmb_xmap_rank).

    ``X``: torch float32 [N][T] on this rank's device (valid on rank 0; the
    broadcast overwrites it elsewhere).  ``rho``: on rank 0 a torch float32
    [N][N] device buffer that receives rho[lib, tgt]; None on other ranks."""
    N, T = X.shape
    assert X.is_contiguous() and (rho is None or rho.is_contiguous())
    est = np.ascontiguousarray(estar, dtype=np.int32)
    dev = X.device.index if device is None else device
    nat.call("cmb_xmap_rank", dev, X.data_ptr(), N, T, nat.ptr(est), tau,
             None if rho is None else rho.data_ptr(), stream_handle, nat.ptr(stats))


def xmap_multi(values: np.ndarray, estar, devices, tau: int = 1) -> np.ndarray:
    """Single-process multi-device cross map (cmb_xmap_multi): ``values`` (series,
    time) float32 host array; returns rho[lib, tgt] float32."""
    X = np.ascontiguousarray(values, dtype=np.float32)
    N, T = X.shape
    est = np.ascontiguousarray(estar, dtype=np.int32)
    devs = np.ascontiguousarray(devices, dtype=np.int32)
    out = nat.host_empty((N, N), np.float32)
    st = np.zeros(8)
    nat.call("cmb_xmap_multi", nat.ptr(devs), devs.size, nat.ptr(X), N, T, nat.ptr(est), tau, nat.ptr(out),
             nat.ptr(st))
    return out
