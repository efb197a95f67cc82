"""Multi-process (gloo, world size 2) checks of the library-row sharding plumbing.

The device kernel is replaced by an oracle-backed compute for the CPU run;
broadcast, shard bounds, slab layout, gather and assembly are the production
code paths of paper_2105_12301_b200.distributed.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2105_12301_b200.distributed import assemble, shard_bounds, slab_width, xmap_sharded


def test_shard_bounds_partition():
    for n in (1, 7, 8, 53053, 100):
        for g in (1, 2, 3, 8):
            spans = [shard_bounds(n, g, r) for r in range(g)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
            assert slab_width(n, g) >= max(sizes) and slab_width(n, g) % 4 == 0


def _oracle_compute(X, estar, tau, lo, hi, slab):
    import crossmap_oracle as O
    series = [X[i].double().numpy() for i in range(X.shape[0])]
    rho, _ = O.xmap(series, [int(e) for e in estar], tau, workers=1, libraries=list(range(lo, hi)))
    slab[:, : hi - lo] = torch.from_numpy(rho[lo:hi].T.astype(np.float32))


def _worker(rank, world, port, X, estar, out):
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    Xl = X.clone() if rank == 0 else torch.zeros_like(X)
    res = xmap_sharded(Xl, estar, 1, compute=_oracle_compute)
    if rank == 0:
        out.copy_(torch.from_numpy(assemble(res, X.shape[0], world)))
    else:
        assert res is None
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2])
def test_sharded_xmap_matches_single_process(world):
    import crossmap_oracle as O
    from paper_2105_12301_b200.synthetic import mixed_dataset
    X = torch.from_numpy(mixed_dataset(7, 150, seed=11))
    estar = np.array([1, 2, 2, 3, 1, 0, 2], dtype=np.int32)
    out = torch.full((7, 7), float("nan"))
    out.share_memory_()
    mp.spawn(_worker, args=(world, _free_port(), X, estar, out), nprocs=world, join=True)
    ref, _ = O.xmap([X[i].double().numpy() for i in range(7)], estar.tolist(), 1, workers=1)
    assert np.allclose(out.numpy(), ref.astype(np.float32), equal_nan=True, atol=0)
    assert np.all(np.isnan(out.numpy()[5, :])) and np.all(np.isnan(out.numpy()[:, 5]))


def _gather_worker(rank, world, port, n, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2105_12301_b200.distributed import all_gather_rows, broadcast_
    lo, hi = shard_bounds(n, world, rank)
    full = all_gather_rows(torch.arange(lo, hi, dtype=torch.int32) * 3, n)
    x = torch.arange(5.0) if rank == 0 else torch.zeros(5)
    broadcast_(x, src=0)
    if rank == 1:
        out[: n].copy_(full.float())
        out[n:].copy_(x)
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [7, 8])
def test_uneven_all_gather_and_broadcast(n):
    """E* shards of uneven size (N not divisible by the world size) are padded for
    the collective and reassembled in shard order on every rank."""
    out = torch.full((n + 5,), -1.0)
    out.share_memory_()
    mp.spawn(_gather_worker, args=(3, _free_port(), n, out), nprocs=3, join=True)
    assert out[:n].tolist() == [3.0 * i for i in range(n)]
    assert out[n:].tolist() == [0.0, 1.0, 2.0, 3.0, 4.0]


def _comm_worker(rank, world, port, out):
    """init_native_comm's plumbing with libcmb200's entry points replaced by a
    recorder: rank 0's 128-byte id must reach every rank's cmb_nccl_init_rank."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2105_12301_b200 import distributed as D
    seen = {}

    def fake_call(name, *args):
        if name == "cmb_nccl_unique_id":
            arr = np.ctypeslib.as_array((np.ctypeslib.ctypes.c_uint8 * 128).from_address(args[0]))
            arr[:] = np.arange(128, dtype=np.uint8) + 7
        elif name == "cmb_nccl_init_rank":
            dev, uid_ptr, nranks, r = args
            uid = np.ctypeslib.as_array((np.ctypeslib.ctypes.c_uint8 * 128).from_address(uid_ptr)).copy()
            seen.update(dev=dev, uid=uid, nranks=nranks, rank=r)
        elif name == "cmb_nccl_info":
            for ptr, v in zip(args[1:], (seen["nranks"], seen["rank"], 22809)):
                np.ctypeslib.as_array((np.ctypeslib.ctypes.c_int32 * 1).from_address(ptr))[0] = v

    D.nat.call = fake_call
    info = D.init_native_comm(3)
    ok = (info == {"nranks": world, "rank": rank, "nccl_version": 22809} and seen["dev"] == 3 and
          np.array_equal(seen["uid"], np.arange(128, dtype=np.uint8) + 7))
    out[rank] = 1.0 if ok else 0.0
    dist.destroy_process_group()


def test_native_comm_id_exchange():
    """The libcmb200 NCCL communicator of the N > 1 bench path is created from one
    id that rank 0 draws and torch.distributed (gloo, CPU) hands to the others."""
    out = torch.zeros(3)
    out.share_memory_()
    mp.spawn(_comm_worker, args=(3, _free_port(), out), nprocs=3, join=True)
    assert out.tolist() == [1.0, 1.0, 1.0]
