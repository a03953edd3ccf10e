"""CUDA IPC plumbing of the peer-memory strip transport, across processes (GPU).

Two processes on the one GPU of the test box exchange their 64-byte IPC
handles over gloo, map each other's p2p regions (xmhd_p2p_connect) and write
into every rank's board (xmhd_p2p_probe); after a host barrier each reads its
own board.  No kernel waits on another process's kernel, so this is safe on a
single device; the spinning exchange itself is covered by the one-launch
emulation in test_strips_gpu.py.
"""

import ctypes
import os
import socket

import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2108_13622_b200 import _lib
        lib = _lib.load()
        torch.cuda.set_device(0)
        ctx = _lib.Context(32, 6, 0.1, 0.1, 0.01, 0.01, 0.01, 5.0 / 3.0, 1.0,
                           _lib.BC_PERIODIC, _lib.BC_HALO)
        buf = (ctypes.c_char * 64)()
        _lib.check(lib.xmhd_p2p_alloc(ctx.h, buf), "xmhd_p2p_alloc")
        handles = [None] * world
        dist.all_gather_object(handles, bytes(buf))
        blob = (ctypes.c_char * (64 * world)).from_buffer_copy(b"".join(handles))
        _lib.check(lib.xmhd_p2p_connect(ctx.h, rank, world, blob, 1), "xmhd_p2p_connect")
        _lib.check(lib.xmhd_p2p_probe(ctx.h, 100.0 + rank), "xmhd_p2p_probe")
        dist.barrier()
        board = (ctypes.c_double * 32)()
        _lib.check(lib.xmhd_p2p_read_board(ctx.h, board), "xmhd_p2p_read_board")
        with open(f"{out_path}.{rank}", "w") as fh:
            fh.write(" ".join(repr(board[4 * q + k]) for q in range(world) for k in (0, 1)))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_peer_regions_mapped_across_processes(tmp_path):
    import torch.multiprocessing as mp
    world = 2
    out = str(tmp_path / "board")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for rank in range(world):
        vals = [float(x) for x in open(f"{out}.{rank}").read().split()]
        # entry q: (100 + q, q) written by rank q into this rank's board
        assert vals == [100.0, 0.0, 101.0, 1.0]


def _strip_worker(rank, world, port, out_path, fail_rank):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2108_13622_b200 as xb
        from paper_2108_13622_b200 import _lib, strips
        torch.cuda.set_device(0)
        if rank == fail_rank:
            # this rank cannot map its peers (what a box without P2P access would report)
            lib = _lib.load()
            lib.xmhd_p2p_connect = lambda *a: 3
        mhd = strips.StripMhd(xb.StateGrid(32, 12, 0.1, 0.1, None),
                              xb.MHDParams(0.01, 0.01, 0.01), strips.Comm())
        first = mhd.peer_transport()
        again = mhd.peer_transport()
        with open(f"{out_path}.{rank}", "w") as fh:
            fh.write(f"{int(first)} {int(again)}")
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fail_rank", [-1, 1])
def test_strip_peer_link_is_verified_or_all_ranks_fall_back(tmp_path, fail_rank):
    """StripMhd.peer_transport(): handles, mapping and a probe write per peer are
    checked on every rank; when any rank fails, every rank reports False (NCCL
    transport) instead of some ranks spinning on a peer that never posts."""
    import torch.multiprocessing as mp
    world = 2
    out = str(tmp_path / "peer")
    mp.spawn(_strip_worker, args=(world, _free_port(), out, fail_rank), nprocs=world, join=True)
    want = "1 1" if fail_rank < 0 else "0 0"
    for rank in range(world):
        assert open(f"{out}.{rank}").read() == want
