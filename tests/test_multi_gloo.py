"""Row-sharded multi-process path on CPU (gloo, world size 2): band split, per-rank
reconstruction of its own band, all-gather of the output planes, all-reduce of the
depth profile and the max-over-ranks timing reduction.  The per-rank compute here is
the CPU oracle (no GPU on this box); on the GPU box bench.py runs the same host logic
over NCCL with the CUDA library."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2201_13309_b200 import multi


def test_row_bands_cover_and_align():
    for world in (1, 2, 3, 4, 8):
        b = multi.row_bands(world, 2048)
        assert b[0][0] == 0 and b[-1][1] == 2048
        assert all(b[g][1] == b[g + 1][0] for g in range(world - 1))
        assert all(e > s for s, e in b)
        if 2048 // 128 >= world:
            assert all(s % 128 == 0 for s, _ in b)
    assert multi.row_bands(8, 2048) == [(g * 256, (g + 1) * 256) for g in range(8)]
    # too few aligned blocks: even split
    assert multi.row_bands(3, 200) == [(0, 66), (66, 133), (133, 200)]
    with pytest.raises(ValueError):
        multi.row_bands(4, 3)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = synth.geometry("C1")
        maps = synth.make_maps("C1")
        R = g["n_rows"]
        bands = multi.row_bands(world, R, align=16)
        b0, b1 = bands[rank]
        # each rank generates only its band of the stack and reconstructs only its rows
        band_stack = synth.stack_numpy(maps, "f64", noise=True, rows=(b0, b1))
        rows = np.repeat(np.arange(b0, b1), g["n_cols"])
        cols = np.tile(np.arange(g["n_cols"]), b1 - b0)
        ser = band_stack.reshape(band_stack.shape[0], -1).T
        out_band = oracle.reconstruct_pixels(g, rows, cols, ser).T.reshape(-1, b1 - b0, g["n_cols"])
        full = multi.gather_rows(torch.from_numpy(np.ascontiguousarray(out_band)), bands)
        prof = torch.from_numpy(out_band.sum(axis=(1, 2)))
        multi.allreduce_profile(prof)
        tmax = multi.max_over_ranks([1.0 + rank, 5.0 - rank])
        # the daxm_select_cutoff_sharded callback: a uint64 histogram summed over the ranks in
        # place, called through a C function pointer as the library calls it
        from paper_2201_13309_b200 import binding
        hist = (C.c_ulonglong * 256)(*[(rank + 1) * i + (1 << 40) for i in range(256)])
        red = multi.hist_allreduce()

        def cb(h, n, ctx):
            red(np.ctypeslib.as_array(h, shape=(n,)))
            return 0
        fn = binding.HIST_REDUCE_FN(cb)
        assert fn(hist, 256, None) == 0
        if rank == 0:
            ret["hist"] = list(hist)
            ret["full"] = full.numpy()
            ret["prof"] = prof.numpy()
            ret["tmax"] = tmax
    finally:
        dist.destroy_process_group()


def test_gloo_world2_band_gather_profile():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        ret = mgr.dict()
        mp.spawn(_worker, args=(world, port, ret), nprocs=world, join=True)
        full, prof, tmax = ret["full"], ret["prof"], ret["tmax"]
        ret_hist = ret["hist"]
    g = synth.geometry("C1")
    ref = oracle.reconstruct(g, synth.stack_numpy(synth.make_maps("C1"), "f64", noise=True))
    assert np.allclose(full, ref, rtol=0, atol=1e-9)
    assert np.allclose(prof, ref.sum(axis=(1, 2)), rtol=1e-12, atol=1e-6)
    assert ret_hist == [3 * i + (2 << 40) for i in range(256)]
    assert tmax == [2.0, 5.0]
