"""Multi-rank superstep on the one B200 the test box has.

NCCL refuses two ranks on one device, and ranks whose kernels wait on one
another must not share a GPU, so on one B200 the device path is exercised
two ways:

* the engine's own transport (``fcsg_engine_attach_comm``: pack, grouped
  ncclSend/Recv, unpack and ncclAllReduce(MIN) enqueued on the engine stream)
  on a real one-rank NCCL communicator: the all-reduce is then a real NCCL
  launch inside the captured CUDA graph of every steady superstep; bitwise
  equal to the plain engine;
* two ranks on cuda:0 with the caller-driven transport over gloo (host
  staging: the host, not a kernel, waits for the peer), so the pack / unpack
  kernels and the halo slots run on the GPU with real cross-rank donors;
  bitwise equal to one rank.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2506_19370_b200 import distributed as D, problems as P


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port, backend):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group(backend, rank=rank, world_size=world)
    return dist


def _nccl_world1(rank, world, port, out_dir, steps):
    dist = _init(rank, world, port, "nccl")
    from paper_2506_19370_b200 import _native as N, engine as EN

    ctx = N.Context(0)
    dec, ic, _ = P.vortex_tiles(r=2, s=2)
    owner = D.partition_tiles(dec, world)
    rp = D.split_plan(dec, owner, rank, world)
    DE = D.DistributedEngine(ctx, dec, rp, ic, EN.EngineConfig(cfl=0.5), transport="native")
    assert DE.run(steps) == steps  # step 0 eager, then graph replays with the NCCL all-reduce inside
    for l, g in enumerate(rp.local):
        np.save(os.path.join(out_dir, f"sub{g}.npy"), DE.E.get_state(l))
    np.save(os.path.join(out_dir, "time.npy"), np.array(DE.E.time()))
    DE.E.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_native_transport_nccl_graph_bitwise(tmp_path, gpu_ctx):
    from paper_2506_19370_b200 import engine as EN

    steps = 4
    mp.start_processes(_nccl_world1, args=(1, _free_port(), str(tmp_path), steps), nprocs=1, join=True,
                       start_method="spawn")
    dec, ic, _ = P.vortex_tiles(r=2, s=2)
    E = EN.Engine(gpu_ctx, dec, ic, EN.EngineConfig(cfl=0.5))
    E.run(steps)
    for g in range(len(dec.subs)):
        assert np.array_equal(np.load(tmp_path / f"sub{g}.npy"), E.get_state(g)), g
    t, st = np.load(tmp_path / "time.npy")
    assert (t, st) == E.time()


def _gloo_two_ranks(rank, world, port, out_dir, steps):
    dist = _init(rank, world, port, "gloo")
    from paper_2506_19370_b200 import _native as N, engine as EN

    ctx = N.Context(0)
    dec, ic, _ = P.vortex_tiles(r=4, s=2, n0=62)
    owner = D.partition_tiles(dec, world)
    rp = D.split_plan(dec, owner, rank, world)
    DE = D.DistributedEngine(ctx, dec, rp, ic, EN.EngineConfig(cfl=0.5), transport="torch")
    assert DE.stage is not None  # gloo carries the CUDA rank's halos through host memory
    DE.run(steps)
    for l, g in enumerate(rp.local):
        np.save(os.path.join(out_dir, f"sub{g}.npy"), DE.E.get_state(l))
    DE.E.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_two_ranks_on_one_gpu_gloo_bitwise(tmp_path, gpu_ctx):
    from paper_2506_19370_b200 import engine as EN

    steps = 3
    mp.start_processes(_gloo_two_ranks, args=(2, _free_port(), str(tmp_path), steps), nprocs=2, join=True,
                       start_method="spawn")
    dec, ic, _ = P.vortex_tiles(r=4, s=2, n0=62)
    E = EN.Engine(gpu_ctx, dec, ic, EN.EngineConfig(cfl=0.5))
    E.run(steps)
    for g in range(len(dec.subs)):
        assert np.array_equal(np.load(tmp_path / f"sub{g}.npy"), E.get_state(g)), g
