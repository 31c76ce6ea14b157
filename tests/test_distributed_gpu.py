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


def _self_exchange(rank, world, port, out_dir, steps, emulate=False, tiles=8):
    """One engine with every subpatch of an 8 x 8 tiling, but every solution
    and viscosity copy whose donor lies in the right half and whose recipient
    lies in the left half routed through the engine's transport as a send to
    itself (NCCL self send/recv): pack, grouped send/recv and unpack inside
    each captured superstep, the edge-first slot order and, per RK stage, the
    edge run's passes + halo on one stream while the interior run's passes run
    on another. Must be bitwise equal to the plain engine."""
    if emulate:  # CPU: gloo for the rendezvous, the emulation build's shared-memory transport
        import torch.distributed as dist

        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
    else:
        dist = _init(rank, world, port, "nccl")
    import numpy as np

    from paper_2506_19370_b200 import _native as N, engine as EN, geometry as G

    ctx = N.Context(emulate=True) if emulate else N.Context(0)
    dec, ic, _ = P.vortex_tiles(r=tiles, s=tiles, n0=30 if emulate else 238)
    pl = dec.plan
    i0s = sorted({d.sp.i0 for d in dec.subs})
    right = np.array([d.sp.i0 >= i0s[len(i0s) // 2] for d in dec.subs])
    n = len(dec.subs)

    def route(dst_sub, src_sub, src):
        cross = (~right[dst_sub]) & right[src_sub]
        send_sub, send_loc = src_sub[cross].astype(np.int32), src[cross].astype(np.int32)
        new_src_sub, new_src = src_sub.copy(), src.copy()
        new_src_sub[cross] = -1
        new_src[cross] = np.arange(int(cross.sum()))
        return new_src_sub, new_src, (send_sub, send_loc), int(cross.sum())

    s_sub, s_src, e_send, ne = route(pl.sol_dst_sub, pl.sol_src_sub, pl.sol_src)
    v_sub, v_src, mu_send, nm = route(pl.v_dst_sub, pl.v_src_sub, pl.v_src)
    plan = G.Plan(pl.sol_dst_sub, pl.sol_dst, s_sub, s_src, pl.v_dst_sub, pl.v_dst, v_sub, v_src, pl.v_w)
    assert ne > 0 and nm > 0
    rp = D.RankPlan(0, 1, np.zeros(n, dtype=np.int64), list(range(n)), plan, {0: e_send}, {0: ne}, {0: mu_send},
                    {0: nm})
    DE = D.DistributedEngine(ctx, dec, rp, ic, EN.EngineConfig(cfl=0.5), transport="native")
    assert DE.run(steps) == steps
    for k in range(n):
        np.save(os.path.join(out_dir, f"sub{k}.npy"), DE.E.get_state(k))
    DE.E.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_native_transport_self_exchange_edge_first_bitwise(tmp_path, gpu_ctx):
    from paper_2506_19370_b200 import engine as EN

    steps = 4
    mp.start_processes(_self_exchange, args=(1, _free_port(), str(tmp_path), steps), nprocs=1, join=True,
                       start_method="spawn")
    dec, ic, _ = P.vortex_tiles(r=8, s=8)
    E = EN.Engine(gpu_ctx, dec, ic, EN.EngineConfig(cfl=0.5))
    E.run(steps)
    for g in range(len(dec.subs)):
        assert np.array_equal(np.load(tmp_path / f"sub{g}.npy"), E.get_state(g)), g


def test_self_exchange_routing_cpu(tmp_path, emu_ctx):
    """The self-exchange routing and the edge-first layout on the CPU
    (emulation build, shared-memory transport): bitwise equal to the plain
    engine."""
    from paper_2506_19370_b200 import engine as EN

    steps = 2
    mp.start_processes(_self_exchange, args=(1, _free_port(), str(tmp_path), steps, True, 4), nprocs=1, join=True,
                       start_method="spawn")
    dec, ic, _ = P.vortex_tiles(r=4, s=4, n0=30)
    E = EN.Engine(emu_ctx, dec, ic, EN.EngineConfig(cfl=0.5))
    E.run(steps)
    for g in range(len(dec.subs)):
        assert np.array_equal(np.load(tmp_path / f"sub{g}.npy"), E.get_state(g)), g
