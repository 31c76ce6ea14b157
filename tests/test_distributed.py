"""Multi-rank superstep on CPU: world-size-2 gloo runs of the product engine
(emulation build) against the single-rank engine, plus the plan split."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2506_19370_b200 import distributed as D, problems as P


def test_partition_blocks_and_plan_split():
    dec, ic, _ = P.vortex_tiles(r=4, s=2, n0=30)
    owner = D.partition_tiles(dec, 2)
    assert sorted(np.bincount(owner)) == [4, 4]
    # contiguous blocks: each rank owns a 2x2 block of the 4x2 tiling
    rps = [D.split_plan(dec, owner, r, 2) for r in range(2)]
    for a, b in ((0, 1), (1, 0)):
        assert sum(len(v[0]) for v in rps[a].e_send.values()) == rps[b].e_recv.get(a, 0)
        assert sum(len(v[0]) for v in rps[a].mu_send.values()) == rps[b].mu_recv.get(a, 0)
    pl = dec.plan
    assert sum(len(rp.plan.sol_dst) for rp in rps) == len(pl.sol_dst)
    assert sum(len(rp.plan.v_dst) for rp in rps) == len(pl.v_dst)
    # every remote donor is addressed through a halo slot
    for rp in rps:
        assert np.all((rp.plan.sol_src_sub >= 0) | (rp.plan.sol_src >= 0))
        assert rp.e_recv and rp.mu_recv
    with pytest.raises(ValueError):
        D.partition_tiles(dec, 3)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir, steps, classifier="ann", transport="native"):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_19370_b200 import _native as N, engine as EN

    ctx = N.Context(emulate=True)
    dec, ic, _ = P.vortex_tiles(r=4, s=2, n0=30)
    owner = D.partition_tiles(dec, world)
    rp = D.split_plan(dec, owner, rank, world)
    DE = D.DistributedEngine(ctx, dec, rp, ic, EN.EngineConfig(cfl=0.5, classifier=classifier), transport=transport)
    DE.run(steps)
    for l, g in enumerate(rp.local):
        np.save(os.path.join(out_dir, f"sub{g}.npy"), DE.E.get_state(l))
    t, st = DE.E.time()
    np.save(os.path.join(out_dir, f"time{rank}.npy"), np.array([t, st]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("classifier,transport", [("ann", "native"), ("ann", "torch"), ("fallback", "native")])
def test_two_ranks_bitwise_equal_single_rank(tmp_path, emu_ctx, classifier, transport):
    """The same 4x2 tiling stepped by 2 ranks (2x2 subpatches each) and by
    one rank: identical states after 2 supersteps (bitwise), identical t;
    with either classifier variant, and through either transport: the
    engine's own device-ordered one (halos and the dt all-reduce inside the
    superstep; shared-memory mailboxes in the emulation build) or gloo
    point-to-point between the caller-driven parts."""
    from paper_2506_19370_b200 import engine as EN

    steps = 2
    mp.start_processes(_worker, args=(2, _free_port(), str(tmp_path), steps, classifier, transport), nprocs=2,
                       join=True, start_method="spawn")
    dec, ic, _ = P.vortex_tiles(r=4, s=2, n0=30)
    E = EN.Engine(emu_ctx, dec, ic, EN.EngineConfig(cfl=0.5, classifier=classifier))
    E.run(steps)
    for g in range(len(dec.subs)):
        assert np.array_equal(np.load(tmp_path / f"sub{g}.npy"), E.get_state(g)), g
    t, st = E.time()
    for r in range(2):
        tr = np.load(tmp_path / f"time{r}.npy")
        assert tr[0] == t and tr[1] == st


def _worker_interp(rank, world, port, out_dir, steps, transport="native"):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_19370_b200 import _native as N, engine as EN, multipatch as M

    from tests import test_multipatch as TM

    ctx = N.Context(emulate=True)
    patches, validate = TM._geometry(1)
    dec = M.build_decomposition(patches, TM._bcs(), TM.NV, validate_overlap=validate, fast=True)
    owner = np.array([0, 1, 1])  # the Cartesian patch on rank 0, the bilinear one on rank 1
    rp = D.split_plan(dec, owner, rank, world)
    np.save(os.path.join(out_dir, f"ninterp{rank}.npy"), np.array([len(rp.e_interps), len(rp.mu_interps)]))
    DE = D.DistributedEngine(ctx, dec, rp, TM._ic(1), EN.EngineConfig(cfl=0.5), transport=transport)
    DE.run(steps)
    for l, g in enumerate(rp.local):
        np.save(os.path.join(out_dir, f"sub{g}.npy"), DE.E.get_state(l))
        np.save(os.path.join(out_dir, f"mu{g}.npy"), DE.E.get(l, "mu"))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("transport", ["native", "torch"])
def test_two_ranks_with_interpolation_donors_across_ranks(tmp_path, emu_ctx, transport):
    """Two patches with non-coincident lattices on two gloo ranks: every
    solution and viscosity interpolation between them has its donor stencil on
    the other rank, is evaluated there while packing and arrives as a halo
    value. Bitwise equal to the single-rank run after 2 supersteps."""
    from paper_2506_19370_b200 import engine as EN, multipatch as M

    from tests import test_multipatch as TM

    steps = 2
    mp.start_processes(_worker_interp, args=(2, _free_port(), str(tmp_path), steps, transport), nprocs=2,
                       join=True, start_method="spawn")
    for r in range(2):
        ne, nm = np.load(tmp_path / f"ninterp{r}.npy")
        assert ne > 0 and nm > 0
    patches, validate = TM._geometry(1)
    dec = M.build_decomposition(patches, TM._bcs(), TM.NV, validate_overlap=validate, fast=True)
    E = EN.Engine(emu_ctx, dec, TM._ic(1), EN.EngineConfig(cfl=0.5))
    E.run(steps)
    for g in range(len(dec.subs)):
        assert np.array_equal(np.load(tmp_path / f"sub{g}.npy"), E.get_state(g)), g
        assert np.array_equal(np.load(tmp_path / f"mu{g}.npy"), E.get(g, "mu")), g


def test_partition_subpatches_balances_points():
    from paper_2506_19370_b200 import multipatch as M

    from tests import test_multipatch as TM

    patches, validate = TM._geometry(1)
    dec = M.build_decomposition(patches, TM._bcs(), TM.NV, validate_overlap=validate, fast=True)
    owner = D.partition_subpatches(dec, 2)
    assert sorted(set(owner.tolist())) == [0, 1]
    with pytest.raises(ValueError):
        D.partition_subpatches(dec, 5)
