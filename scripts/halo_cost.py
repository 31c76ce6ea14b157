"""Device cost of the multi-rank transport inside a superstep, on one B200:
the config-5 8x8 tiling stepped plainly and with every copy from the right
half into the left half routed through the engine's transport as an NCCL
send to self (pack, grouped send/recv, unpack in each captured step; the
edge run's passes + halo on one stream next to the interior run's passes).
The routed volume (half the tiling's cut, 8 subpatch sides) is what one rank
of an 8-GPU weak-scaling run exchanges across ~2 of its 4 sides.
    python scripts/halo_cost.py"""
import os
import socket
import sys

import torch
import torch.multiprocessing as mp

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def worker(rank, world, port):
    import numpy as np
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world)
    from paper_2506_19370_b200 import _native as N, distributed as D, engine as EN, geometry as G, problems as P

    ctx = N.Context(0)
    dec, ic, _ = P.vortex_tiles(r=8, s=8)

    def timed(E, steps=20):
        E.run(3)
        torch.cuda.synchronize()
        st = torch.cuda.ExternalStream(E.stream())
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        E.enqueue(steps)
        b.record(st)
        torch.cuda.synchronize()
        E.check_error()
        return a.elapsed_time(b) / steps

    plain = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=0.5))
    t0 = timed(plain)
    plain.close()
    pl = dec.plan
    i0s = sorted({d.sp.i0 for d in dec.subs})
    right = np.array([d.sp.i0 >= i0s[len(i0s) // 2] for d in dec.subs])

    def route(dst_sub, src_sub, src):
        cross = (~right[dst_sub]) & right[src_sub]
        ns, nsrc = src_sub.copy(), src.copy()
        ns[cross] = -1
        nsrc[cross] = np.arange(int(cross.sum()))
        return ns, nsrc, (src_sub[cross].astype(np.int32), src[cross].astype(np.int32)), int(cross.sum())

    s_sub, s_src, e_send, ne = route(pl.sol_dst_sub, pl.sol_src_sub, pl.sol_src)
    v_sub, v_src, mu_send, nm = route(pl.v_dst_sub, pl.v_src_sub, pl.v_src)
    plan = G.Plan(pl.sol_dst_sub, pl.sol_dst, s_sub, s_src, pl.v_dst_sub, pl.v_dst, v_sub, v_src, pl.v_w)
    n = len(dec.subs)
    rp = D.RankPlan(0, 1, np.zeros(n, dtype=np.int64), list(range(n)), plan, {0: e_send}, {0: ne}, {0: mu_send},
                    {0: nm})
    DE = D.DistributedEngine(ctx, dec, rp, ic, EN.EngineConfig(cfl=0.5), transport="native")
    t1 = timed(DE.E)
    print(f"plain {t0:.3f} ms/step; with the transport ({ne} state points = {ne * 32 / 1e6:.2f} MB per stage, "
          f"{nm} mu_hat values per step, NCCL self send/recv + pack/unpack, edge-first streams) {t1:.3f} ms/step: "
          f"+{100 * (t1 / t0 - 1):.1f}%", flush=True)
    DE.E.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.start_processes(worker, args=(1, port), nprocs=1, join=True, start_method="spawn")
