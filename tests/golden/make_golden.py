"""Regenerate the committed golden fixtures from the UNMODIFIED reference.

Run here (where /root/reference exists and oracle/_ref is built):

    make -C oracle && python tests/golden/make_golden.py

Outputs (small, committed):
  fc_golden.npz      blend matrix (n_cont=25), FcOperator sizes/profiles and
                     d1/d2/filter/smear outputs of seeded config-1 lines for
                     N in {50, 64, 100, 101, 128, 147, 256, 512}
  engine_golden.npz  reference Engine runs: config-2-style Riemann quadrants on
                     one 64x64 subpatch (phase-level snapshots of step 1 and the
                     state after 3 steps) and the vortex tiling on 2x2
                     subpatches of 48x48 (geometry + state after 2 steps)
  classifier_golden.npz
                     Classifier::classify_line, fallback variant (FC-spectrum
                     decay), on seeded lines of lengths 12..256 (smooth,
                     noisy, step, kink, white noise) at windows 32 and 16
  ../../paper_2506_19370_b200/data/fcnn_v1.bin
                     train_classifier(TrainConfig{}) weights (seed 20240601,
                     include/fcs/viscosity.hpp:91-98) saved as FCNN v1
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2506_19370_b200 import engine as EN, problems as P  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
NS = (50, 64, 100, 101, 128, 147, 256, 512)


def fc_golden():
    d = {"blend_25": ref.blend_matrix(25)}
    for n in NS:
        ne, per, fp, sp = ref.fc_info(n)
        _, f, _ = P.fc_lines_config1(n_lines=8, n=n, seed=100 + n)
        d[f"n{n}_info"] = np.array([ne, per])
        d[f"n{n}_filter_profile"] = fp
        d[f"n{n}_smear_profile"] = sp
        d[f"n{n}_in"] = f
        for mode in ("d1", "d2", "filter", "smear", "cont"):
            d[f"n{n}_{mode}"] = ref.fc_apply(f, mode)
    np.savez_compressed(os.path.join(OUT, "fc_golden.npz"), **d)


def ref_rect_engine(dec, ic, cfl=0.5):
    p = dec.patches[0]
    r = len({sp.i0 for sp in p.subpatches})
    s = len({sp.j0 for sp in p.subpatches})
    sp0 = p.subpatches[0]
    n0 = (sp0.i1 - sp0.i0 + 1) - 2 * p.nv
    kinds = [5 if sd.on_gamma else -1 for sd in p.sides]
    R = ref.RefEngine(p.origin[0], p.origin[1], p.e1[0], p.e2[1], r, s, n0, p.nv, kinds, cfl=cfl, workers=1,
                      weight_path=EN.DEFAULT_WEIGHTS)
    for k in range(len(dec.subs)):
        R.set_state(k, P.initial_state(dec, ic, k))
    R.finish_ic()
    return R


def engine_golden():
    d = {}
    dec, ic, _ = P.riemann_quadrants(n=64, seed=2)
    R = ref_rect_engine(dec, ic)
    d["r64_e_init"] = R.get_state(0)
    for k in ("x", "y", "iq1x", "iq2x", "iq1y", "iq2y", "h_min", "h_max", "w_norm", "mask"):
        d[f"r64_geo_{k}"] = R.get(0, k)
    R.phase(0)
    d["r64_s1_tau"], d["r64_s1_mu_hat"], d["r64_s1_speed"] = R.get(0, "tau"), R.get(0, "mu_hat"), R.get(0, "speed")
    R.phase(1)
    d["r64_s1_mu"] = R.get(0, "mu")
    R.phase(2)
    d["r64_s1_e_p2"] = R.get_state(0)
    d["r64_s1_m01"] = R.get(0, "m01")
    d["r64_s1_dt"] = np.array([R.reduce_dt()])
    for s in range(5):
        R.phase(3, s)
        d[f"r64_s1_rhs{s}"] = R.get_state(0, "rhs")
        R.phase(6)
        d[f"r64_s1_e{s}"] = R.get_state(0)
    R.advance()
    R.step()
    R.step()
    d["r64_s3_e"] = R.get_state(0)
    d["r64_s3_t"] = np.array([R.time()[0]])

    dec, ic, _ = P.vortex_tiles(r=2, s=2, n0=30)
    R = ref_rect_engine(dec, ic)
    for k in range(4):
        d[f"v2_sub{k}_e_init"] = R.get_state(k)
        for f in ("w_norm", "mask", "h_min", "h_max", "x", "y"):
            d[f"v2_sub{k}_geo_{f}"] = R.get(k, f)
    R.step()
    R.step()
    for k in range(4):
        d[f"v2_sub{k}_e2"] = R.get_state(k)
        d[f"v2_sub{k}_tau2"] = R.get(k, "tau")
    # rotated affine channel: all metric terms nonzero, one side of each BC kind
    dec, ic, meta = P.rotated_channel()
    states = np.zeros(16)
    states[0:4] = meta["inflow"]
    press = np.array([1.0, meta["pressure"], 1.0, 1.0])
    R = ref.RefEngine(0, 0, 0, 0, 2, 1, 30, 9, meta["kinds"], side_states=states, side_pressure=press,
                      weight_path=EN.DEFAULT_WEIGHTS, e1=meta["e1"], e2=meta["e2"])
    for k in range(len(dec.subs)):
        R.set_state(k, P.initial_state(dec, ic, k))
    R.finish_ic()
    for k in range(len(dec.subs)):
        d[f"rc_sub{k}_e_init"] = R.get_state(k)
        for f in ("w_norm", "mask", "iq1x", "iq2x", "iq1y", "iq2y"):
            d[f"rc_sub{k}_geo_{f}"] = R.get(k, f)
    for _ in range(3):
        R.step()
    for k in range(len(dec.subs)):
        d[f"rc_sub{k}_e3"] = R.get_state(k)
        d[f"rc_sub{k}_tau3"] = R.get(k, "tau")
    np.savez_compressed(os.path.join(OUT, "engine_golden.npz"), **d)


def classifier_lines(seed=7):
    """Seeded test lines for the fallback classifier: lengths and kinds."""
    rng = np.random.default_rng(seed)
    out = []
    for n in (12, 20, 31, 32, 40, 64, 100, 256):
        x = np.linspace(0.0, 1.0, n)
        for kind in range(5):
            if kind == 0:
                v = np.sin(2 * np.pi * x * rng.uniform(0.5, 4))
            elif kind == 1:
                v = np.sin(2 * np.pi * x * rng.uniform(0.5, 4)) + rng.normal(0, 10 ** rng.uniform(-6, -1), n)
            elif kind == 2:
                v = np.where(x > rng.uniform(0.2, 0.8), 1.0, 0.0) + 0.01 * x
            elif kind == 3:
                v = np.abs(x - rng.uniform(0.3, 0.7)) ** rng.uniform(0.5, 3)
            else:
                v = rng.normal(size=n)
            out.append(v)
    return out


def classifier_golden():
    d = {}
    for k, v in enumerate(classifier_lines()):
        d[f"line{k}"] = v
        for w in (32, 16):
            d[f"line{k}_w{w}"] = ref.classify_line_fallback(v, w)
    np.savez_compressed(os.path.join(OUT, "classifier_golden.npz"), **d)


if __name__ == "__main__":
    if sys.argv[1:] == ["classifier"]:
        classifier_golden()
        sys.exit(0)
    if not os.path.exists(EN.DEFAULT_WEIGHTS) or "--retrain" in sys.argv:
        print("holdout accuracy", ref.train_classifier(EN.DEFAULT_WEIGHTS))
    fc_golden()
    engine_golden()
    classifier_golden()
    for f in ("fc_golden.npz", "engine_golden.npz"):
        print(f, os.path.getsize(os.path.join(OUT, f)))
