"""Generate the golden fixtures in tests/golden/ from the REFERENCE library
itself (oracle/_ref/libwost_ref.so, compiled from /root/reference/proj/src by
oracle/Makefile). Run here (the reference is only present in the build
container): python tests/golden/make_golden.py

Fixtures (all small, npz):
  geometry.npz  closest_point / silhouette / ray / star radius on the
                reference unit tests' random scenes (test_geom2d.cpp seeds)
  field.npz     initial parameters digest + eval outputs of a seeded field
  walks.npz     per-walk uniform and guided estimates on presets
  train.npz     minibatch gradient + one train_batch step on fixed records
  presets.npz   preset segment arrays (make_preset)
"""
import ctypes as C
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from fixtures import Rng, probes, random_scene  # noqa: E402
from oracle_lib import Oracle  # noqa: E402
from paper_2410_18944_b200 import abi  # noqa: E402
from paper_2410_18944_b200.scene import PRESET_NAMES, cell_centers, make_preset  # noqa: E402


def main():
    ref = Oracle("ref")
    out = {}
    # ---- geometry on the reference tests' scenes
    sc = random_scene(Rng(101, 0), 1000)
    h = ref.scene(sc)
    xy = probes(Rng(1101, 0), 512, -0.2, 1.2)
    for kinds in (1, 2, 3):
        pt, d, seg = ref.closest_point(h, xy, kinds)
        out[f"cp_pt_{kinds}"], out[f"cp_d_{kinds}"], out[f"cp_seg_{kinds}"] = pt, d, seg
    out["cp_xy"] = xy
    out["sil_d"] = ref.closest_silhouette(h, xy)
    rng = Rng(14, 0)
    o = probes(rng, 512, 0.0, 1.0)
    ang = np.array([rng.uniform(0.0, 2 * np.pi) for _ in range(512)])
    d = np.stack([np.cos(ang), np.sin(ang)], 1)
    t, p, n, s, k = ref.ray_first_hit(h, o, d, 2.0, 3)
    out.update(ray_o=o, ray_d=d, ray_t=t, ray_p=p, ray_n=n, ray_seg=s, ray_kind=k)
    out["t_eps"] = np.array([ref.fn("t_epsilon")(h)])
    np.savez_compressed(os.path.join(HERE, "geometry.npz"), **out)

    # ---- field
    cfg = abi.field_config()
    f = ref.field(cfg, (0.0, 0.0, 1.0, 1.0), 1234)
    params = ref.field_params(f)
    fxy = probes(Rng(22, 0), 256, -0.2, 1.2)
    np.savez_compressed(os.path.join(HERE, "field.npz"), sha256=np.frombuffer(
        hashlib.sha256(params.tobytes()).digest(), dtype=np.uint8), params_head=params[:64],
        params_tail=params[-64:], xy=fxy, out=ref.field_eval(f, fxy, 33))

    # ---- walks (per-walk estimates, uniform and learnable MIS)
    wout = {}
    for name in ("neumann-strip-vlin", "harmonic-disk", "curves"):
        pr = make_preset(name)
        hh = ref.scene(pr.scene)
        wxy = cell_centers(16, 16, pr.eval_bbox)
        est, esc, nrec = ref.walks(hh, None, abi.solver_config("uniform"), wxy, 1, 0, records=True)
        wout[f"{name}_xy"], wout[f"{name}_uniform"], wout[f"{name}_uniform_esc"] = wxy, est, esc
        wout[f"{name}_uniform_steps"] = nrec
        ff = ref.field(cfg, pr.scene.bbox, 7)
        est, esc, _ = ref.walks(hh, ff, abi.solver_config("learnable_mis"), wxy, 1, 0)
        wout[f"{name}_guided"] = est
    np.savez_compressed(os.path.join(HERE, "walks.npz"), **wout)

    # ---- training
    pr = make_preset("curves")
    hh = ref.scene(pr.scene)
    ff = ref.field(cfg, pr.scene.bbox, 31)
    st = np.zeros(400, dtype=abi.POINT_STATS_DTYPE)
    txy = cell_centers(20, 20, pr.eval_bbox)
    recs = ref.solve_batch(hh, ff, abi.solver_config("learnable_mis"), txy, st, 7, 0, collect=True)
    tc = abi.train_config(seed=1)
    g = ref.field_grad(ff, recs[:1024], tc)
    ts = ref.train_batch(ff, recs, tc, 0)
    after = ref.field_params(ff)
    np.savez_compressed(os.path.join(HERE, "train.npz"), recs=recs, grad=g, stats_mean=st["mean"],
                        stats_m2=st["m2"], consumed=ts.records_consumed, steps=ts.steps,
                        norm=ts.mean_grad_norm, after_sha=np.frombuffer(
                            hashlib.sha256(after.tobytes()).digest(), dtype=np.uint8))

    # ---- presets
    pout = {}
    for name in PRESET_NAMES:
        nseg = C.c_int32()
        eb, sb, eps = (C.c_double * 4)(), (C.c_double * 4)(), C.c_double()
        ref.lib.ref_preset(name.encode(), None, None, C.byref(nseg), eb, sb, C.byref(eps))
        seg = np.zeros((nseg.value, 4))
        kind = np.zeros(nseg.value, dtype=np.int32)
        ref.lib.ref_preset(name.encode(), abi.ptr(seg), abi.ptr(kind, C.c_int32), C.byref(nseg), eb,
                           sb, C.byref(eps))
        pout[f"{name}_seg"], pout[f"{name}_kind"] = seg, kind
        pout[f"{name}_eval_bbox"], pout[f"{name}_bbox"] = np.array(eb[:]), np.array(sb[:])
        pout[f"{name}_eps"] = np.array([eps.value])
    np.savez_compressed(os.path.join(HERE, "presets.npz"), **pout)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
