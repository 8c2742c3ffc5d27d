"""Guided training rounds on any preset (like tools/profile_cfg2.py) for the
phase / sub-phase profilers: python tools/profile_scene.py PRESET [--grid G]
[--rounds R] [--warmup-rounds W]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2410_18944_b200 import abi, api  # noqa: E402
from paper_2410_18944_b200.scene import cell_centers, make_preset  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("preset")
ap.add_argument("--grid", type=int, default=128)
ap.add_argument("--rounds", type=int, default=4)
ap.add_argument("--warmup-rounds", type=int, default=32)
a = ap.parse_args()
p = make_preset(a.preset)
pts = cell_centers(a.grid, a.grid, p.eval_bbox)
f = api.GuidingField(abi.field_config(), p.scene.bbox, 1)
s = api.Solver(api.Accel(p.scene), f, abi.solver_config("learnable_mis"), api.MLP_TENSOR)
s.set_points(pts)
if a.warmup_rounds:
    s.run(1, a.warmup_rounds, 256, abi.train_config(seed=1))  # a trained field: realistic walks
st, ms = s.run(2, a.rounds, 256, abi.train_config(seed=1))
prof = s.run_profile()
print(f"per round: walk {prof['walk_ms'] / a.rounds:.3f} ms, train {prof['train_ms'] / a.rounds:.3f} ms, "
      f"steps/walk {prof['steps'] / max(prof['walks'], 1):.1f}")
