"""Batched 3D queries on the cfg-4 mesh for per-query kernel timing (ncu
gpu__time_duration of cp3_kernel / sil3_kernel / ray3_kernel / star3_kernel):
1M probes uniform in the box interior, rays with t_max = the star radius."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2410_18944_b200 import abi  # noqa: E402
from paper_2410_18944_b200._lib import init  # noqa: E402
from paper_2410_18944_b200.api3 import Accel3  # noqa: E402
from paper_2410_18944_b200.scene3 import make_preset3  # noqa: E402

init(0)
n = 1 << 20
rng = np.random.default_rng(1)
x = rng.uniform(0.01, 0.99, (n, 3))
d = rng.normal(size=(n, 3))
d /= np.linalg.norm(d, axis=1)[:, None]
acc = Accel3(make_preset3("box-strip-vlin").scene)
print(acc.info())
for _ in range(2):
    acc.closest_point(x, abi.KIND_DIRICHLET)
    acc.closest_silhouette(x)
    r = acc.star_radius(x, 1e-3)
    acc.ray_first_hit(x, d, r, abi.KIND_NEUMANN)
