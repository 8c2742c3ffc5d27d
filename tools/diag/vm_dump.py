"""Diagnostic: dump fp32-sampler directions for one mixture to gpurun_out/."""
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2410_18944_b200 import _lib, api  # noqa: E402

_lib.init(0)
kap = float(sys.argv[1])
raw = np.zeros(33)
raw[24:32] = -30.0
raw[0], raw[1] = 1.0, 0.0
raw[16] = math.log(kap)
raw[24] = 0.0
nu = api.mixture32_sample(raw.astype(np.float32), 2_000_000, 2024)
np.save(os.path.join(ROOT, "gpurun_out", "vm_dump.npy"), nu.astype(np.float64))
