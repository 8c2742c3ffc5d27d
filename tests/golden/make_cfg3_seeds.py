"""relMSE of the REFERENCE on cfg 3 at 128^2 (const-source-disk, 256 wpp,
learnable MIS with train_until 256, and uniform) for seeds 1-8, through the
reference's own run_solve (oracle/_ref/libwost_ref_fast.so). Writes
tests/golden/ref_cfg3_seeds.json, the reference side of the cfg-3 quality
comparison (tools/cfg3_check.py, tests/test_gpu_quality.py); the committed
file holds seeds 1-31.

Runs ~40 min per 8 seeds on 8 cores: python tests/golden/make_cfg3_seeds.py [first last]
(seeds first..last, merged into the existing file; default 1-8)
"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle_lib import REF_FAST_SO, Oracle  # noqa: E402
from paper_2410_18944_b200 import abi  # noqa: E402


def main():
    ref = Oracle("ref", REF_FAST_SO)
    P = C.POINTER(C.c_double)
    first, last = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (1, 8)
    path = os.path.join(HERE, "ref_cfg3_seeds.json")
    out = {"source": "oracle/_ref/libwost_ref_fast.so run_solve, const-source-disk 128x128, 256 wpp, "
                     "train_until 256 (tests/golden/make_cfg3_seeds.py)",
           "learnable_mis": {}, "uniform": {}, "seconds_learnable": {}, "cores": os.cpu_count()}
    if os.path.exists(path):
        with open(path) as f:
            out = json.load(f)
    for seed in range(first, last + 1):
        for name, mode in (("uniform", 0), ("learnable_mis", 3)):
            st = np.zeros(128 * 128, dtype=abi.POINT_STATS_DTYPE)
            sec, rel, tsec = np.zeros(1), np.zeros(1), np.zeros(1)
            t0 = time.time()
            rc = ref.lib.ref_run_solve(b"const-source-disk", 128, 128, 256, mode, 256, seed,
                                       C.c_void_p(st.ctypes.data), sec.ctypes.data_as(P),
                                       rel.ctypes.data_as(P), tsec.ctypes.data_as(P))
            assert rc == 0
            out[name][str(seed)] = float(rel[0])
            if mode == 3:
                out["seconds_learnable"][str(seed)] = round(float(sec[0]), 1)
            print(seed, name, rel[0], f"{time.time() - t0:.1f}s", flush=True)
            with open(path, "w") as f:
                json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
