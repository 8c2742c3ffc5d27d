"""Per-point statistics of the REFERENCE on cfg 2 (neumann-strip-vlin, 128^2
cell centres, 256 wpp, seed 1) for the uniform sampler and for learnable MIS
with online training (train_until 256), through the reference's own run_solve
(oracle/_ref/libwost_ref_fast.so). Stored as tests/golden/ref_cfg2_<mode>_seed1.npz
with the mean and the standard error of every point, for the "per-point
estimates agree within 3 MC standard errors" parity check
(tests/test_gpu_quality.py, tools/quality_cfg2.py).

Runs ~1-2 min on 8 cores: python tests/golden/make_cfg2_reference.py
"""
import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle_lib import REF_FAST_SO, Oracle  # noqa: E402
from paper_2410_18944_b200 import abi  # noqa: E402


def main():
    ref = Oracle("ref", REF_FAST_SO)
    for name, mode in (("uniform", 0), ("learnable", 3)):
        st = np.zeros(128 * 128, dtype=abi.POINT_STATS_DTYPE)
        sec, rel, tsec = np.zeros(1), np.zeros(1), np.zeros(1)
        P = C.POINTER(C.c_double)
        rc = ref.lib.ref_run_solve(b"neumann-strip-vlin", 128, 128, 256, mode, 256, 1,
                                   C.c_void_p(st.ctypes.data), sec.ctypes.data_as(P),
                                   rel.ctypes.data_as(P), tsec.ctypes.data_as(P))
        assert rc == 0
        c = st["count"].astype(np.float64)
        se = np.sqrt(st["m2"] / (c * (c - 1)))
        np.savez_compressed(os.path.join(HERE, f"ref_cfg2_{name}_seed1.npz"), mean=st["mean"], se=se,
                            escaped=st["escaped"], relmse=rel, seconds=sec)
        print(name, "relmse", rel[0], "seconds", sec[0], "escaped", int(st["escaped"].sum()))


if __name__ == "__main__":
    main()
