"""Per-point statistics of the REFERENCE on cfg 3 at its configured size
(const-source-disk 512^2, 256 wpp, learnable MIS with train_until 256,
seed 1) through the reference's own run_solve (oracle/_ref/libwost_ref_fast.so).
Writes tests/golden/ref_cfg3_512_seed1.npz (per-point mean and standard
error as float32, relMSE, seconds): the reference side of the cfg-3 parity
test that runs the product's wavefront pair (tests/test_gpu_quality.py).

Runs ~2 h on 8 cores: python tests/golden/make_cfg3_512.py
"""
import ctypes as C
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
    g, seed = 512, 1
    st = np.zeros(g * g, dtype=abi.POINT_STATS_DTYPE)
    sec, rel, tsec = np.zeros(1), np.zeros(1), np.zeros(1)
    t0 = time.time()
    rc = ref.lib.ref_run_solve(b"const-source-disk", g, g, 256, 3, 256, seed, C.c_void_p(st.ctypes.data),
                               sec.ctypes.data_as(P), rel.ctypes.data_as(P), tsec.ctypes.data_as(P))
    assert rc == 0, ref.fn("last_error")()
    c = st["count"].astype(np.float64)
    se = np.sqrt(st["m2"] / (c * (c - 1)))
    np.savez_compressed(os.path.join(HERE, "ref_cfg3_512_seed1.npz"), mean=st["mean"].astype(np.float32),
                        se=se.astype(np.float32), escaped=st["escaped"].astype(np.int32),
                        relmse=np.array([rel[0]]), seconds=np.array([sec[0]]),
                        train_seconds=np.array([tsec[0]]), cores=np.array([os.cpu_count()]))
    print("relmse", rel[0], "seconds", sec[0], f"wall {time.time() - t0:.0f}s", flush=True)


if __name__ == "__main__":
    main()
