"""Traversal work per query type on the cfg-4 shape (diagnostic build with
-DWG3_COUNT: WOSTGPU_LIB=paper_2410_18944_b200/libwostgpu_dbg.so)."""
import ctypes as C
import os
import sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2410_18944_b200 import _lib, abi
from paper_2410_18944_b200.api3 import MLP_TENSOR, Accel3, GuidingField3, Solver3
from paper_2410_18944_b200.scene3 import make_preset3, slice_points
lib = _lib.load()
out = (C.c_ulonglong * 16)()
p = make_preset3("box-strip-vlin")
f = GuidingField3(abi.field_config3(), (0, 0, 0, 1, 1, 1), 1)
s = Solver3(Accel3(p.scene), f, abi.solver_config("learnable_mis"), MLP_TENSOR)
s.set_points(slice_points(512, 512))
s.run(1, 4, 0, None)
lib.wostgpu_debug_counts3(out, 1)
s.run(1, 8, 0, None)
lib.wostgpu_debug_counts3(out, 0)
c = list(out)
steps = s.run_profile()["steps"]
for name, i in (("cp", 0), ("sil", 3), ("ray", 6)):
    print(f"{name}: queries {c[i]} per step {c[i] / steps:.2f}; interior visits / query {c[i + 1] / max(c[i], 1):.2f}; "
          f"primitive tests / query {c[i + 2] / max(c[i], 1):.2f}")
print("steps", steps)
