"""CPU suite: host-side logic and the C-ABI library (no GPU compute)."""
import ctypes as C
import math
import os
import re

import numpy as np
import pytest

from paper_2410_18944_b200 import _lib, abi
from paper_2410_18944_b200.scene import (PRESET_NAMES, cell_centers, make_preset, relmse,
                                         strip_vlin_solution)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "tests", "golden")


def test_presets_bit_identical_to_reference():
    g = np.load(os.path.join(G, "presets.npz"))
    for name in PRESET_NAMES:
        p = make_preset(name)
        assert np.array_equal(p.scene.seg, g[f"{name}_seg"]), name
        assert np.array_equal(p.scene.kind, g[f"{name}_kind"]), name
        assert tuple(g[f"{name}_eval_bbox"]) == tuple(p.eval_bbox)
        assert tuple(g[f"{name}_bbox"]) == tuple(p.scene.bbox)
        assert g[f"{name}_eps"][0] == p.scene.epsilon_shell


def test_cell_centers_row_major():
    # SolutionImage::cell_center, proj/include/wost/image.hpp:26-31
    pts = cell_centers(4, 2, (0.0, 0.0, 1.0, 1.0))
    assert pts.shape == (8, 2)
    assert tuple(pts[0]) == (0.125, 0.25) and tuple(pts[5]) == (0.375, 0.75)


def test_relmse_formula():
    # compute_relmse, proj/src/image.cpp:211-230: delta = (0.01 max|ref|)^2
    ref = np.array([1.0, -2.0, 0.0, 4.0])
    est = np.array([1.5, -2.0, 0.1, 4.0])
    delta = (0.01 * 4.0) ** 2
    want = (0.25 / (1.0 + delta) + 0.01 / delta) / 4
    assert relmse(est, ref) == pytest.approx(want, rel=1e-14)
    assert relmse(ref, ref) == 0.0


def test_strip_vlin_solution_boundary_values():
    assert strip_vlin_solution(0.0, 0.3) == pytest.approx(0.0, abs=1e-12)
    # truncated cosine series: slow convergence right on the x = 1 edge
    assert strip_vlin_solution(1.0, 0.3) == pytest.approx(0.3, abs=1e-4)
    assert strip_vlin_solution(0.5, 0.5) == pytest.approx(0.25, abs=1e-9)  # odd symmetry about y=1/2


def test_strip_vlin_matches_reference(ref):
    for x, y in ((0.1, 0.2), (0.5, 0.9), (0.77, 0.01)):
        assert strip_vlin_solution(x, y) == ref.lib.ref_strip_vlin_solution(x, y)


def test_library_exports_every_header_symbol():
    """libwostgpu.so exports exactly the entry points include/wostgpu.h and
    include/wostgpu3.h declare."""
    hdr = "".join(open(os.path.join(ROOT, "include", h)).read() for h in ("wostgpu.h", "wostgpu3.h"))
    declared = sorted(set(re.findall(r"\b(wostgpu_[a-z_0-9]+)\s*\(", hdr)))
    lib = C.CDLL(_lib.LIB_PATH)
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared) == set(_lib.EXPORTED_SYMBOLS), set(declared) ^ set(_lib.EXPORTED_SYMBOLS)


def test_library_is_built_for_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_no_gpu_fails_loudly():
    """Without a usable sm_100 device the C-ABI returns WG_ERR_CUDA; there is
    no CPU fallback."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = _lib.load()
    rc = lib.wostgpu_init(0)
    assert rc == abi.WG_ERR_CUDA
    assert lib.wostgpu_last_error()


def test_ctypes_struct_layouts_match_header(tmp_path):
    """The Python mirrors have the C structs' sizes (probe compiled with gcc)."""
    import subprocess
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include "%s"\nint main(){printf("%%zu %%zu %%zu %%zu %%zu '
                   '%%zu %%zu\\n", sizeof(wg_solver_config), sizeof(wg_train_config), '
                   'sizeof(wg_guide_record), sizeof(wg_point_stats), sizeof(wg_value_spec), '
                   'sizeof(wg_field_config), sizeof(wg_mixture));}\n'
                   % os.path.join(ROOT, "include", "wostgpu_types.h"))
    exe = tmp_path / "sz"
    subprocess.run(["/usr/bin/gcc", str(src), "-o", str(exe)], check=True)
    sizes = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    assert sizes == [C.sizeof(abi.SolverConfig), C.sizeof(abi.TrainConfig),
                     abi.GUIDE_RECORD_DTYPE.itemsize, abi.POINT_STATS_DTYPE.itemsize,
                     C.sizeof(abi.ValueSpec), C.sizeof(abi.FieldConfig), abi.MIXTURE_DTYPE.itemsize]
    assert abi.field_param_count(abi.field_config()) == 94433  # guide_field.hpp defaults
    src3 = tmp_path / "sz3.c"
    src3.write_text('#include <stdio.h>\n#include "%s"\nint main(){printf("%%zu %%zu\\n", '
                    'sizeof(wg_value3_spec), sizeof(wg_guide_record3));}\n'
                    % os.path.join(ROOT, "include", "wostgpu_types.h"))
    exe3 = tmp_path / "sz3"
    subprocess.run(["/usr/bin/gcc", str(src3), "-o", str(exe3)], check=True)
    sizes3 = [int(x) for x in subprocess.run([str(exe3)], capture_output=True, text=True).stdout.split()]
    assert sizes3 == [C.sizeof(abi.Value3Spec), abi.GUIDE_RECORD3_DTYPE.itemsize]
    assert C.sizeof(abi.GuideRecord3) == abi.GUIDE_RECORD3_DTYPE.itemsize


def build_cpp(out_dir, name):
    """Compile tests/cpp/<name>.cpp (a C++ caller of the facade / C-ABI) with g++."""
    import subprocess
    exe = os.path.join(str(out_dir), name)
    lib_dir = os.path.dirname(_lib.LIB_PATH)
    subprocess.run(["/usr/bin/g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", name + ".cpp"), "-o", exe, "-L", lib_dir,
                    "-lwostgpu", f"-Wl,-rpath,{lib_dir}"], check=True)
    return exe


def build_facade_demo(out_dir):
    return build_cpp(out_dir, "facade_demo")


def test_cpp_facade_compiles_and_links(tmp_path):
    assert os.path.exists(build_facade_demo(tmp_path))
    assert os.path.exists(build_cpp(tmp_path, "accel_queries"))
