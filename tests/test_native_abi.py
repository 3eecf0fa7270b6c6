"""The C-ABI library builds, loads without a GPU, and exports every symbol
include/treescore_gpu.h declares (no compute calls here)."""

import os
import re

import numpy as np
import pytest

from conftest import has_cuda
from paper_1212_2287_b200 import _lib
from paper_1212_2287_b200._build import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "treescore_gpu.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ts_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    build()
    lib = _lib.load()
    names = header_functions()
    assert len(names) >= 8
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_lib.EXPORTS)
    assert lib.ts_version().decode().endswith("sm_100a")


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.SO_PATH], capture_output=True,
                         text=True).stdout
    archs = set(re.findall(r"sm_\d+a?", out))
    assert archs == {"sm_100a"}, archs


def test_pack_rejects_bad_models_without_gpu():
    # Validation happens before any device call, so it runs on the CPU.
    import ctypes
    import numpy as np
    lib = _lib.load()
    off = np.array([0, 3], np.int64)
    w = np.array([1.0])
    fid = np.array([5, -1, -1], np.int32)        # fid 5 >= num_features 2
    val = np.array([0.5, 1, 2], np.float32)
    lc = np.array([1, -1, -1], np.int32)
    rc = np.array([2, -1, -1], np.int32)
    desc = _lib.ModelDesc(2, 1, *[a.ctypes.data for a in (off, w, fid, val, lc, rc)])
    h = ctypes.c_void_p()
    assert lib.ts_pack(ctypes.byref(desc), 0, ctypes.byref(h)) == _lib.TS_ERR_INVALID
    assert "out of range" in _lib.last_error()
    fid[0] = 0
    val[0] = np.inf
    assert lib.ts_pack(ctypes.byref(desc), 0, ctypes.byref(h)) == _lib.TS_ERR_INVALID
    assert "finite" in _lib.last_error()


def test_package_build_is_the_reference_build_function():
    # the native-library builder is a private module, so importing it never
    # rebinds the package attribute `build` (the reference's build(ensemble, kind))
    import paper_1212_2287_b200 as pkg
    import paper_1212_2287_b200._build  # noqa: F401
    assert callable(pkg.build) and pkg.build.__module__ == "paper_1212_2287_b200.evaluator"


def _compile_example(tmp_path):
    import shutil
    import subprocess
    cc = shutil.which("cc") or shutil.which("gcc")
    if cc is None:
        pytest.skip("no C compiler")
    exe = tmp_path / "score_fvec"
    libdir = os.path.join(ROOT, "paper_1212_2287_b200")
    subprocess.run([cc, "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "score_fvec.c"), "-L", libdir,
                    "-l:_ts_gpu.so", f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    return exe


def test_c_example_compiles_against_the_header(tmp_path):
    """examples/score_fvec.c uses only include/treescore_gpu.h and the .so."""
    assert _compile_example(tmp_path).exists()


@pytest.mark.gpu
@pytest.mark.skipif(not has_cuda(), reason="needs a CUDA device")
def test_c_example_scores_golden_case(tmp_path):
    import subprocess
    from paper_1212_2287_b200 import Dataset, write_fvec
    from conftest import GOLDEN_DIR
    exe = _compile_example(tmp_path)
    g = np.load(os.path.join(GOLDEN_DIR, "mixed.npz"))
    write_fvec(tmp_path / "x.fvec", Dataset(g["X"]))
    res = subprocess.run([str(exe), os.path.join(GOLDEN_DIR, "mixed.model.txt"),
                          str(tmp_path / "x.fvec")], capture_output=True, text=True, check=True)
    got = np.array([float(v) for v in res.stdout.split()])
    assert np.array_equal(got, g["scores"])
