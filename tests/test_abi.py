"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every symbol include/qvg.h declares, and the host mirror validates like the
reference — without running any GPU compute."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "qvg.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(qvg_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("qvg_index_create", "qvg_index_load", "qvg_search", "qvg_search_ex",
              "qvg_beam_search", "qvg_encode", "qvg_index_destroy", "qvg_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2605_02171_b200 import _native as N
    lib = ctypes.CDLL(N.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(N.EXPORTED_SYMBOLS) == set(declared_symbols())


def test_library_is_sm100a_and_static_cudart():
    from paper_2605_02171_b200 import _native as N
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", N.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    deps = subprocess.run(["ldd", N.LIB_PATH], capture_output=True, text=True).stdout
    assert "libcudart" not in deps


def test_abi_version_and_error_channel():
    from paper_2605_02171_b200 import _native as N
    L = N.lib()
    assert L.qvg_abi_version() == 1
    # null-argument validation runs before any CUDA call
    h = ctypes.c_void_p()
    rc = L.qvg_index_create(None, 0, 0, None, 0, None, 0, 0, ctypes.byref(h))
    assert rc == N.QVG_INVALID_ARGUMENT
    assert "null" in N.last_error()


def test_search_params_validate_like_reference():
    from paper_2605_02171_b200 import InvalidArgument, SearchParams
    SearchParams(64, 10).validate()
    with pytest.raises(InvalidArgument, match="k must be >= 1"):
        SearchParams(ef=4, k=0).validate()
    with pytest.raises(InvalidArgument, match="ef must be >= k"):
        SearchParams(ef=4, k=5).validate()
    assert issubclass(InvalidArgument, ValueError)


def test_package_has_no_oracle_dependency():
    """The product never imports or links the checker."""
    pkg = os.path.join(ROOT, "paper_2605_02171_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "libqivr_ref" not in src and "liboracle" not in src, f


def test_dataset_generator_is_seeded_and_unit_norm():
    from workloads.datasets import mixture
    a, qa = mixture(500, 96, 10, 0.3, seed=1, nq=20)
    b, qb = mixture(500, 96, 10, 0.3, seed=1, nq=20)
    assert np.array_equal(a, b) and np.array_equal(qa, qb)
    assert np.allclose(np.linalg.norm(a, axis=1), 1.0, atol=1e-5)
    c, _ = mixture(500, 96, 10, 0.3, seed=2)
    assert not np.array_equal(a, c)
    d, _ = mixture(200, 64, 5, 0.25, seed=3, aniso=True)
    assert d.shape == (200, 64)


def test_reference_arm_never_loads_the_product_library():
    """bench.py --impl reference imports only workloads/ and oracle/: the CUDA
    library must not be dlopen'ed in that process (driver: native_so_loaded)."""
    import subprocess
    import sys
    code = ("import sys; sys.argv=['bench.py']; sys.path.insert(0, %r)\n"
            "import bench\n"
            "from workloads import datasets, graphs\n"
            "from oracle import oracle\n"
            "bad = [m for m in sys.modules if m.startswith('paper_2605_02171_b200')]\n"
            "maps = open('/proc/self/maps').read()\n"
            "assert not bad, bad\n"
            "assert 'libqvg.so' not in maps\n"
            "print('clean')\n") % ROOT
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 0 and "clean" in r.stdout, r.stderr[-2000:]


def test_tensor_inputs_are_validated_before_any_launch():
    """Raw-pointer hand-off of torch tensors: wrong dtype, non-contiguous
    layout or wrong row width is rejected on the host."""
    import torch

    import paper_2605_02171_b200 as Q
    f = Q._f32
    with pytest.raises(Q.InvalidArgument, match="dtype"):
        f(torch.zeros((4, 8), dtype=torch.float16), 8)
    with pytest.raises(Q.InvalidArgument, match="dtype"):
        f(torch.zeros((4, 8), dtype=torch.float64), 8)
    with pytest.raises(Q.InvalidArgument, match="contiguous"):
        f(torch.zeros((8, 4), dtype=torch.float32).t(), 8)
    with pytest.raises(Q.InvalidArgument, match="dimension"):
        f(torch.zeros((4, 7), dtype=torch.float32), 8)
    with pytest.raises(Q.InvalidArgument, match="dimension"):
        f(np.zeros((4, 7), np.float32), 8)
    ok = torch.zeros((4, 8), dtype=torch.float32)
    assert f(ok, 8) is ok
    with pytest.raises(Q.InvalidArgument, match=">= 40"):
        Q._out(torch.zeros(39, dtype=torch.int32), (4, 10), ("uint32", "int32"), "ids")
    with pytest.raises(Q.InvalidArgument):
        Q._out(np.zeros((4, 10), np.float64), (4, 10), ("float32",), "scores")
