"""The C-ABI library loads on a CPU-only host and exports every symbol include/ffca.h declares.

No compute calls: there is no GPU here.  (gpu-marked tests exercise them.)
"""

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "ffca.h")
LIB = os.path.join(ROOT, "paper_1805_09498_b200", "libffca_b200.so")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|void|float|const char\*)\s+(ffca_\w+)\s*\(", text, re.M)))


def test_header_declares_the_entry_points():
    names = declared()
    for must in ("ffca_fastfca_run", "ffca_fastfca_stats", "ffca_fastfca_images", "ffca_back_transform",
                 "ffca_fastfca_loglik", "ffca_fixed_point_update_P", "ffca_fca_run", "ffca_fca_estep",
                 "ffca_fca_loglik", "ffca_fca_mstep", "ffca_mstep_diag", "ffca_power_floor"):
        assert must in names


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built (run __graft_entry__.build())")
def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, f"declared in ffca.h but not exported: {missing}"


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built")
def test_binding_table_matches_header():
    from paper_1805_09498_b200 import _lib
    assert set(_lib.SIGNATURES) == set(declared())
    lib = _lib.load()
    assert lib.ffca_version() >= 100
    # no device in this container: the query must say so instead of crashing
    assert lib.ffca_device_count() >= 0


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built")
def test_plan_introspection_without_device():
    import numpy as np

    from paper_1805_09498_b200 import _lib
    lib = _lib.load()
    out = np.zeros(6, np.int32)
    # config 3 shape (c64, I=J=3, N=626), plain loop: 4 lane-interleaved bins per 128-thread CTA with the
    # y records in tensor memory (128 columns per CTA; shared memory holds only the powers)
    out8 = np.zeros(8, np.int32)
    assert lib.ffca_plan_loop(0, _lib.C64, 256, 3, 3, 626, 513, _lib.VF_AUTO, out.ctypes.data_as(_lib._ip)) == 0
    assert out[0] == 4 and out[1] == 1 and out[3] == 128 and out[4] == 1 and out[5] < 48 * 1024
    assert lib.ffca_plan_loop_ex(0, _lib.C64, 256, 3, 3, 626, 513, _lib.VF_AUTO, 1, out8.ctypes.data_as(_lib._ip)) == 0
    assert list(out8[:6]) == list(out) and out8[6] == 1 and out8[7] == 128
    # ... from one wave of 16 bins per SM on; a single mixture keeps 2 bins per CTA in shared memory
    assert lib.ffca_plan_loop_ex(0, _lib.C64, 1, 3, 3, 626, 513, _lib.VF_AUTO, 1, out8.ctypes.data_as(_lib._ip)) == 0
    assert out8[0] == 2 and out8[3] == 128 and out8[6] == 0
    # ... the loop with the likelihood record runs the same plan; a full floor array (vf_mode 2) needs the
    # shared-memory plan (2 bins per 128-thread CTA)
    assert lib.ffca_plan_loop_ex(0, _lib.C64, 256, 3, 3, 626, 513, _lib.VF_AUTO, 0, out8.ctypes.data_as(_lib._ip)) == 0
    assert out8[0] == 4 and out8[3] == 128 and out8[6] == 1
    assert lib.ffca_plan_loop_ex(0, _lib.C64, 256, 3, 3, 626, 513, 2, 0, out8.ctypes.data_as(_lib._ip)) == 0
    assert out8[0] == 2 and out8[3] == 128 and out8[4] == 1 and out8[6] == 0
    # ... and so do bins longer than the 640 frames a CTA's 128 columns hold
    assert lib.ffca_plan_loop_ex(0, _lib.C64, 256, 3, 3, 642, 513, _lib.VF_AUTO, 1, out8.ctypes.data_as(_lib._ip)) == 0
    assert out8[0] == 2 and out8[6] == 0
    # other complex64 hot shapes keep 4 lane-interleaved bins
    assert lib.ffca_plan_loop(0, _lib.C64, 64, 2, 2, 626, 513, _lib.VF_AUTO, out.ctypes.data_as(_lib._ip)) == 0
    assert out[0] == 4
    # config 2 shape (c64, I=J=4, N=9375): a cluster splits the frames
    assert lib.ffca_plan_loop(0, _lib.C64, 1, 4, 4, 9375, 1025, _lib.VF_AUTO, out.ctypes.data_as(_lib._ip)) == 0
    assert out[1] > 1 and out[4] == 1
    # config 4 shape (c64, I=8, J=6, N=4000): a CTA pair per bin, interleaved records resident
    assert lib.ffca_plan_loop(0, _lib.C64, 1, 8, 6, 4000, 2049, _lib.VF_AUTO, out.ctypes.data_as(_lib._ip)) == 0
    assert out[1] == 2 and out[4] == 1 and out[3] == 256
    # a longer 8-channel bin no longer fits a CTA quad: slab in L2-resident global scratch
    assert lib.ffca_plan_loop(0, _lib.C64, 1, 8, 6, 12000, 2049, _lib.VF_AUTO, out.ctypes.data_as(_lib._ip)) == 0
    assert out[1] == 1 and out[4] == 0 and out[3] == 256
    # complex128 (config 0 shape, 513 bins): one bin per 128-thread CTA ...
    assert lib.ffca_plan_loop(0, _lib.C128, 1, 3, 3, 626, 513, _lib.VF_AUTO, out.ctypes.data_as(_lib._ip)) == 0
    assert out[0] == 1 and out[1] == 1 and out[3] == 128
    # ... at every batch size (measured faster than 2-bin CTAs at the batched config-3 shape too)
    assert lib.ffca_plan_loop(0, _lib.C128, 256, 3, 3, 626, 513, _lib.VF_AUTO, out.ctypes.data_as(_lib._ip)) == 0
    assert out[0] == 1 and out[3] == 128


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built")
def test_every_plan_launches_whole_warps():
    # the kernels shuffle with the full mask: a CTA whose thread count is not a multiple of 32 is a bug
    # (complex128, 130 <= N <= 448 once planned 80..112-thread CTAs)
    import numpy as np

    from paper_1805_09498_b200 import _lib
    lib = _lib.load()
    out = np.zeros(8, np.int32)
    for code in (_lib.C64, _lib.C128):
        for I, J in ((1, 2), (2, 2), (3, 3), (4, 4), (3, 5), (6, 3), (8, 6)):
            for N in list(range(1, 700, 9)) + [2000, 4000, 9375, 12000]:
                for U in (1, 64):
                    for lean in (0, 1):
                        assert lib.ffca_plan_loop_ex(0, code, U, I, J, N, 513, _lib.VF_AUTO, lean,
                                                     out.ctypes.data_as(_lib._ip)) == 0
                        assert out[3] >= 32 and out[3] % 32 == 0, (code, I, J, N, U, lean, out[:6])


def test_product_has_no_cpu_fallback(monkeypatch):
    """Without a device the product path must fail loudly, never compute on the CPU."""
    import numpy as np

    from paper_1805_09498_b200 import _lib, errors, fastfca
    from paper_1805_09498_b200.stft import ObservationTensor
    if os.path.exists(LIB) and _lib.load().ffca_device_count() > 0:
        pytest.skip("a GPU is visible")
    obs = ObservationTensor(np.ones((2, 3, 4), complex))
    params = fastfca.FastFcaParams(np.broadcast_to(np.eye(2), (4, 2, 2)), np.ones((1, 4, 2)), np.ones((1, 3, 4)))
    with pytest.raises(errors.BackendUnavailable):
        fastfca.run_fastfca(obs, params, iterations=1)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1805_09498_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith(".py"):
                src = open(os.path.join(dirpath, fn)).read()
                assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, re.M), fn
