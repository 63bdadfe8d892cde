"""Host-side checks of the C-ABI library (no GPU compute): it loads and exports every
symbol include/cavs.h declares; host-only entry points behave."""
import ctypes
import os
import re

import pytest

from workloads import gen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "cavs.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cavs_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_1712_04048_b200 as pkg
    lib = ctypes.CDLL(pkg.LIB_PATH)
    names = _declared()
    assert len(names) >= 13
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(pkg.EXPORTS) == names


@pytest.mark.parametrize("cell,N,h,d", [("tree_lstm", 2, 512, 512), ("tree_lstm", 1, 16, 8),
                                        ("tree_fc", 2, 2048, 2048), ("tree_fc", 2, 16, 3)])
def test_param_count_matches_packed_layout(cell, N, h, d):
    import paper_1712_04048_b200 as pkg
    assert pkg.param_count(cell, N, h, d) == gen.n_params(cell, N, h, d)


def test_create_rejects_bad_descriptors_without_gpu():
    import paper_1712_04048_b200 as pkg
    from paper_1712_04048_b200.cavs import _Desc
    lib = pkg.lib()
    out = ctypes.c_void_p()
    bad = [_Desc(7, 2, 16, 16, 0, 1, 10, 10), _Desc(0, 0, 16, 16, 0, 1, 10, 10),
           _Desc(0, 2, 16, 16, 9, 1, 10, 10), _Desc(1, 3, 16, 16, 0, 1, 10, 10),
           _Desc(0, 2, 100, 64, 1, 1, 10, 10)]
    codes = [lib.cavs_create(ctypes.byref(b), 0, None, ctypes.byref(out)) for b in bad]
    assert codes == [1, 1, 1, 8, 8]


def test_binding_rejects_wrong_dtypes_and_devices():
    """int64 index arrays / CPU tensors must not reach the C-ABI as raw pointers."""
    import numpy as np
    import torch
    from paper_1712_04048_b200.cavs import _ptr
    with pytest.raises(TypeError):
        _ptr(np.zeros(4, np.int64), "i32")
    with pytest.raises(TypeError):
        _ptr(torch.zeros(4, dtype=torch.int64), "i32")
    with pytest.raises(TypeError):                      # CPU tensor where a device pointer is required
        _ptr(torch.zeros(4, dtype=torch.float32), "f32", torch.device("cuda", 0))
    assert _ptr(np.zeros(4, np.int32), "i32") != 0
    assert _ptr(torch.zeros(4, dtype=torch.float32), "f32", torch.device("cuda", 0), host_ok=True) != 0
