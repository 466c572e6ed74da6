"""CPU: the C-ABI library loads, exports every symbol include/lseforge_b200.h
declares, and rejects bad arguments with the reference's messages — all
without touching a GPU (argument checks run before any CUDA call)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lseforge_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"LF_API\s+[\w\s\*]+?\b(lf_\w+)\s*\(", src)))


def test_library_loads_and_exports_header_symbols():
    from paper_2509_09682_b200 import _capi
    L = _capi.lib()
    names = declared_symbols()
    assert len(names) >= 16
    for name in names:
        assert hasattr(L, name), name
    assert set(names) == set(_capi.EXPORTS)
    assert L.lf_abi_version() == 1


def _cfg(dtype=2, eps=0.0):
    from paper_2509_09682_b200 import _capi
    return _capi.CceConfigC(eps, dtype, 0)


def test_argument_errors_use_reference_messages():
    from paper_2509_09682_b200 import _capi
    L = _capi.lib()
    c = _cfg()
    rc = L.lf_cce_forward(None, None, None, 0, 64, 10, C.byref(c), None, None, None, None)
    assert rc == _capi.LF_EINVAL
    assert "zero rows; the mean loss is undefined" in L.lf_last_error().decode()  # losses.cpp:50
    bad = _cfg(eps=-1.0)
    rc = L.lf_cce_backward(None, None, None, None, 1.0, 4, 64, 10, C.byref(bad), None, None, None,
                           None)
    assert rc == _capi.LF_EINVAL
    assert "filter_eps must be >= 0" in L.lf_last_error().decode()  # cce.cpp:24
    odd = _cfg(dtype=2)
    rc = L.lf_cce_forward(None, None, None, 4, 48, 10, C.byref(odd), None, None, None, None)
    assert rc == _capi.LF_EUNSUPPORTED
    rc = L.lf_ccem_forward(None, None, None, 4, 8, 10, 0, C.byref(_cfg(0)), None, None, None, None)
    assert rc == _capi.LF_EINVAL
    assert "width must be at least 1" in L.lf_last_error().decode()  # neg_index.cpp:10
    with pytest.raises(ValueError, match="must all be >= 1"):
        import paper_2509_09682_b200 as lf
        lf.estimate_flops(0, 1, 1, 0, lf.Backend.kCe)


def test_estimate_flops_through_the_c_abi():
    import paper_2509_09682_b200 as lf
    assert lf.estimate_flops(25600, 256, 1000000, 0, lf.Backend.kCe).forward == 6553600000000
    e = lf.estimate_flops(100, 32, 5000, 0, lf.Backend.kCce)
    assert e.backward == 3 * e.forward
    s = lf.estimate_flops(77, 16, 4096, 63, lf.Backend.kCcem)
    f = lf.estimate_flops(77, 16, 4096, 0, lf.Backend.kCce)
    assert s.forward * 4096 == f.forward * 64


def test_python_mirror_rejects_cpu_tensors():
    import torch
    import paper_2509_09682_b200 as lf
    X = torch.zeros(4, 64)
    E = torch.zeros(10, 64)
    x = torch.zeros(4, dtype=torch.int64)
    with pytest.raises(ValueError, match="CUDA device"):
        lf.cce_forward(X, E, x)


def test_config_validation_messages():
    import paper_2509_09682_b200 as lf
    with pytest.raises(ValueError, match="block sizes must be >= 1"):
        lf.CceConfig(row_block=0).validate()
    with pytest.raises(ValueError, match="filter_eps must be >= 0"):
        lf.CceConfig(filter_eps=float("nan")).validate()
    assert lf.CceConfig.Fp16SaturationPreset().filter_eps == lf.kFp16MinPositive == 6e-8


def test_new_entry_points_validate_before_touching_the_gpu():
    from paper_2509_09682_b200 import _capi
    L = _capi.lib()
    # metrics.cpp:16-22
    assert L.lf_evaluate(None, None, None, 0, 64, 10, 10, 2, None, None, None) == _capi.LF_EINVAL
    assert "no eval pairs" in L.lf_last_error().decode()
    assert L.lf_evaluate(None, None, None, 4, 64, 10, 0, 2, None, None, None) == _capi.LF_EINVAL
    assert "k must be >= 1" in L.lf_last_error().decode()
    assert L.lf_eval_rank_topk(None, None, None, None, 4, 64, 100, 0, 17, 2, None, None, None,
                               None) == _capi.LF_EUNSUPPORTED
    # adam.cpp:14-19
    assert L.lf_adam_step(None, None, 0, None, None, 4, 1e-3, 1.0, 0.999, 1e-8, 1, None, -1,
                          None) == _capi.LF_EINVAL
    assert "betas must lie in [0, 1)" in L.lf_last_error().decode()
    assert L.lf_adam_step(None, None, 0, None, None, 4, 1e-3, 0.9, 0.999, 0.0, 1, None, -1,
                          None) == _capi.LF_EINVAL
    assert "eps must be positive" in L.lf_last_error().decode()
    # encoder.cpp:23-25 analogue
    assert L.lf_encode_batch(None, None, 1, None, None, None, 0, 4, 1, 2, None, None, None, None,
                             None, None, None) == _capi.LF_EINVAL
    assert "catalog and hidden must be >= 1" in L.lf_last_error().decode()
