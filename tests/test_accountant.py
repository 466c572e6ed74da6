"""CPU: MemAccountant mirror (accountant.hpp:25-82) and the retained-memory
arithmetic of the paper (test_memory.cpp:35-56)."""
import pytest

from paper_2509_09682_b200 import MemAccountant, ScalarKind


def test_retained_vs_scratch_classes_and_peaks():
    a = MemAccountant()
    a.record_alloc("retained/cce/lse", 10)
    a.record_alloc("scratch/x", 5)
    a.record_alloc("scratch/y", 7)
    a.record_free("scratch/x", 5)
    a.record_alloc("retained/ccem/inds", 3, ScalarKind.kIndex)
    r = a.report()
    assert r.current.retained_real == 10 and r.current.scratch_real == 7
    assert r.peak.scratch_real == 12 and r.current.retained_index == 3
    assert r.retained_bytes(4) == 10 * 4 + 3 * 8
    with pytest.raises(RuntimeError, match="scratch tag 'scratch/y' still holds 7"):
        a.expect_scratch_released()
    a.record_free("scratch/y", 7)
    a.expect_scratch_released()


def test_record_ensure_charges_only_the_missing_part():
    a = MemAccountant()
    a.record_ensure("retained/cce/lse", 8)
    a.record_ensure("retained/cce/lse", 8)
    a.record_ensure("retained/cce/lse", 10)
    assert a.live("retained/cce/lse") == 10
    assert a.report().peak.retained_real == 10


def test_misuse_raises():
    a = MemAccountant()
    with pytest.raises(ValueError, match="never allocated"):
        a.record_free("scratch/z", 1)
    a.record_alloc("t", 1)
    with pytest.raises(ValueError, match="different scalar kind"):
        a.record_alloc("t", 1, ScalarKind.kIndex)


def test_free_prefix():
    a = MemAccountant()
    a.record_alloc("retained/a/x", 2)
    a.record_alloc("retained/a/y", 3)
    a.record_alloc("retained/b/z", 4)
    a.record_free_prefix("retained/a/")
    assert a.report().current.retained_real == 4


def test_paper_logit_memory_arithmetic():
    """test_memory.cpp:35-56: bs*sl = 25600 rows x 1M items of fp32 logits is
    102.4 GB; CCE retains 2N scalars (pos + lse)."""
    n, v = 256 * 100, 1_000_000
    assert n * v * 4 == 102_400_000_000
    assert 2 * n * 4 == 204_800
