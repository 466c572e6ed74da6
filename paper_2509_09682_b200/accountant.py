"""MemAccountant — logical peak-memory ledger of the loss layer.

Host-side mirror of proj/include/lseforge/accountant.hpp:25-82 and
proj/src/accountant.cpp (same tag semantics, same exceptions): buffers tagged
``retained/...`` outlive the op; every other tag is scratch that must be freed
before the op returns.  Counts are scalars; ``Report.retained_bytes`` applies
the dtype width (indices always 8 bytes, accountant.hpp:15).
"""
from __future__ import annotations

import enum
from dataclasses import dataclass, field
from typing import Dict

K_INDEX_BYTES = 8  # accountant.hpp:15


class ScalarKind(enum.Enum):  # accountant.hpp:12
    kReal = 0
    kIndex = 1


@dataclass
class TagStat:
    current: int = 0
    peak: int = 0
    kind: ScalarKind = ScalarKind.kReal


@dataclass
class Totals:
    retained_real: int = 0
    retained_index: int = 0
    scratch_real: int = 0
    scratch_index: int = 0

    def _key(self, retained: bool, kind: ScalarKind) -> str:
        return ("retained_" if retained else "scratch_") + (
            "real" if kind == ScalarKind.kReal else "index")


@dataclass
class Report:
    tags: Dict[str, TagStat] = field(default_factory=dict)
    current: Totals = field(default_factory=Totals)
    peak: Totals = field(default_factory=Totals)

    def retained_bytes(self, dtype_bytes: int) -> int:  # accountant.hpp:41-44
        return self.peak.retained_real * dtype_bytes + self.peak.retained_index * K_INDEX_BYTES

    def scratch_bytes(self, dtype_bytes: int) -> int:  # accountant.hpp:45-48
        return self.peak.scratch_real * dtype_bytes + self.peak.scratch_index * K_INDEX_BYTES


class MemAccountant:
    def __init__(self):
        self.reset()

    @staticmethod
    def _is_retained(tag: str) -> bool:  # accountant.cpp:9
        return tag.startswith("retained/")

    def record_alloc(self, tag: str, scalars: int, kind: ScalarKind = ScalarKind.kReal):
        st = self._tags.get(tag)
        if st is None:
            st = self._tags[tag] = TagStat(0, 0, kind)
        elif st.kind != kind:  # accountant.cpp:15-17
            raise ValueError(f"MemAccountant::record_alloc: tag '{tag}' reused with a different "
                             "scalar kind")
        st.current += scalars
        st.peak = max(st.peak, st.current)
        key = self._current._key(self._is_retained(tag), kind)
        cur = getattr(self._current, key) + scalars
        setattr(self._current, key, cur)
        setattr(self._peak, key, max(getattr(self._peak, key), cur))

    def record_free(self, tag: str, scalars: int, kind: ScalarKind = ScalarKind.kReal):
        st = self._tags.get(tag)
        if st is None or st.kind != kind or st.current < scalars:  # accountant.cpp:36-40
            raise ValueError(f"MemAccountant::record_free: tag '{tag}' freeing {scalars} scalars "
                             "that were never allocated")
        st.current -= scalars
        key = self._current._key(self._is_retained(tag), kind)
        setattr(self._current, key, getattr(self._current, key) - scalars)

    def record_ensure(self, tag: str, scalars: int, kind: ScalarKind = ScalarKind.kReal):
        have = self.live(tag)  # accountant.cpp:50-53
        if have < scalars:
            self.record_alloc(tag, scalars - have, kind)

    def record_free_prefix(self, prefix: str):
        pending = [(t, s.current, s.kind) for t, s in sorted(self._tags.items())
                   if s.current > 0 and t.startswith(prefix)]
        for t, c, k in pending:
            self.record_free(t, c, k)

    def live(self, tag: str) -> int:
        st = self._tags.get(tag)
        return 0 if st is None else st.current

    def report(self) -> Report:
        import copy
        return Report(copy.deepcopy(self._tags), copy.deepcopy(self._current),
                      copy.deepcopy(self._peak))

    def expect_scratch_released(self):  # accountant.cpp:70-77 (std::logic_error)
        for tag, st in sorted(self._tags.items()):
            if not self._is_retained(tag) and st.current != 0:
                raise RuntimeError(f"MemAccountant: scratch tag '{tag}' still holds "
                                   f"{st.current} scalars")

    def reset(self):
        self._tags: Dict[str, TagStat] = {}
        self._current = Totals()
        self._peak = Totals()
