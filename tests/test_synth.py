"""CPU: the bench's vectorised SplitMix64 instance generator
(paper_2509_09682_b200/synth.py) draws bit-for-bit the instance the
reference's make_instance builds (support.hpp:27-37, via the pinned oracle),
and derived seeds follow rng.hpp:46-48."""
import numpy as np
import pytest

import oracle_bind as ob
from paper_2509_09682_b200 import synth


@pytest.mark.parametrize("n,d,v,hw", [(1, 1, 1, 1.0), (37, 5, 101, 1.0), (300, 64, 4096, 2.0),
                                      (1000, 64, (1 << 20) | 5, 1.0), (64, 3, 3, 0.5)])
def test_make_instance_bitwise(n, d, v, hw):
    for seed in (0xB2000002, 7):
        E, C, t = synth.make_instance(seed, n, d, v, hw)
        inst = ob.make_instance(ob.Rng(seed), n, d, v, hw)
        assert np.array_equal(E, inst.E) and np.array_equal(C, inst.C)
        assert np.array_equal(t, inst.targets)


def test_draws_and_derived_seed():
    seed = 0xB2000003
    r = ob.Rng(seed)
    assert [int(x) for x in synth.draws(seed, 0, 5)] == [r.next() for _ in range(5)]
    # derived(i) opens SplitMix64(mix(seed + golden (i + 1))) (rng.hpp:46-48):
    # its first draw equals draw 1 of the derived seed's own stream
    s7 = synth.derived_seed(seed, 7)
    assert s7 == int(synth.mix(np.uint64((seed + 0x9E3779B97F4A7C15 * 8) % (1 << 64))))
    assert int(synth.draws(s7, 0, 1)[0]) == ob.Rng(s7).next()
