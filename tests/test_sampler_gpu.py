"""GPU: the device uniform sampler reproduces the reference's sample_uniform
(proj/src/sampler.cpp:44-75) index for index — checked against the C oracle
(oracle/oracle.c, itself pinned to the reference) and, when the in-place
reference build travelled with the snapshot, against the reference itself."""
import os

import numpy as np
import pytest
import torch

import oracle_bind as ob

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lf(cuda):
    import paper_2509_09682_b200 as lf
    return lf


@pytest.mark.parametrize("n,ns,catalog,seed", [(1, 5, 7, 0), (300, 63, 4096, 0xB2000003),
                                               (777, 512, 1000000, 42), (64, 1, 2, 9),
                                               (50, 0, 10, 3), (40, 31, 33, 0xDEADBEEF)])
def test_matches_oracle_exactly(lf, n, ns, catalog, seed):
    rng = ob.Rng(seed ^ 0x55)
    pos = np.array([rng.bounded(catalog) for _ in range(n)], dtype=np.int64)
    want = ob.sample_uniform(pos, ns, catalog, seed)
    got = lf.sample_uniform(torch.from_numpy(pos).cuda(), ns, catalog, seed).cpu().numpy()
    assert got.shape == (n, 1 + ns)
    assert np.array_equal(got, want)
    if os.path.exists(os.path.join(ROOT, "oracle", "_ref", "liblseforge_ref.so")):
        assert np.array_equal(got, ob.ref_sample_uniform(pos, ns, catalog, seed))


def test_errors_use_reference_messages(lf):
    pos = torch.tensor([0, 9, 2], dtype=torch.int64, device="cuda")
    with pytest.raises(ValueError, match="row 1 positive 9 outside catalog of 8"):
        lf.sample_uniform(pos, 2, 8, 1)
    with pytest.raises(ValueError, match="exceeds catalog minus positive"):
        lf.sample_uniform(pos, 10, 10, 1)


def test_feeds_ccem_directly(lf):
    """Device-sampled indices drive CCE- without a host round trip; the loss
    equals the oracle's on the same (bit-identical) index matrix."""
    n, d, v, ns = 256, 64, 8192, 127
    inst = ob.make_instance(ob.Rng(0xB2000004), n, d, v)
    X = torch.from_numpy(inst.E).cuda().to(torch.bfloat16)
    E = torch.from_numpy(np.ascontiguousarray(inst.C.T)).cuda().to(torch.bfloat16)
    x = torch.from_numpy(inst.targets).cuda()
    inds = lf.sample_uniform(x, ns, v, 0xB2000003)
    out = lf.ccem_forward(X, E, inds)
    Eh, Ch = X.float().cpu().numpy(), E.float().cpu().numpy().T.copy()
    loss, _, _ = ob.ccem_forward(Eh, Ch, inds.cpu().numpy())
    assert abs(float(out.loss) - loss) <= 1e-2 * max(1.0, abs(loss))
