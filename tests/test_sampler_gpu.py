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


GOLDEN = os.path.join(ROOT, "tests", "golden")


def test_popularity_matches_reference_golden(lf):
    g = np.load(os.path.join(GOLDEN, "popularity_ref.npz"))
    for c in range(int(g["count"])):
        if float(g[f"{c}_exp"]) != 1.0:
            continue  # device pow may differ from glibc's in the last ulp (documented)
        got = lf.sample_popularity(torch.from_numpy(g[f"{c}_pos"]).cuda(), int(g[f"{c}_ns"]),
                                   torch.from_numpy(g[f"{c}_counts"]), int(g[f"{c}_seed"])).cpu().numpy()
        assert np.array_equal(got, g[f"{c}_inds"])


@pytest.mark.parametrize("cat,n,ns,seed", [(1_000_000, 2048, 512, 3), (50, 300, 49, 9), (2, 10, 1, 1)])
def test_popularity_matches_oracle(lf, cat, n, ns, seed):
    rng = np.random.default_rng(seed)
    counts = rng.integers(0, 100, cat).astype(np.int64)
    pos = rng.integers(0, cat, n).astype(np.int64)
    counts[pos] += 1  # keep positives drawable; other items may have weight 0
    if cat == 2:
        counts[:] = 5
    want = ob.sample_popularity(pos, ns, counts, seed)
    got = lf.sample_popularity(torch.from_numpy(pos).cuda(), ns, torch.from_numpy(counts), seed).cpu().numpy()
    assert np.array_equal(got, want)


def test_popularity_errors(lf):
    pos = torch.tensor([0, 1], device="cuda")
    with pytest.raises(ValueError, match="all item weights are zero"):
        lf.sample_popularity(pos, 1, torch.zeros(5, dtype=torch.int64), 1)
    with pytest.raises(ValueError, match="item 2 has negative count -3"):
        lf.sample_popularity(pos, 1, torch.tensor([1, 1, -3, 1]), 1)
    with pytest.raises(ValueError, match="exceeds catalog minus positive"):
        lf.sample_popularity(pos, 4, torch.ones(4, dtype=torch.int64), 1)
    with pytest.raises(RuntimeError, match="rejection retries"):
        # only the positive has weight: every draw is rejected
        lf.sample_popularity(torch.tensor([0], device="cuda"), 1, torch.tensor([5, 0, 0]), 1, retry_cap=7)
