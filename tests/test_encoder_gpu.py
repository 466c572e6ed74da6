"""GPU: encode_batch / encoder_backward on the device (lf_encoder.cu) against
the reference's own outputs (tests/golden/encoder_ref.npz, made by running
encoder.cpp) and the C oracle: pooled means bitwise; h within 2 ulp (CUDA's
tanh vs glibc's); gradients within 1e-12 relative (they inherit h's last bit)."""
import os

import numpy as np
import pytest
import torch

import oracle_bind as ob

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def enc(cuda):
    from paper_2509_09682_b200 import encoder
    return encoder


def _run(enc, emb, W, b, items, win_off, dh, x_dtype=torch.float64):
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    batch = enc.encode_batch(t(emb), t(W), t(b), t(items), t(win_off), x_dtype)
    grads = enc.encoder_backward(emb.shape[0], t(W), batch, t(dh))
    return batch, grads


def _close(got, want, rel):
    scale = max(1.0, float(np.abs(want).max()))
    assert np.abs(got - want).max() <= rel * scale, np.abs(got - want).max()


def test_matches_reference_golden(enc):
    g = np.load(os.path.join(GOLDEN, "encoder_ref.npz"))
    batch, (d_emb, d_W, d_b) = _run(enc, g["emb"], g["W"], g["b"], g["items"], g["win_off"], g["dh"])
    assert np.array_equal(batch.a.cpu().numpy(), g["a"])
    assert np.array_equal(batch.targets.cpu().numpy(), g["targets"])
    h = batch.h.cpu().numpy()
    assert np.abs(h - g["h"]).max() <= 4 * np.finfo(np.float64).eps
    assert np.array_equal(batch.X.cpu().numpy().astype(np.float32), g["e"]) or \
        np.abs(batch.X.cpu().numpy() - g["e"]).max() <= 1e-7
    _close(d_W.cpu().numpy(), g["d_W"], 1e-12)
    _close(d_b.cpu().numpy(), g["d_b"], 1e-12)
    _close(d_emb.cpu().numpy(), g["d_emb"], 1e-12)


@pytest.mark.parametrize("cat,d,nw,maxlen", [(1000, 64, 256, 50), (77, 128, 9, 3), (5, 256, 4, 9)])
def test_matches_oracle(enc, cat, d, nw, maxlen):
    rng = np.random.default_rng(cat + d)
    emb = (rng.standard_normal((cat, d)) * 0.2).astype(np.float32)
    W = (rng.standard_normal((d, d)) * 0.2).astype(np.float32)
    b = (rng.standard_normal(d) * 0.1).astype(np.float32)
    lens = rng.integers(2, maxlen + 1, nw)
    win_off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    items = rng.integers(0, cat, int(win_off[-1])).astype(np.int64)
    dh = rng.standard_normal((int(np.sum(lens - 1)), d))
    o = ob.encoder(emb, W, b, items, win_off, dh)
    batch, (d_emb, d_W, d_b) = _run(enc, emb, W, b, items, win_off, dh, torch.bfloat16)
    assert np.array_equal(batch.a.cpu().numpy(), o["a"])
    assert np.abs(batch.h.cpu().numpy() - o["h"]).max() <= 4 * np.finfo(np.float64).eps
    assert torch.equal(batch.X, torch.from_numpy(o["e"]).cuda().to(torch.bfloat16))
    assert np.array_equal(batch.position_of.cpu().numpy(), o["row_pos"])
    _close(d_W.cpu().numpy(), o["d_W"], 1e-12)
    _close(d_b.cpu().numpy(), o["d_b"], 1e-12)
    _close(d_emb.cpu().numpy(), o["d_emb"], 1e-12)


def test_errors(enc):
    emb = torch.zeros(10, 4, device="cuda")
    W = torch.zeros(4, 4, device="cuda")
    b = torch.zeros(4, device="cuda")
    with pytest.raises(ValueError, match="at least 2 items"):
        enc.encode_batch(emb, W, b, torch.tensor([1, 2, 3], device="cuda"),
                         torch.tensor([0, 2, 3], device="cuda"))
    with pytest.raises(ValueError, match="outside catalog of size 10"):
        enc.encode_batch(emb, W, b, torch.tensor([1, 12], device="cuda"), torch.tensor([0, 2], device="cuda"))
