"""GPU: the device Adam (lf_adam_step) reproduces AdamState::step
(adam.cpp:22-55) bit for bit — against the golden fixture made by the
reference itself (tests/golden/adam_ref.npz) and the C oracle — for f64 and
f32 gradients, with the fused bf16 shadow equal to the rounded parameters."""
import os

import numpy as np
import pytest
import torch

import oracle_bind as ob

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def lf(cuda):
    import paper_2509_09682_b200 as lf
    return lf


def test_matches_reference_golden(lf):
    g = np.load(os.path.join(GOLDEN, "adam_ref.npz"))
    lr, b1, b2, eps = (float(x) for x in g["hp"])
    p = torch.from_numpy(g["p0"].copy()).cuda()
    opt = lf.DeviceAdam([p], lf.AdamConfig(lr, b1, b2, eps))
    for gr in g["grads"]:
        opt.step([torch.from_numpy(gr).cuda()])
    assert opt.steps_taken == len(g["grads"])
    assert np.array_equal(p.cpu().numpy(), g["want"])


@pytest.mark.parametrize("gdt", [torch.float64, torch.float32])
def test_matches_oracle_with_shadow(lf, gdt):
    rng = np.random.default_rng(3)
    v, d = 100_003, 64
    p0 = (rng.standard_normal(v * d) * 0.05).astype(np.float32)
    p = torch.from_numpy(p0.copy()).cuda().view(v, d)
    sh = torch.empty(v, d, dtype=torch.bfloat16, device="cuda")
    opt = lf.DeviceAdam([p], lf.AdamConfig(lr=3e-3))
    ph, m, vv = p0.copy(), np.zeros(v * d), np.zeros(v * d)
    for t in range(1, 4):
        gr = (rng.standard_normal(v * d) * 10.0 ** rng.integers(-7, 1, v * d))
        gr = gr.astype(np.float32).astype(np.float64) if gdt == torch.float32 else gr
        opt.step([torch.from_numpy(gr).to(gdt).cuda().view(v, d)], [sh])
        ob.adam_apply(ph, gr, m, vv, 3e-3, 0.9, 0.999, 1e-8, t)
    assert np.array_equal(p.cpu().numpy().reshape(-1), ph)
    assert torch.equal(sh, p.to(torch.bfloat16))
    assert np.array_equal(opt.m[0].cpu().numpy().reshape(-1), m)
    assert np.array_equal(opt.v[0].cpu().numpy().reshape(-1), vv)


def test_errors(lf):
    p = torch.zeros(4, device="cuda")
    with pytest.raises(ValueError, match="betas"):
        lf.DeviceAdam([p], lf.AdamConfig(beta1=1.0))
    with pytest.raises(ValueError, match="eps must be positive"):
        lf.DeviceAdam([p], lf.AdamConfig(eps=0.0))
    opt = lf.DeviceAdam([p])
    with pytest.raises(ValueError, match="gradient shapes"):
        opt.step([torch.zeros(5, device="cuda")])
