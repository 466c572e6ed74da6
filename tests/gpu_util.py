"""Shared helpers for the GPU parity tests (test infrastructure)."""
import numpy as np
import torch

import oracle_bind as ob

# Stated tolerances (north star + SURVEY.md §8(c)):
#   f64 "exact": reference rel_err (|got-want|/max(1,|want|)) < 1e-6, pos bitwise.
#   f32: loss rel 1e-5; dX/dE per element |d| <= 1e-4|want| + 1e-6 max|want|.
#   bf16: loss rel 1e-2 (north star); dX/dE normwise <= 1e-2 and per element
#         |d| <= 2e-2|want| + 1e-2 max|want| (G is rounded to bf16 before the
#         tensor-core GEMM, fp32 accumulate).
TOL = {
    torch.float64: dict(loss=1e-6, lse=1e-6, grad_rel=1e-6, grad_abs=0.0, norm=1e-6),
    torch.float32: dict(loss=1e-5, lse=1e-5, grad_rel=1e-4, grad_abs=1e-6, norm=1e-5),
    torch.bfloat16: dict(loss=1e-2, lse=1e-3, grad_rel=2e-2, grad_abs=1e-2, norm=1e-2),
}


def bf16_round(a: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).float().numpy()


def prepare(E_ref: np.ndarray, C_ref: np.ndarray, dtype):
    """Reference layout (E n x d, C d x v) -> device X [n,d], E [v,d] in `dtype`,
    plus the host copies the oracle must see (bf16-rounded for bf16)."""
    if dtype == torch.bfloat16:
        E_ref, C_ref = bf16_round(E_ref), bf16_round(C_ref)
    X = torch.from_numpy(np.ascontiguousarray(E_ref)).to("cuda").to(dtype)
    E = torch.from_numpy(np.ascontiguousarray(C_ref.T)).to("cuda").to(dtype)
    return X, E, E_ref, C_ref


def instance(seed, n, d, v, dtype, half_width=1.0):
    rng = ob.Rng(seed)
    inst = ob.make_instance(rng, n, d, v, half_width)
    X, E, Eh, Ch = prepare(inst.E, inst.C, dtype)
    return X, E, torch.from_numpy(inst.targets).to("cuda"), Eh, Ch, inst.targets


def check_grad(got: torch.Tensor, want: np.ndarray, dtype, what=""):
    t = TOL[dtype]
    g = got.double().cpu().numpy()
    if dtype == torch.float64:
        err = ob.rel_err(g, want)
        assert err.max() < t["grad_rel"], (what, err.max())
        return
    mx = np.abs(want).max() if want.size else 0.0
    bound = t["grad_rel"] * np.abs(want) + t["grad_abs"] * mx
    diff = np.abs(g - want)
    assert (diff <= bound + 1e-30).all(), (what, float((diff - bound).max()))
    nrm = np.linalg.norm(g - want) / max(np.linalg.norm(want), 1e-300)
    assert nrm <= t["norm"], (what, nrm)
