"""Parity tolerances shared by the GPU tests (readings R4 and R21).

Forward (north star, BASELINE.json): max |O - O_ref| <= 2e-2 and mean <= 2e-3
on unit-variance bf16 inputs.

Gradients (R21; eq:ba, PAPER.md:157-165 -- the paper states no tolerance):
the north-star bound scaled by each tensor's own magnitude, plus the
gradient's final bf16 rounding, which the fp64 oracle does not have.  bf16
keeps 8 significant bits, so the unit roundoff is u = 2^-8: one RNE rounding
moves x by at most ulp(x)/2 <= 2^-8 |x| (worst case).  Over many elements
the discarded low bits are uniformly distributed, so the EXPECTED rounding
error is ulp(x)/4 = 2^-9 * 2^floor(log2|x|) <= 2^-9 |x|; the mean term is
therefore 2^-9 * mean|g_ref|.  That expectation is checked on every tensor
against the oracle's own values (mean |rne_bf16(g_ref) - g_ref| <= 2^-9 *
mean|g_ref|, exact arithmetic on the fp64 reference), so the term is pinned
by measurement, not assumed.
"""
import numpy as np
import torch

MAX_TOL = 2e-2
MEAN_TOL = 2e-3
BF16_U = 2.0 ** -8          # unit roundoff (worst case per element, relative)
BF16_MEAN_RNE = 2.0 ** -9   # expected relative RNE error (ulp/4 <= 2^-9 |x|)


def bf16_rne_mean_error(ref: np.ndarray) -> float:
    """Exact mean |rne_bf16(x) - x| of an fp64 array (torch rounds fp64 -> bf16 to nearest even)."""
    r = torch.from_numpy(np.ascontiguousarray(ref, dtype=np.float64))
    return float((r.to(torch.bfloat16).double() - r).abs().mean())


def grad_bounds(ref: np.ndarray):
    """(max bound, mean bound) of reading R21 for one gradient tensor; also
    checks the rounding model on the reference itself."""
    a = np.abs(ref)
    rne = bf16_rne_mean_error(ref)
    assert rne <= BF16_MEAN_RNE * a.mean() + 1e-300, (rne, a.mean())
    assert np.abs(ref - torch.from_numpy(ref).to(torch.bfloat16).double().numpy()).max() <= BF16_U * a.max()
    return MAX_TOL * max(1.0, a.max()), MEAN_TOL * max(1.0, a.mean()) + BF16_MEAN_RNE * a.mean()


def check_grad(name: str, got, ref: np.ndarray) -> None:
    g = got.float().cpu().numpy().astype(np.float64) if isinstance(got, torch.Tensor) else got
    assert np.isfinite(g).all(), f"{name}: non-finite"
    err = np.abs(g - ref)
    mx, mn = grad_bounds(ref)
    assert err.max() <= mx, f"{name}: max err {err.max():.3e} > {mx:.3e}"
    assert err.mean() <= mn, f"{name}: mean err {err.mean():.3e} > {mn:.3e}"
