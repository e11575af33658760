"""The rounding model behind the gradient tolerance (reading R21),
checked on CPU: bf16 RNE moves x by at most u|x| with u = 2^-8, and by
2^-9 |x| or less on average over many values (expected error ulp/4)."""
import numpy as np
import torch

from tolerance import BF16_MEAN_RNE, BF16_U, bf16_rne_mean_error, grad_bounds


def test_bf16_unit_roundoff_worst_case():
    rng = np.random.default_rng(0)
    x = rng.standard_normal(200000) * np.exp(rng.uniform(-20, 20, 200000))
    r = torch.from_numpy(x).to(torch.bfloat16).double().numpy()
    rel = np.abs(r - x) / np.abs(x)
    assert rel.max() <= BF16_U
    assert rel.max() > 0.9 * BF16_U  # the bound is attained (not a loose constant)


def test_bf16_mean_rounding_error_model():
    rng = np.random.default_rng(1)
    for scale in (1e-3, 1.0, 37.0):
        x = rng.standard_normal(100000) * scale
        m = bf16_rne_mean_error(x)
        assert m <= BF16_MEAN_RNE * np.abs(x).mean()
        # expected ulp/4 with the mantissa spread over the binade: about 2^-9 / 1.44
        assert m >= 0.5 * BF16_MEAN_RNE * np.abs(x).mean()


def test_grad_bounds_exact_values():
    ref = np.array([0.0, 1.0, -2.0, 0.5])  # exactly representable: no rounding term beyond the model
    mx, mn = grad_bounds(ref)
    assert mx == 2e-2 * 2.0
    assert abs(mn - (2e-3 * 1.0 + 2.0 ** -9 * 0.875)) < 1e-15
