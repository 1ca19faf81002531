"""Pins of the learner-update oracle (oracle/rmsprop_oracle.py)
against facts that do not come from the oracle itself: closed forms of the
RMSProp recurrence, exact clip scales, invariants, and the special case that
reduces to a library optimiser (torch.optim.RMSprop with eps = 0 is the same
update; torch's clip_grad_norm_ is the same clip up to its 1e-6 guard).
CPU only."""
import numpy as np
import pytest
import torch

from oracle import rmsprop_oracle as ro


def test_global_norm_pythagorean_triple():
    g = np.zeros(1000)
    g[7], g[911] = 3.0, 4.0
    assert ro.global_norm(g) == 5.0


def test_clip_scale_is_exact_power_of_two():
    # ||(48, 64)|| = 80 = 2 x 40: the clip halves every component exactly
    g, norm = ro.clip_by_global_norm(np.array([48.0, -64.0, 0.0]), 40.0)
    assert norm == 80.0
    assert g.tolist() == [24.0, -32.0, 0.0]


def test_clip_leaves_small_gradients_alone():
    g0 = np.array([24.0, 32.0])  # norm exactly 40: not above the threshold
    g, norm = ro.clip_by_global_norm(g0, 40.0)
    assert norm == 40.0 and g.tolist() == g0.tolist()
    g, _ = ro.clip_by_global_norm(g0, 0.0)  # disabled
    assert g.tolist() == g0.tolist()


def test_mean_square_closed_form_under_constant_gradient():
    # ms_k = decay ms_{k-1} + (1 - decay) g^2  =>  ms_k = g^2 + decay^k (ms_0 - g^2)
    rng = np.random.default_rng(3)
    g = rng.normal(size=64)
    ms0 = rng.uniform(0.0, 2.0, size=64)
    theta, ms = rng.normal(size=64), ms0.copy()
    decay, k = 0.99, 25
    for _ in range(k):
        theta, ms, _ = ro.rmsprop_step(theta, ms, g, 6e-4, decay, 0.01, 0.0)
    np.testing.assert_allclose(ms, g * g + decay ** k * (ms0 - g * g), rtol=1e-13, atol=1e-15)


def test_fixed_point_mean_square_gives_constant_steps():
    # ms_0 = g^2 is the fixed point: every step moves theta by lr g / sqrt(g^2 + eps)
    g = np.array([0.5, -2.0, 1e-3])
    theta0 = np.array([1.0, 2.0, 3.0])
    theta, ms = theta0.copy(), g * g
    lr, eps, k = 1e-3, 0.01, 10
    for _ in range(k):
        theta, ms, _ = ro.rmsprop_step(theta, ms, g, lr, 0.9, eps, 0.0)
    np.testing.assert_allclose(ms, g * g, rtol=1e-15)
    np.testing.assert_allclose(theta, theta0 - k * lr * g / np.sqrt(g * g + eps), rtol=1e-14)


def test_zero_gradient_moves_nothing_and_decays_the_mean_square():
    theta0, ms0 = np.array([0.3, -1.0]), np.array([1.0, 0.25])
    theta, ms, norm = ro.rmsprop_step(theta0, ms0, np.zeros(2), 1e-2, 0.99, 0.1, 40.0)
    assert norm == 0.0
    assert theta.tolist() == theta0.tolist()
    np.testing.assert_allclose(ms, 0.99 * ms0, rtol=1e-15)


def test_clipped_update_is_invariant_to_gradient_scale():
    rng = np.random.default_rng(5)
    g = rng.normal(size=300) * 10.0  # norm ~ 170 > 40
    theta, ms = rng.normal(size=300), rng.uniform(0.1, 1.0, size=300)
    a = ro.rmsprop_step(theta, ms, g, 6e-4, 0.99, 0.01, 40.0)
    b = ro.rmsprop_step(theta, ms, 3.0 * g, 6e-4, 0.99, 0.01, 40.0)
    np.testing.assert_allclose(a[0], b[0], rtol=1e-14)
    np.testing.assert_allclose(a[1], b[1], rtol=1e-13)
    assert b[2] == pytest.approx(3.0 * a[2], rel=1e-15)


def test_matches_torch_rmsprop_when_epsilon_is_zero():
    # torch: ms <- alpha ms + (1-alpha) g^2; theta <- theta - lr g / (sqrt(ms) + eps);
    # with eps = 0 this is the TF form with epsilon = 0 (reading r9)
    rng = np.random.default_rng(11)
    theta0 = rng.normal(size=200)
    grads = [rng.normal(size=200) for _ in range(5)]
    p = torch.nn.Parameter(torch.tensor(theta0, dtype=torch.float64))
    opt = torch.optim.RMSprop([p], lr=5e-3, alpha=0.95, eps=0.0, momentum=0.0, centered=False)
    theta, ms = theta0.copy(), np.zeros(200)  # torch starts its square average at 0
    for g in grads:
        p.grad = torch.tensor(g, dtype=torch.float64)
        opt.step()
        theta, ms, _ = ro.rmsprop_step(theta, ms, g, 5e-3, 0.95, 0.0, 0.0)
    np.testing.assert_allclose(p.detach().numpy(), theta, rtol=1e-13, atol=1e-15)


def test_clip_matches_torch_clip_grad_norm():
    rng = np.random.default_rng(2)
    parts = [rng.normal(size=n) * 5.0 for n in (100, 37, 1000)]
    ps = [torch.nn.Parameter(torch.zeros(len(x), dtype=torch.float64)) for x in parts]
    for p, x in zip(ps, parts):
        p.grad = torch.tensor(x, dtype=torch.float64)
    total = torch.nn.utils.clip_grad_norm_(ps, 40.0)
    g, norm = ro.clip_by_global_norm(np.concatenate(parts), 40.0)
    assert norm == pytest.approx(float(total), rel=1e-14)
    got = np.concatenate([p.grad.numpy() for p in ps])
    np.testing.assert_allclose(g, got, rtol=1e-6)  # torch divides by (norm + 1e-6)


def test_learner_gradients_add_up_to_the_batch_gradient():
    # loss summed over the batch: L = sum_b w . x_b, dL/dw = sum_b x_b; each
    # learner holds a block of the batch, and the blocks' gradients sum to the whole
    rng = np.random.default_rng(9)
    x = rng.normal(size=(24, 7))
    full = x.sum(axis=0)
    shards = [x[i:j].sum(axis=0) for i, j in ((0, 5), (5, 16), (16, 24))]
    np.testing.assert_allclose(ro.sum_learner_grads(shards), full, rtol=1e-14)
