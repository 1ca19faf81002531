"""Pins for the output-layer oracle (oracle/output_layer_oracle.py).
Each test ties it to something other than itself: the bare path it must reduce to,
central differences of the paper's loss with the stop-gradient
quantities frozen (reading c10), and the summed loss.  P:n = PAPER.md line n."""
import numpy as np
import pytest

import oracle
from oracle import output_layer_oracle as ol


def _rest(T, B, A, seed, p_done=0.25):
    """Behaviour logits, actions, rewards, discounts, bootstrap (fp32 layout)."""
    rng = np.random.default_rng(seed)
    done = rng.random((T, B)) < p_done
    return dict(T=T, B=B, A=A, dtype=oracle.DTYPE_F32,
                target_logits=np.zeros((T, B, A), np.float32),
                behaviour_logits=rng.normal(size=(T, B, A)).astype(np.float32),
                actions=rng.integers(0, A, size=(T, B)).astype(np.int32),
                rewards=rng.normal(size=(T, B)).astype(np.float32),
                values=np.zeros((T, B), np.float32),
                bootstrap_value=rng.normal(size=B).astype(np.float32),
                discounts=np.where(done, 0.0, 0.99).astype(np.float32))


def _dyadic_head(T, B, H, A, seed):
    """h on a 2^-6 grid, W and b on a 2^-3 grid: h @ W + b and every +-2^-10
    perturbation below are exact in fp32, so the fp32 rounding of the head's
    outputs does not enter the differences."""
    rng = np.random.default_rng(seed)
    h = rng.integers(-48, 49, size=(T, B, H)) / 64.0
    W = rng.integers(-8, 9, size=(H, A + 1)) / 8.0
    b = rng.integers(-8, 9, size=A + 1) / 8.0
    return h, W, b


def test_identity_head_reduces_to_the_bare_path():
    """W = I, b = 0, h = [z | V]: the head passes the path's inputs through, so dh is
    [dL/dz | dL/dV] of the bare path and dW = h^T dZ."""
    T, B, A = 6, 5, 4
    inp = _rest(T, B, A, 1)
    rng = np.random.default_rng(2)
    z = rng.normal(size=(T, B, A)).astype(np.float32)
    V = rng.normal(size=(T, B)).astype(np.float32)
    h = np.concatenate([z, V[..., None]], axis=2).astype(np.float64)
    got = ol.loss_and_grad_from_hidden(inp, h, np.eye(A + 1), np.zeros(A + 1), entropy_cost=0.05)
    bare = dict(inp, target_logits=z, values=V)
    ref = oracle.loss_and_grad(bare, entropy_cost=0.05)
    np.testing.assert_array_equal(got["grad_hidden"][..., :A], ref["grad_target_logits"])
    np.testing.assert_array_equal(got["grad_hidden"][..., A], ref["grad_values"])
    np.testing.assert_array_equal(got["vs"], ref["vs"])
    np.testing.assert_array_equal(got["partials"], ref["partials"])


def _frozen_loss(inp, h, W, b, pg_adv0, vs0, c_v, c_e):
    """P:254-261 with v_s and pg_adv held at the base point (reading c10):
    -sum pg_adv0 log pi(a) + c_v/2 sum (v0 - V)^2 - c_e sum H."""
    z, V = ol.output_layer(h, W, b)
    run = dict(inp, target_logits=z.astype(np.float32), values=V.astype(np.float32))
    tlp = oracle.from_logits(run)["target_action_log_probs"]
    ent = oracle.loss_and_grad(run, baseline_cost=c_v, entropy_cost=c_e)["partials"][2]
    return -(pg_adv0 * tlp).sum() + 0.5 * c_v * ((vs0 - V) ** 2).sum() - c_e * ent


@pytest.mark.parametrize("seed", range(3))
def test_chain_rule_against_central_differences(seed):
    rng = np.random.default_rng(100 + seed)
    T, B, H, A = int(rng.integers(1, 5)), 2, 3, 4
    inp = _rest(T, B, A, 200 + seed)
    h, W, b = _dyadic_head(T, B, H, A, 300 + seed)
    c_v, c_e = 0.5, 0.3
    base = ol.loss_and_grad_from_hidden(inp, h, W, b, baseline_cost=c_v, entropy_cost=c_e)
    pg0, v0 = base["pg_advantages"], base["vs"]
    e = 2.0 ** -10

    def fd(arr, idx, which):
        p, m = arr.copy(), arr.copy()
        p[idx] += e
        m[idx] -= e
        args_p = {"h": h, "W": W, "b": b, which: p}
        args_m = {"h": h, "W": W, "b": b, which: m}
        lp = _frozen_loss(inp, args_p["h"], args_p["W"], args_p["b"], pg0, v0, c_v, c_e)
        lm = _frozen_loss(inp, args_m["h"], args_m["W"], args_m["b"], pg0, v0, c_v, c_e)
        return (lp - lm) / (2 * e)

    for name, arr, grad in (("h", h, base["grad_hidden"]), ("W", W, base["grad_W"]),
                            ("b", b, base["grad_b"])):
        for idx in np.ndindex(arr.shape):
            d = fd(arr, idx, name)
            assert abs(d - grad[idx]) < 1e-5 * max(1.0, abs(grad[idx])), (name, idx, d, grad[idx])


def test_weight_gradient_sums_over_columns():
    """The loss is summed over the batch and V-trace is per column: the head's
    gradient on columns [0, B1) + [B1, B) equals that of the concatenated batch."""
    T, B1, B2, H, A = 5, 3, 4, 6, 5
    i1, i2 = _rest(T, B1, A, 7), _rest(T, B2, A, 8)
    rng = np.random.default_rng(9)
    W = rng.normal(size=(H, A + 1)) * 0.5
    b = rng.normal(size=A + 1) * 0.1
    h1, h2 = rng.normal(size=(T, B1, H)), rng.normal(size=(T, B2, H))
    cat = {k: (np.concatenate([i1[k], i2[k]], axis=1 if np.ndim(i1[k]) >= 2 else 0)
               if isinstance(i1[k], np.ndarray) else i1[k]) for k in i1}
    cat["B"] = B1 + B2
    g1 = ol.loss_and_grad_from_hidden(i1, h1, W, b)
    g2 = ol.loss_and_grad_from_hidden(i2, h2, W, b)
    g = ol.loss_and_grad_from_hidden(cat, np.concatenate([h1, h2], axis=1), W, b)
    np.testing.assert_allclose(g["grad_W"], g1["grad_W"] + g2["grad_W"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(g["grad_b"], g1["grad_b"] + g2["grad_b"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(g["grad_hidden"][:, :B1], g1["grad_hidden"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(g["partials"][:4], g1["partials"][:4] + g2["partials"][:4],
                               rtol=1e-12)
