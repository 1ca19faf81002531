"""GPU parity of vtrace_head_loss_and_grad (NEXT #3 second half: the output layer with the
whole V-trace path as its epilogue and the head's backward; Section 4) against
oracle/output_layer_oracle.loss_and_grad_from_hidden, through the C ABI.

Inputs: h on a 2^-6 grid and W, b on a 2^-3 grid, so z^pi = h W + b is exact in the tensor
cores' fp32 accumulation and equals the oracle's fp32-rounded head outputs; the path's
outputs then follow the library-wide tolerance (1e-6 abs + 1e-5 rel per dZ element).
Bounds derived from the arithmetic:
  grad_hidden  bf16 output: 2^-8 |ref| (round-to-nearest) + sum_j |W_hj| (1e-6 + 1e-5 |dZ_j|)
               (the dZ tolerance carried through W) + 2^-15 sum_j |dZ_j W_hj| (hi + lo and
               the fp32 accumulation)
  grad_w_t     fp32: 1e-4 sum_rows |h| |dZ| (dZ tolerance + fp32 accumulation over a CTA's
               rows, random-walk bound with margin) + 1e-6
  grad_bias    1e-5 sum_rows |dZ| + 1e-6;  partials: 1e-6 relative (fp64 accumulators)."""
import numpy as np
import pytest
import torch

import oracle
import paper_1802_01561_b200 as pkg
from oracle import output_layer_oracle as ol

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _case(T, B, H, A, seed, bias=True, p_done=0.05, lag=0.3):
    rng = np.random.default_rng(seed)
    h = rng.integers(-48, 49, size=(T, B, H)) / 64.0
    W = rng.integers(-8, 9, size=(H, A + 1)) / 8.0 * (8.0 / np.sqrt(H))  # z ~ N(0, ~2)
    W = np.round(W * 8.0) / 8.0
    b = rng.integers(-8, 9, size=A + 1) / 8.0 if bias else np.zeros(A + 1)
    z = (h.reshape(T * B, H) @ W + b)[:, :A].reshape(T, B, A)
    mu = (z + rng.normal(scale=lag, size=z.shape)).astype(np.float32)
    g = rng.gumbel(size=mu.shape)
    actions = np.argmax(mu + g, axis=-1).astype(np.int32)
    done = rng.random((T, B)) < p_done
    inp = dict(T=T, B=B, A=A, dtype=oracle.DTYPE_F32,
               target_logits=np.zeros((T, B, A), np.float32), behaviour_logits=mu,
               actions=actions, rewards=rng.normal(size=(T, B)).astype(np.float32),
               values=np.zeros((T, B), np.float32),
               bootstrap_value=rng.normal(size=B).astype(np.float32),
               discounts=np.where(done, 0.0, 0.99).astype(np.float32))
    return inp, h, W, b


def _run(inp, h, W, b, bias=True, **kw):
    t = lambda x, dt=torch.float32: torch.tensor(x, dtype=dt, device=DEV)  # noqa: E731
    ht = t(h).to(torch.bfloat16)
    wt = t(W.T.copy()).to(torch.bfloat16)
    out = pkg.head_loss_and_grad(ht, wt, t(b) if bias else None, t(inp["behaviour_logits"]),
                                 t(inp["actions"], torch.int32), t(inp["discounts"]),
                                 t(inp["rewards"]), t(inp["bootstrap_value"]), **kw)
    torch.cuda.synchronize()
    return {k: v.float().cpu().numpy().astype(np.float64) if v.dtype != torch.float64
            else v.cpu().numpy() for k, v in out.items()}


def _check(inp, h, W, got, ref):
    T, B, H = h.shape
    A = W.shape[1] - 1
    dZ = np.concatenate([ref["grad_target_logits"].reshape(T * B, A),
                         ref["grad_values"].reshape(T * B, 1)], axis=1)
    # grad_hidden
    tol_dz = 1e-6 + 1e-5 * np.abs(dZ)
    bound = (2.0 ** -8 * np.abs(ref["grad_hidden"]).reshape(T * B, H)
             + tol_dz @ np.abs(W).T + 2.0 ** -15 * (np.abs(dZ) @ np.abs(W).T) + 1e-30)
    err = np.abs(got["grad_hidden"].reshape(T * B, H) - ref["grad_hidden"].reshape(T * B, H))
    assert (err <= bound).all(), ("grad_hidden", float((err / bound).max()), int((err > bound).sum()))
    # grad_w_t = grad_W^T
    S = np.abs(h.reshape(T * B, H)).T @ np.abs(dZ)
    errw = np.abs(got["grad_w_t"].T - ref["grad_W"])
    bw = 1e-4 * S + 1e-6
    assert (errw <= bw).all(), ("grad_w_t", float((errw / bw).max()))
    errb = np.abs(got["grad_bias"] - ref["grad_b"])
    bb = 1e-5 * np.abs(dZ).sum(axis=0) + 1e-6
    assert (errb <= bb).all(), ("grad_bias", float((errb / bb).max()))
    np.testing.assert_allclose(got["partials"][:7], ref["partials"][:7], rtol=1e-6, atol=1e-9)
    assert got["partials"][7] == ref["partials"][7]  # the clip count


@pytest.mark.parametrize("T,B,H,A", [(20, 36, 256, 18),    # ragged in T (16 + 4) and B (8k + 4)
                                     (40, 512, 256, 18),
                                     (33, 64, 128, 9),
                                     (16, 8, 128, 3),
                                     (100, 32, 256, 9),    # dmlab-shaped
                                     (20, 32, 256, 18),    # atari-shaped
                                     (7, 12, 256, 6), (48, 200, 128, 4)])
def test_fused_head_matches_oracle(T, B, H, A):
    inp, h, W, b = _case(T, B, H, A, seed=T * 1000 + B + H + A)
    ref = ol.loss_and_grad_from_hidden(inp, h, W, b, baseline_cost=0.5, entropy_cost=0.01)
    got = _run(inp, h, W, b)
    _check(inp, h, W, got, ref)


def test_fused_head_no_bias_terminals_and_truncation():
    """No bias; many episode ends; c_bar < rho_bar = pg_rho_bar; entropy and baseline
    weights off their defaults; a wide batch (several blocks per CTA)."""
    T, B, H, A = 50, 2400, 256, 18
    inp, h, W, b = _case(T, B, H, A, seed=5, bias=False, p_done=0.3, lag=0.8)
    kw = dict(rho_bar=2.0, c_bar=0.9, baseline_cost=0.25, entropy_cost=0.05)
    ref = ol.loss_and_grad_from_hidden(inp, h, W, b, **kw)
    got = _run(inp, h, W, b, bias=False, **kw)
    _check(inp, h, W, got, ref)


def test_fused_head_deterministic():
    T, B, H, A = 30, 160, 256, 18
    inp, h, W, b = _case(T, B, H, A, seed=9)
    g1 = _run(inp, h, W, b)
    g2 = _run(inp, h, W, b)
    for k in g1:
        np.testing.assert_array_equal(g1[k], g2[k])


def test_fused_head_argument_errors():
    lib = pkg.load_library()
    with pytest.raises(ValueError):
        pkg.head_loss_and_grad(torch.zeros(4, 6, 256, dtype=torch.bfloat16, device=DEV),
                               torch.zeros(19, 256, dtype=torch.bfloat16, device=DEV), None,
                               torch.zeros(4, 6, 18, device=DEV),
                               torch.zeros(4, 6, dtype=torch.int32, device=DEV),
                               torch.zeros(4, 6, device=DEV), torch.zeros(4, 6, device=DEV),
                               torch.zeros(5, device=DEV))  # bootstrap of the wrong size
    assert lib.vtrace_head_workspace_bytes(10, 8, 256, 18) > 0
    assert lib.vtrace_head_workspace_bytes(10, 8, 256, 40) == 0
