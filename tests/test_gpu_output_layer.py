"""GPU parity of vtrace_output_layer (NEXT #3, reading r12) against
oracle/output_layer_oracle.py, through the C ABI.

Dyadic inputs (h on a 2^-6 grid, W and b on a 2^-3 grid) make every partial sum exact in
fp32, so those cases are compared bitwise; normal-distributed bf16 inputs are compared
within the fp32 accumulation bound K * 2^-24 * sum_k |h_k W_kj| (doubled)."""
import numpy as np
import pytest
import torch

import oracle
import paper_1802_01561_b200 as pkg
from oracle import output_layer_oracle as ol

pytestmark = pytest.mark.gpu


def _dyadic(M, H, A, seed):
    rng = np.random.default_rng(seed)
    h = rng.integers(-48, 49, size=(M, H)) / 64.0
    W = rng.integers(-8, 9, size=(H, A + 1)) / 8.0
    b = rng.integers(-8, 9, size=A + 1) / 8.0
    return h, W, b


def _run(h, W, b):
    dev = "cuda:0"
    ht = torch.tensor(h, dtype=torch.float32).to(torch.bfloat16).to(dev)
    wt = torch.tensor(W.T.copy(), dtype=torch.float32).to(torch.bfloat16).to(dev)
    bt = None if b is None else torch.tensor(b, dtype=torch.float32, device=dev)
    z, v = pkg.output_layer(ht, wt, bt)
    torch.cuda.synchronize()
    return z.cpu().numpy().astype(np.float64), v.cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("M,H,A", [(3200, 256, 9),      # dmlab T*B, A = 9
                                   (640, 256, 18),      # atari T*B
                                   (1000, 256, 18),     # ragged last tile
                                   (1, 64, 1), (129, 128, 31), (4097, 192, 5),
                                   (300, 64, 17)])
def test_dyadic_bitwise(M, H, A):
    h, W, b = _dyadic(M, H, A, M + H + A)
    z, v = _run(h, W, b)
    zr, vr = ol.output_layer(h.reshape(M, 1, H), W, b)
    np.testing.assert_array_equal(z, zr.reshape(M, A))
    np.testing.assert_array_equal(v, vr.reshape(M))


def test_no_bias_and_empty():
    h, W, _ = _dyadic(257, 128, 6, 3)
    z, v = _run(h, W, None)
    zr, vr = ol.output_layer(h.reshape(257, 1, 128), W, np.zeros(7))
    np.testing.assert_array_equal(z, zr.reshape(257, 6))
    np.testing.assert_array_equal(v, vr.reshape(257))
    dev = "cuda:0"
    e = torch.empty((0, 128), dtype=torch.bfloat16, device=dev)
    w = torch.zeros((7, 128), dtype=torch.bfloat16, device=dev)
    z0, v0 = pkg.output_layer(e, w)
    assert z0.shape == (0, 6) and v0.shape == (0,)


def test_large_config_sampled_rows():
    """The `large` config's T*B = 819,200 rows, H = 256, A = 18, normal bf16 inputs; 4096
    sampled rows (plus the first and last tile) against the fp64 oracle."""
    M, H, A = 100 * 8192, 256, 18
    g = torch.Generator(device="cuda:0").manual_seed(7)
    ht = torch.randn((M, H), generator=g, device="cuda:0").to(torch.bfloat16)
    wt = (torch.randn((A + 1, H), generator=g, device="cuda:0") * 0.1).to(torch.bfloat16)
    bt = torch.randn(A + 1, generator=g, device="cuda:0")
    z, v = pkg.output_layer(ht, wt, bt)
    torch.cuda.synchronize()
    rng = np.random.default_rng(1)
    rows = np.unique(np.concatenate([rng.integers(0, M, 4096), np.arange(128),
                                     np.arange(M - 128, M)]))
    h = ht[rows].float().cpu().numpy().astype(np.float64)
    W = wt.float().cpu().numpy().astype(np.float64).T
    b = bt.cpu().numpy().astype(np.float64)
    zr, vr = ol.output_layer(h.reshape(len(rows), 1, H), W, b)
    bound = 2 * H * 2.0 ** -24 * (np.abs(h) @ np.abs(W) + np.abs(b)) + 1e-30
    gz = z[rows].cpu().numpy().astype(np.float64)
    gv = v[rows].cpu().numpy().astype(np.float64)
    assert (np.abs(gz - zr.reshape(-1, A)) <= bound[:, :A]).all()
    assert (np.abs(gv - vr.reshape(-1)) <= bound[:, A]).all()


def test_head_then_path_matches_oracle_chain():
    """output_layer -> loss_and_grad (the product path) against
    oracle.loss_and_grad_from_hidden on a dmlab-shaped batch with fp32 logits."""
    T, B, H, A = 100, 32, 256, 9
    rng = np.random.default_rng(11)
    h, W, b = _dyadic(T * B, H, A, 12)
    h = h.reshape(T, B, H)
    done = rng.random((T, B)) < 0.05
    inp = dict(T=T, B=B, A=A, dtype=oracle.DTYPE_F32,
               target_logits=np.zeros((T, B, A), np.float32),
               behaviour_logits=rng.normal(size=(T, B, A)).astype(np.float32),
               actions=rng.integers(0, A, size=(T, B)).astype(np.int32),
               rewards=rng.normal(size=(T, B)).astype(np.float32),
               values=np.zeros((T, B), np.float32),
               bootstrap_value=rng.normal(size=B).astype(np.float32),
               discounts=np.where(done, 0.0, 0.99).astype(np.float32))
    ref = ol.loss_and_grad_from_hidden(inp, h, W, b, baseline_cost=0.5, entropy_cost=0.01)
    dev = "cuda:0"
    ht = torch.tensor(h, dtype=torch.float32).to(torch.bfloat16).to(dev)
    wt = torch.tensor(W.T.copy(), dtype=torch.float32).to(torch.bfloat16).to(dev)
    z, v = pkg.output_layer(ht, wt, torch.tensor(b, dtype=torch.float32, device=dev))
    t = lambda x, dt=torch.float32: torch.tensor(x, dtype=dt, device=dev)  # noqa: E731
    out = pkg.loss_and_grad(t(inp["behaviour_logits"]), z, t(inp["actions"], torch.int32),
                            t(inp["discounts"]), t(inp["rewards"]), v, t(inp["bootstrap_value"]),
                            baseline_cost=0.5, entropy_cost=0.01)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(z.cpu().numpy(), ref["target_logits"])
    np.testing.assert_array_equal(v.cpu().numpy(), ref["values"])
    for k, got in (("vs", out["vs"]), ("pg_advantages", out["pg_advantages"]),
                   ("grad_values", out["grad_values"]),
                   ("grad_target_logits", out["grad_target_logits"])):
        g = got.float().cpu().numpy().astype(np.float64)
        bad = np.abs(g - ref[k]) > 1e-6 + 1e-5 * np.abs(ref[k])
        assert not bad.any(), (k, int(bad.sum()))


def test_parameter_errors():
    dev = "cuda:0"
    lib = pkg.load_library()
    h = torch.zeros((128, 256), dtype=torch.bfloat16, device=dev)
    w = torch.zeros((10, 256), dtype=torch.bfloat16, device=dev)
    z = torch.zeros((128, 9), device=dev)
    v = torch.zeros(128, device=dev)
    p = lambda x: x.data_ptr()  # noqa: E731
    assert lib.vtrace_output_layer(128, 100, 9, p(h), p(w), None, p(z), p(v), None) == 2
    assert lib.vtrace_output_layer(128, 256, 31 + 1, p(h), p(w), None, p(z), p(v), None) == 2
    assert lib.vtrace_output_layer(128, 256, 9, None, p(w), None, p(z), p(v), None) == 1
    assert lib.vtrace_output_layer(128, 256, 9, p(h) + 2, p(w), None, p(z), p(v), None) == 5
    assert lib.vtrace_output_layer(128, 256, 9, p(h), p(w), None, p(z), p(v), None) == 0
