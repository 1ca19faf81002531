"""GPU parity of the learner update (vtrace_rmsprop_step)
against the fp64 oracle (oracle/rmsprop_oracle.py), through the C ABI.  Sizes
cover the register-resident kernel (V = 1, 2, 4, 6 float4 a thread; its capacity
148 x 512 x 6 x 4 = 1,818,624 parameters exactly), the two-pass streaming kernel
beyond it (2,000,003), ragged n % 4 tails and unaligned views (scalar kernel).

Tolerance (learner update): the kernel computes in fp32 (1/sqrt by the
MUFU rsqrt, relative error < 2^-22), so the new mean square is within a few fp32
ulps (rtol 1e-6) and the new parameter within 1e-6 of the step size plus 2 ulps of
the parameter.  The
hyperparameters cross the ABI as fp32; the oracle gets those same fp32 values.
The clip decision and the norm are fp64 on both sides (norm rtol 1e-12).
"""
import ctypes

import numpy as np
import pytest
import torch

import paper_1802_01561_b200 as pkg
from oracle import rmsprop_oracle as ro
from paper_1802_01561_b200 import workload as wl

pytestmark = pytest.mark.gpu

LR, DECAY, EPS, CLIP = 6e-4, 0.99, 0.01, 40.0  # P:950-953 (decay: reading r9)


def _f32(x):
    return float(np.float32(x))


def _check(theta_gpu, ms_gpu, theta0, theta_ref, ms_ref):
    step = np.abs(theta_ref - np.asarray(theta0, np.float64))
    err = np.abs(theta_gpu.astype(np.float64) - theta_ref)
    bound = 1e-6 * step + 2.4e-7 * np.abs(theta_ref) + 1e-30
    worst = float(np.max(err / bound)) if err.size else 0.0
    assert worst <= 1.0, f"theta off by {worst:.3f} x tolerance"
    np.testing.assert_allclose(ms_gpu.astype(np.float64), ms_ref, rtol=1e-6, atol=1e-30)


def _run(inp, lr=LR, decay=DECAY, eps=EPS, clip=CLIP, offset=0, steps=1, ws=None):
    dev = "cuda"
    n = inp["n"]

    def put(x):  # `offset` elements in: a 4-byte-aligned, not 16-byte-aligned view
        buf = torch.zeros(n + offset, dtype=torch.float32, device=dev)
        buf[offset:] = torch.from_numpy(np.ascontiguousarray(x))
        return buf[offset:]

    theta, ms = put(inp["params"]), put(inp["mean_square"])
    norm = torch.zeros(1, dtype=torch.float64, device=dev)
    ws = ws if ws is not None else pkg.RmspropWorkspace(n, dev)
    norms = []
    for k in range(steps):
        g = put(inp["grads"][k % len(inp["grads"])])
        pkg.rmsprop_step(theta, ms, g, lr, decay, eps, clip, global_norm_out=norm, workspace=ws)
        norms.append(float(norm.item()))
    torch.cuda.synchronize()
    return theta.cpu().numpy(), ms.cpu().numpy(), norms


def _oracle(inp, lr=LR, decay=DECAY, eps=EPS, clip=CLIP, steps=1):
    theta, ms = inp["params"].astype(np.float64), inp["mean_square"].astype(np.float64)
    norms = []
    for k in range(steps):
        theta, ms, nrm = ro.rmsprop_step(theta, ms, inp["grads"][k % len(inp["grads"])],
                                         _f32(lr), _f32(decay), _f32(eps), _f32(clip))
        norms.append(nrm)
    return theta, ms, norms


@pytest.mark.parametrize("n", [1, 3, 4, 7, 1000, 4099, 262147, 1_600_000, 1_818_624, 2_000_003])
@pytest.mark.parametrize("norm", [80.0, 10.0])
def test_rmsprop_matches_oracle(n, norm):
    inp = wl.update_inputs(n, seed=n % 97, norm=norm)
    th, ms, nr = _run(inp)
    th_ref, ms_ref, nr_ref = _oracle(inp)
    _check(th, ms, inp["params"], th_ref, ms_ref)
    assert nr[0] == pytest.approx(nr_ref[0], rel=1e-12)
    if n >= 1000:  # (a handful of draws need not reach the requested norm)
        assert (nr_ref[0] > CLIP) == (norm > CLIP)


@pytest.mark.parametrize("offset", [1, 2, 3])
def test_rmsprop_unaligned_views_take_the_scalar_path(offset):
    inp = wl.update_inputs(5003, seed=offset, norm=80.0)
    th, ms, nr = _run(inp, offset=offset)
    th_ref, ms_ref, nr_ref = _oracle(inp)
    _check(th, ms, inp["params"], th_ref, ms_ref)
    assert nr[0] == pytest.approx(nr_ref[0], rel=1e-12)


def test_rmsprop_successive_steps_share_a_workspace():
    # the workspace's epoch tags separate the calls' partial-sum records
    inp = wl.update_inputs(300_001, seed=2, norm=60.0, learners=3)  # 3 different gradients
    th, ms, nr = _run(inp, steps=5)
    th_ref, ms_ref, nr_ref = _oracle(inp, steps=5)
    step = np.abs(th_ref - inp["params"])
    err = np.abs(th.astype(np.float64) - th_ref)
    assert np.max(err / (5e-6 * step + 1e-6 * np.abs(th_ref) + 1e-30)) <= 1.0
    np.testing.assert_allclose(ms, ms_ref, rtol=5e-6)
    np.testing.assert_allclose(nr, nr_ref, rtol=1e-12)


def test_rmsprop_clip_disabled_and_lr_decay_extremes():
    inp = wl.update_inputs(70_000, seed=8, norm=500.0)
    for kw in ({"clip": 0.0}, {"decay": 0.0}, {"decay": 0.999, "eps": 1e-7}, {"eps": 0.1}):
        th, ms, _ = _run(inp, **kw)
        th_ref, ms_ref, _ = _oracle(inp, **kw)
        _check(th, ms, inp["params"], th_ref, ms_ref)


def test_rmsprop_zero_gradient_and_empty():
    inp = wl.update_inputs(4096, seed=1)
    inp["grads"] = [np.zeros(4096, np.float32)]
    th, ms, nr = _run(inp)
    assert nr[0] == 0.0
    assert np.array_equal(th, inp["params"])
    np.testing.assert_allclose(ms, _f32(DECAY) * inp["mean_square"].astype(np.float64), rtol=1e-6)
    empty = torch.zeros(0, dtype=torch.float32, device="cuda")
    norm = torch.full((1,), 7.0, dtype=torch.float64, device="cuda")
    pkg.rmsprop_step(empty, empty.clone(), empty.clone(), LR, DECAY, EPS, CLIP,
                     global_norm_out=norm)
    assert float(norm.item()) == 0.0


def test_rmsprop_is_deterministic():
    inp = wl.update_inputs(1_200_000, seed=6, norm=45.0)
    a = _run(inp)
    b = _run(inp)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]


def test_rmsprop_in_a_cuda_graph():
    inp = wl.update_inputs(400_003, seed=3, norm=90.0, learners=2)
    dev = "cuda"
    theta = torch.from_numpy(inp["params"]).to(dev)
    ms = torch.from_numpy(inp["mean_square"]).to(dev)
    g = torch.from_numpy(inp["grads"][0]).to(dev)
    ws = pkg.RmspropWorkspace(inp["n"], dev)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            pkg.rmsprop_step(theta, ms, g, LR, DECAY, EPS, CLIP, workspace=ws)
    torch.cuda.synchronize()
    # capture does not run the kernel: reset, then replay twice with two gradients
    theta.copy_(torch.from_numpy(inp["params"]))
    ms.copy_(torch.from_numpy(inp["mean_square"]))
    for k in range(2):
        g.copy_(torch.from_numpy(inp["grads"][k]))
        graph.replay()
    torch.cuda.synchronize()
    th_ref, ms_ref, _ = _oracle(inp, steps=2)
    step = np.abs(th_ref - inp["params"])
    err = np.abs(theta.cpu().numpy().astype(np.float64) - th_ref)
    assert np.max(err / (3e-6 * step + 1e-6 * np.abs(th_ref) + 1e-30)) <= 1.0
    np.testing.assert_allclose(ms.cpu().numpy(), ms_ref, rtol=3e-6)


def test_rmsprop_errors_raise():
    t = torch.zeros(8, dtype=torch.float32, device="cuda")
    with pytest.raises(pkg.VtraceError):
        pkg.rmsprop_step(t, t.clone(), t.clone(), 0.0, DECAY, EPS, CLIP)
    with pytest.raises(ValueError):
        pkg.rmsprop_step(t, t.clone(), torch.zeros(9, device="cuda"), LR, DECAY, EPS, CLIP)


# ---- several learners' gradients summed in the kernel (vtrace_rmsprop_step_multi) ----

@pytest.mark.parametrize("n,learners", [(4099, 2), (262147, 3), (1_600_000, 2), (70_001, 8),
                                        (2_000_003, 2)])
def test_rmsprop_multi_matches_oracle_on_the_sum(n, learners):
    inp = wl.update_inputs(n, seed=n % 31, norm=80.0, learners=learners)
    dev = "cuda"
    theta = torch.from_numpy(inp["params"]).to(dev)
    ms = torch.from_numpy(inp["mean_square"]).to(dev)
    gs = [torch.from_numpy(g).to(dev) for g in inp["grads"]]
    norm = torch.zeros(1, dtype=torch.float64, device=dev)
    pkg.rmsprop_step(theta, ms, gs, LR, DECAY, EPS, CLIP, global_norm_out=norm)
    torch.cuda.synchronize()
    total = ro.sum_learner_grads(inp["grads"])  # (reading r11)
    th_ref, ms_ref, nr_ref = ro.rmsprop_step(inp["params"], inp["mean_square"], total,
                                             _f32(LR), _f32(DECAY), _f32(EPS), _f32(CLIP))
    _check(theta.cpu().numpy(), ms.cpu().numpy(), inp["params"], th_ref, ms_ref)
    assert float(norm.item()) == pytest.approx(nr_ref, rel=1e-6)  # (fp32 sum of the buffers)


def test_rmsprop_multi_sums_in_index_order_bitwise():
    # the kernel adds the buffers in fp32 in index order: the same bits as one buffer
    # holding (g0 + g1) + g2 added by torch (IEEE fp32, elementwise)
    inp = wl.update_inputs(300_001, seed=12, norm=70.0, learners=3)
    dev = "cuda"
    gs = [torch.from_numpy(g).to(dev) for g in inp["grads"]]
    pre = (gs[0] + gs[1]) + gs[2]
    out = []
    for grads in (gs, pre, [pre]):
        theta = torch.from_numpy(inp["params"]).to(dev)
        ms = torch.from_numpy(inp["mean_square"]).to(dev)
        norm = torch.zeros(1, dtype=torch.float64, device=dev)
        pkg.rmsprop_step(theta, ms, grads, LR, DECAY, EPS, CLIP, global_norm_out=norm)
        torch.cuda.synchronize()
        out.append((theta.cpu().numpy(), ms.cpu().numpy(), float(norm.item())))
    for o in out[1:]:
        assert np.array_equal(out[0][0], o[0]) and np.array_equal(out[0][1], o[1])
        assert out[0][2] == o[2]


def test_rmsprop_multi_accepts_raw_device_pointers():
    inp = wl.update_inputs(10_000, seed=13, norm=90.0, learners=2)
    dev = "cuda"
    gs = [torch.from_numpy(g).to(dev) for g in inp["grads"]]
    res = []
    for grads in (gs, [g.data_ptr() for g in gs]):
        theta = torch.from_numpy(inp["params"]).to(dev)
        ms = torch.from_numpy(inp["mean_square"]).to(dev)
        pkg.rmsprop_step(theta, ms, grads, LR, DECAY, EPS, CLIP)
        torch.cuda.synchronize()
        res.append(theta.cpu().numpy())
    assert np.array_equal(res[0], res[1])
    with pytest.raises(ValueError):
        pkg.rmsprop_step(theta, ms, gs * 5, LR, DECAY, EPS, CLIP)  # 10 > 8 buffers


def test_rmsprop_learners_sync_path():
    """vtrace_rmsprop_step_learners on one GPU: learner 0 is this call, learner 1 a
    peer whose flags already read "ready and done" for every epoch (a second
    cooperative grid cannot share the GPU).  Same result as the multi form; the
    call publishes ready = done = epoch + 1 in its own flags, once per call."""
    inp = wl.update_inputs(400_003, seed=21, norm=75.0, learners=2)
    dev = "cuda"
    gs = [torch.from_numpy(g).to(dev) for g in inp["grads"]]
    flags = torch.zeros(2, 2, dtype=torch.int32, device=dev)
    flags[1] = 1 << 30  # the simulated peer: ahead of every epoch used here
    res = []
    for sync in (False, True):
        theta = torch.from_numpy(inp["params"]).to(dev)
        ms = torch.from_numpy(inp["mean_square"]).to(dev)
        ws = pkg.RmspropWorkspace(inp["n"], dev)
        for _ in range(3):
            kw = dict(learner_flags=[flags[0].data_ptr(), flags[1].data_ptr()],
                      self_index=0) if sync else {}
            pkg.rmsprop_step(theta, ms, gs, LR, DECAY, EPS, CLIP, workspace=ws, **kw)
        torch.cuda.synchronize()
        res.append((theta.cpu().numpy(), ms.cpu().numpy()))
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])
    assert flags[0].tolist() == [3, 3]  # three calls: ready and done of epoch 2 + 1


def test_rmsprop_sharded_learner_with_simulated_peer():
    """vtrace_rmsprop_step_sharded on one GPU (a second cooperative grid cannot share the
    GPU, so learner 1 is simulated): learner 0 owns float4 units [0, U/2); the peer's
    flags read "ready and done", and its shard sum of squares is placed in learner 0's
    norm mailbox with each call's tag.  Learner 0 must (a) update its shard of theta and
    ms like the oracle with the GLOBAL norm (own shard + the peer's, learner order),
    (b) write the same new theta into the peer's params for its shard only, (c) leave
    its other shard of theta and ms untouched, (d) report the global norm."""
    n = 200_000
    inp = wl.update_inputs(n, seed=31, norm=75.0, learners=2)
    dev = "cuda"
    gs = [torch.from_numpy(g).to(dev) for g in inp["grads"]]
    theta = torch.from_numpy(inp["params"]).to(dev)
    theta_peer = torch.from_numpy(inp["params"]).to(dev)
    ms = torch.from_numpy(inp["mean_square"]).to(dev)
    flags = torch.zeros(2, 2, dtype=torch.int32, device=dev)
    flags[1] = 1 << 30  # the simulated peer: ahead of every epoch used here
    nb = pkg.vtrace.rmsprop_norm_mailbox_bytes(2)
    assert nb == 2 * 2 * 16
    mbox = [torch.zeros(nb // 8, dtype=torch.float64, device=dev) for _ in range(2)]
    ws = pkg.RmspropWorkspace(n, dev)
    norm = torch.zeros(1, dtype=torch.float64, device=dev)
    U = n // 4
    cut = 4 * (U * 0 // 2), 4 * (U * 1 // 2)  # learner 0: elements [0, 4 * (U // 2))
    lo, hi = 0, cut[1]
    th_ref, ms_ref = inp["params"].copy(), inp["mean_square"].copy()
    total = ro.sum_learner_grads(inp["grads"])
    for call in range(3):
        # the peer's shard sum of squares (fp32 sums of the buffers, as the kernel adds them)
        g32 = (inp["grads"][0] + inp["grads"][1]).astype(np.float32).astype(np.float64)
        ss_peer = float(np.sum(g32[hi:] ** 2))
        tag = call + 1
        slot = (tag & 1) * 2 + 1  # [parity][learner 1]
        mbox[0][2 * slot] = ss_peer
        mbox[0].view(torch.int64)[2 * slot + 1] = tag
        pkg.vtrace.rmsprop_step_sharded(
            [theta.data_ptr(), theta_peer.data_ptr()], ms, [g.data_ptr() for g in gs],
            LR, DECAY, EPS, CLIP, flags=[flags[0].data_ptr(), flags[1].data_ptr()],
            norm_mailboxes=[m.data_ptr() for m in mbox], self_index=0, n=n, workspace=ws,
            global_norm_out=norm)
        torch.cuda.synchronize()
        th0 = th_ref.copy()
        th_ref, ms_ref, nr_ref = ro.rmsprop_step(th_ref, ms_ref, total, _f32(LR), _f32(DECAY),
                                                 _f32(EPS), _f32(CLIP))
        got_t, got_m = theta.cpu().numpy(), ms.cpu().numpy()
        _check(got_t[lo:hi], got_m[lo:hi], th0[lo:hi], th_ref[lo:hi], ms_ref[lo:hi])
        assert np.array_equal(theta_peer.cpu().numpy()[lo:hi], got_t[lo:hi])   # (b)
        assert np.array_equal(got_t[hi:], inp["params"][hi:])                   # (c)
        assert np.array_equal(got_m[hi:], inp["mean_square"][hi:])
        assert np.array_equal(theta_peer.cpu().numpy()[hi:], inp["params"][hi:])
        assert float(norm.item()) == pytest.approx(nr_ref, rel=1e-6)           # (d)
        # (keep the oracle's untouched shard equal to the kernel's for the next call)
        th_ref[hi:], ms_ref[hi:] = inp["params"][hi:], inp["mean_square"][hi:]
    assert flags[0].tolist() == [3, 3]


def test_grad_push_into_every_learners_slot():
    """vtrace_grad_push on one GPU (the learners' receive buffers simulated in local memory):
    learner 1 of 3 stores its gradient into slot 1 of every receive buffer, bit for bit, and
    touches nothing else; then the update summing the local slots equals the multi form."""
    n, N, me = 40_000, 3, 1
    dev = "cuda"
    g = torch.randn(n, device=dev)
    recv = [torch.full((N * n,), -7.0, device=dev) for _ in range(N)]
    pkg.vtrace.grad_push(g, [r.data_ptr() for r in recv], me)
    torch.cuda.synchronize()
    for r in recv:
        assert torch.equal(r[me * n:(me + 1) * n], g)
        assert bool((r[:me * n] == -7.0).all()) and bool((r[(me + 1) * n:] == -7.0).all())
    lib = pkg.load_library()
    assert lib.vtrace_grad_push(None, None, 2, 0, 8, None) == 1
    ptrs = (ctypes.c_void_p * 2)(recv[0].data_ptr(), recv[1].data_ptr())
    assert lib.vtrace_grad_push(ctypes.c_void_p(g.data_ptr()), ptrs, 2, 2, 8, None) == 1
    assert lib.vtrace_grad_push(ctypes.c_void_p(g.data_ptr()), ptrs, 2, 0, 6, None) == 2
