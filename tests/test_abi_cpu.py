"""CPU-only checks of the C-ABI library: it loads, exports every function that
include/vtrace.h declares, and rejects host-checkable bad arguments before
touching the device (no compute calls here)."""
import ctypes
import os
import re

import pytest

import paper_1802_01561_b200 as pkg
from paper_1802_01561_b200 import vtrace as vt

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "vtrace.h")


def _declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(vtrace_[a-z_]+)\s*\(", src)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    from paper_1802_01561_b200 import _build
    _build.build()
    return vt.load_library()


def test_header_declares_the_boundary():
    names = _declared_functions()
    for required in ("vtrace_from_logits", "vtrace_loss_and_grad", "vtrace_workspace_bytes",
                     "vtrace_read_device_status", "vtrace_status_string"):
        assert required in names
    assert set(names) == set(vt.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol(lib):
    for name in _declared_functions():
        assert hasattr(lib, name), name
    out = os.popen(f"nm -D --defined-only {vt.LIB_PATH}").read()
    for name in _declared_functions():
        assert re.search(rf"\bT {name}\b", out), name


def test_library_is_sm100a_only(lib):
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {vt.LIB_PATH}").read()
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out), out


def test_status_strings(lib):
    for s in range(9):
        assert pkg.status_string(s)
    assert pkg.status_string(0) == "ok"
    assert pkg.version() >= 100


def test_workspace_bytes(lib):
    assert pkg.workspace_bytes(0, 1, 1, 0) == 0
    assert pkg.workspace_bytes(5, 2, 3, 7) == 0
    assert pkg.workspace_bytes(5, 2, 3, 0) > 256
    big = pkg.workspace_bytes(100, 8192, 18, 1)
    assert big > pkg.workspace_bytes(100, 4096, 18, 1)
    # depends only on (T, B, A, dtype)
    assert big == pkg.workspace_bytes(100, 8192, 18, 1)


def _call_loss(lib, T=4, B=8, A=3, dt=0, ptr=0x10000, params=None, weights=None, ws=0x20000,
               ws_bytes=1 << 20, nulls=()):
    P = [ctypes.c_void_p(ptr)] * 7
    for i in nulls:
        P[i] = None
    p = params if params is not None else vt.params()
    w = weights if weights is not None else vt._Weights(0.5, 0.01)
    outs = [ctypes.c_void_p(ptr)] * 3 + [None, None]
    return lib.vtrace_loss_and_grad(T, B, A, dt, *P, ctypes.byref(p), ctypes.byref(w), *outs,
                                    ctypes.c_void_p(ws), ws_bytes, None)


def test_host_checks_return_before_launch(lib):
    assert _call_loss(lib, nulls=(0,)) == 1          # VT_ERR_INVALID_ARG
    assert _call_loss(lib, nulls=(6,)) == 1
    assert _call_loss(lib, T=0) == 2                 # VT_ERR_SHAPE
    assert _call_loss(lib, A=5000) == 2
    assert _call_loss(lib, dt=3) == 3                # VT_ERR_DTYPE
    assert _call_loss(lib, params=vt.params(rho_bar=1.0, c_bar=2.0)) == 4  # c_bar > rho_bar
    assert _call_loss(lib, params=vt.params(lambda_=1.5)) == 4
    assert _call_loss(lib, params=vt.params(rho_bar=float("nan"))) == 4
    assert _call_loss(lib, params=vt.params(reward_mode=9)) == 4
    assert _call_loss(lib, params=vt.params(correction=4)) == 4
    assert _call_loss(lib, params=vt.params(correction=-1)) == 4
    assert _call_loss(lib, params=vt.params(correction=2, epsilon=0.0)) == 4
    assert _call_loss(lib, params=vt.params(correction=2, epsilon=float("inf"))) == 4
    assert _call_loss(lib, params=vt.params(q_from_values=2)) == 4
    assert _call_loss(lib, weights=vt._Weights(float("inf"), 0.01)) == 4
    assert _call_loss(lib, ptr=0x10002) == 5         # VT_ERR_ALIGNMENT (fp32 data)
    assert _call_loss(lib, ws_bytes=16) == 6         # VT_ERR_WORKSPACE
    assert _call_loss(lib, ws=0x20010) == 6          # workspace not 256-aligned


def test_from_logits_requires_outputs(lib):
    P = [ctypes.c_void_p(0x10000)] * 7
    p = vt.params()
    st = lib.vtrace_from_logits(4, 8, 3, 0, *P, ctypes.byref(p), None, None, None, None, None,
                                ctypes.c_void_p(0x20000), 1 << 20, None)
    assert st == 1


def test_binding_has_no_cpu_fallback(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    x = torch.zeros(2, 2, 3)
    with pytest.raises((ValueError, RuntimeError, AssertionError)):
        pkg.loss_and_grad(x, x, torch.zeros(2, 2, dtype=torch.int32), torch.zeros(2, 2),
                          torch.zeros(2, 2), torch.zeros(2, 2), torch.zeros(2))


def test_kernel_choice(lib):
    """Host-only query of the kernel a shape takes: the column-block kernel wherever its
    TMA boxes apply (16-byte segments of 4 or 8 trajectories, an instantiated A), else
    the look-back kernel (TMA when the pitches are 16-byte multiples, else plain loads)."""
    cb = "vtrace_cb_kernel"
    assert vt.kernel_for(100, 8192, 18, 1) == cb                          # large
    assert vt.kernel_for(100, 4096, 18, 1) == cb                          # its N=2 shard
    assert vt.kernel_for(100, 1024, 18, 1) == cb                          # its N=8 shard
    assert vt.kernel_for(2000, 1024, 9, 0) == cb                          # stress
    assert vt.kernel_for(20, 32, 18, 0) == cb                             # atari
    assert vt.kernel_for(100, 32, 9, 1) == cb                             # dmlab (8-column segments)
    assert vt.kernel_for(100, 4096, 24, 1) == "vtrace_fused_kernel"       # A not instantiated
    assert vt.kernel_for(100, 4092, 9, 1) == "vtrace_fused_kernel (plain loads)"  # pitch % 16
    assert vt.kernel_for(100, 4096, 40, 1) == "vtrace_fused_kernel (plain loads)"  # 8 A > 256
    assert vt.kernel_for(5, 2, 3, 0) == "vtrace_cb_kernel (plain loads)"   # toy: pitch 24 B
    assert vt.kernel_for(2000, 1022, 9, 0) == "vtrace_fused_kernel (plain loads)"  # big, unaligned
    assert vt.kernel_for(0, 8, 3, 0).startswith("none")
    assert vt.kernel_for(5, 8, 3, 7).startswith("none")


def test_kernel_and_sm_budget_param_checks(lib):
    assert _call_loss(lib, params=vt.params(kernel=3)) == 4
    assert _call_loss(lib, params=vt.params(kernel=-1)) == 4
    assert _call_loss(lib, params=vt.params(sm_budget=-2)) == 4


def test_behaviour_log_prob_param_check(lib):
    assert _call_loss(lib, params=vt.params(behaviour_log_probs=2)) == 4


def test_overlap_previous_param_check(lib):
    assert _call_loss(lib, params=vt.params(overlap_previous=2)) == 4


def _rms(lib, n=10, p=16, m=32, g=48, prm=None, ws=None, wsb=0, norm=None):
    prm = prm if prm is not None else vt._RmsParams(6e-4, 0.99, 0.01, 40.0)
    c = (lambda x: None if x is None else ctypes.c_void_p(x))
    return lib.vtrace_rmsprop_step(n, c(p), c(m), c(g), ctypes.byref(prm), c(norm), c(ws), wsb,
                                   None)


def test_rmsprop_host_checks(lib):
    """vtrace_rmsprop_step (NEXT #4) rejects bad arguments before any launch."""
    assert lib.vtrace_rmsprop_workspace_bytes(1_600_000) >= 256 + 16 * 148
    assert lib.vtrace_rmsprop_workspace_bytes(-1) == 0
    assert _rms(lib, p=None) == 1                                  # INVALID_ARG
    assert _rms(lib, n=-1) == 2                                    # SHAPE
    for bad in ((0.0, 0.99, 0.01, 40.0), (float("nan"), 0.99, 0.01, 40.0),
                (6e-4, 1.0, 0.01, 40.0), (6e-4, -0.1, 0.01, 40.0), (6e-4, 0.99, 0.0, 40.0),
                (6e-4, 0.99, 0.01, -1.0), (6e-4, 0.99, 0.01, float("inf"))):
        assert _rms(lib, prm=vt._RmsParams(*bad)) == 4, bad          # PARAM
    assert _rms(lib, p=18) == 5                                    # ALIGNMENT
    assert _rms(lib, norm=20) == 5
    assert _rms(lib) == 6                                          # WORKSPACE (NULL)
    assert _rms(lib, ws=256, wsb=16) == 6                          # too small
    assert _rms(lib, ws=300, wsb=1 << 20) == 6                     # not 256-aligned


def test_rmsprop_multi_host_checks(lib):
    prm = vt._RmsParams(6e-4, 0.99, 0.01, 40.0)

    def call(ptrs, ng, n=10):
        arr = (ctypes.c_void_p * max(len(ptrs), 1))(*ptrs)
        return lib.vtrace_rmsprop_step_multi(n, ctypes.c_void_p(16), ctypes.c_void_p(32), arr,
                                             ng, ctypes.byref(prm), None, None, 0, None)
    assert call([48, 64], 0) == 1                 # no gradient
    assert call([48] * 9, 9) == 1                 # more than 8
    assert call([48, None], 2) == 1               # a NULL buffer
    assert call([48, 66], 2) == 5                 # a misaligned buffer
    assert call([48, 64], 2) == 6                 # then the workspace check
    assert lib.vtrace_rmsprop_step_multi(10, ctypes.c_void_p(16), ctypes.c_void_p(32), None, 1,
                                         ctypes.byref(prm), None, None, 0, None) == 1


def test_rmsprop_learners_host_checks(lib):
    prm = vt._RmsParams(6e-4, 0.99, 0.01, 40.0)
    g = (ctypes.c_void_p * 2)(48, 64)

    def call(flags, self_index):
        fl = None if flags is None else (ctypes.c_void_p * 2)(*flags)
        return lib.vtrace_rmsprop_step_learners(10, ctypes.c_void_p(16), ctypes.c_void_p(32), g,
                                                fl, 2, self_index, ctypes.byref(prm), None, None,
                                                0, None)
    assert call(None, 0) == 1          # no flags
    assert call([128, None], 0) == 1   # a NULL flag pointer
    assert call([128, 136], 2) == 1    # self out of range
    assert call([128, 132], 0) == 5    # flags not 8-byte aligned
    assert call([128, 136], 1) == 6    # then the workspace check


def test_output_layer_host_checks(lib):
    """vtrace_output_layer (NEXT #3) validates shapes, pointers and alignment on the host,
    before touching a device: H not a multiple of 64 or > 256, A + 1 > 32, M < 0 ->
    VT_ERR_SHAPE; M = 0 -> no-op; NULL -> VT_ERR_INVALID_ARG; misaligned h -> VT_ERR_ALIGNMENT."""
    buf = ctypes.create_string_buffer(1 << 16)
    base = (ctypes.addressof(buf) + 255) & ~255
    p = ctypes.c_void_p(base)
    f = lib.vtrace_output_layer
    assert f(128, 100, 9, p, p, None, p, p, None) == 2
    assert f(128, 320, 9, p, p, None, p, p, None) == 2
    assert f(128, 256, 32, p, p, None, p, p, None) == 2
    assert f(128, 256, 0, p, p, None, p, p, None) == 2
    assert f(-1, 256, 9, p, p, None, p, p, None) == 2
    assert f(0, 256, 9, None, None, None, None, None, None) == 0
    assert f(128, 256, 9, None, p, None, p, p, None) == 1
    assert f(128, 256, 9, p, p, None, p, None, None) == 1
    assert f(128, 256, 9, ctypes.c_void_p(base + 8), p, None, p, p, None) == 5
    assert f(128, 256, 9, p, ctypes.c_void_p(base + 4), None, p, p, None) == 5


def test_partials_allreduce_host_checks(lib):
    """vtrace_partials_allreduce (row a13 over NVLink) checks its arguments on the host:
    mailbox size for 1..16 learners; NULL pointers, learner count or index out of range ->
    VT_ERR_INVALID_ARG; misaligned partials / counter / mailbox -> VT_ERR_ALIGNMENT."""
    assert lib.vtrace_partials_mailbox_bytes(0) == 0
    assert lib.vtrace_partials_mailbox_bytes(17) == 0
    assert lib.vtrace_partials_mailbox_bytes(4) == 2 * 4 * 8 * 16
    p = ctypes.c_void_p(4096)
    mb = (ctypes.c_void_p * 2)(8192, 12288)
    f = lib.vtrace_partials_allreduce
    assert f(None, mb, 2, 0, p, p, None) == 1
    assert f(p, None, 2, 0, p, p, None) == 1
    assert f(p, mb, 0, 0, p, p, None) == 1
    assert f(p, mb, 2, 2, p, p, None) == 1
    assert f(p, (ctypes.c_void_p * 2)(8192, None), 2, 0, p, p, None) == 1
    assert f(ctypes.c_void_p(4100), mb, 2, 0, p, p, None) == 5
    assert f(p, mb, 2, 0, ctypes.c_void_p(4100), p, None) == 5
    assert f(p, (ctypes.c_void_p * 2)(8192, 12296), 2, 0, p, p, None) == 5


def test_head_loss_and_grad_host_checks(lib):
    """vtrace_head_loss_and_grad (NEXT #3 second half) validates on the host before any
    device work: NULL -> 1, H / A / B out of range -> 2, misaligned -> 5, workspace -> 6."""
    buf = ctypes.create_string_buffer(1 << 16)
    base = (ctypes.addressof(buf) + 255) & ~255
    p = ctypes.c_void_p(base)
    prm = vt.params()
    w = vt._Weights(0.5, 0.01)
    f = lib.vtrace_head_loss_and_grad
    big = lib.vtrace_head_workspace_bytes(10, 8, 256, 18)
    assert big > 0 and lib.vtrace_head_workspace_bytes(10, 8, 256, 5 + 27) == 0

    def call(T=10, B=8, H=256, A=18, h=p, ws=p, nbytes=big, grad=p):
        return f(T, B, H, A, h, p, None, p, p, p, p, p, ctypes.byref(prm), ctypes.byref(w),
                 grad, p, p, p, ws, nbytes, None)
    assert call(h=None) == 1
    assert call(grad=None) == 1
    assert call(H=192) == 2
    assert call(A=5) == 2
    assert call(B=6) == 2
    assert call(T=0) == 2
    assert call(h=ctypes.c_void_p(base + 8)) == 5
    assert call(nbytes=16) == 6
    assert call(ws=None) == 6


def test_round2_entry_points_host_checks(lib):
    """Host-side argument checks of the round-2 entry points, before any device work:
    vtrace_partials_allreduce_batched, vtrace_grad_push, vtrace_rmsprop_step_sharded,
    vtrace_loss_and_grad_learners (NULL -> 1, shape -> 2, alignment -> 5)."""
    P = ctypes.c_void_p
    p = P(4096)
    two = (ctypes.c_void_p * 2)(8192, 12288)
    # batched partials sum
    f = lib.vtrace_partials_allreduce_batched
    assert lib.vtrace_partials_mailbox_bytes_batched(2, 0) == 0
    assert lib.vtrace_partials_mailbox_bytes_batched(2, 33) == 0
    assert lib.vtrace_partials_mailbox_bytes_batched(2, 4) == 2 * 2 * 4 * 8 * 16
    assert f(None, 1, 4, two, 2, 0, p, None) == 1
    assert f(two, 0, 4, two, 2, 0, p, None) == 1
    assert f(two, 5, 4, two, 2, 0, p, None) == 1   # batch > batch_max
    assert f(two, 2, 33, two, 2, 0, p, None) == 1
    assert f(two, 2, 4, two, 2, 2, p, None) == 1
    assert f(two, 2, 4, two, 2, 0, P(4100), None) == 5
    assert f((ctypes.c_void_p * 2)(8192, 12292), 2, 4, two, 2, 0, p, None) == 5
    # gradient push
    g = lib.vtrace_grad_push
    assert g(None, two, 2, 0, 8, None) == 1
    assert g(p, None, 2, 0, 8, None) == 1
    assert g(p, two, 2, 2, 8, None) == 1
    assert g(p, two, 2, 0, 6, None) == 2
    assert g(P(4100), two, 2, 0, 8, None) == 5
    # sharded update
    prm = vt._RmsParams(6e-4, 0.99, 0.01, 40.0)
    h = lib.vtrace_rmsprop_step_sharded
    fl = (ctypes.c_void_p * 2)(16384, 16392)
    assert h(8, None, p, two, fl, two, 2, 0, ctypes.byref(prm), None, None, 0, None) == 1
    assert h(8, two, p, two, None, two, 2, 0, ctypes.byref(prm), None, None, 0, None) == 1
    assert h(8, two, p, two, fl, None, 2, 0, ctypes.byref(prm), None, None, 0, None) == 1
    assert h(8, two, p, two, fl, two, 2, 3, ctypes.byref(prm), None, None, 0, None) == 1
    # learners' V-trace
    w = vt._Weights(0.5, 0.01)
    q = vt.params()
    k = lib.vtrace_loss_and_grad_learners
    args = [10, 8, 18, 1] + [p] * 7 + [ctypes.byref(q), ctypes.byref(w)] + [p] * 5 + [p, 0]
    assert k(*args, None, 2, 0, None) == 1
    assert k(*args, two, 0, 0, None) == 1
    assert k(*args, two, 2, 2, None) == 1
    assert k(*args, (ctypes.c_void_p * 2)(8192, 12296), 2, 0, None) == 5
