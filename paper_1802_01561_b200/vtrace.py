"""Thin Python binding of the C ABI in include/vtrace.h (argument marshalling only).

Every computation runs in libvtrace.so's CUDA kernels; this module only turns
torch tensors into pointers and the current CUDA stream into a handle.  There
is no CPU fallback: if the library is missing or the device is not an sm_100
B200, calls raise.

Names follow the C ABI: ``workspace_bytes``, ``Workspace`` (alloc + init),
``from_logits``, ``loss_and_grad``, ``loss_and_grad_from_host``,
``read_device_status``, ``status_string``.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import workload as _wl

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libvtrace.so")

VT_FLOAT32 = 0
VT_BFLOAT16 = 1
P_PG_LOSS, P_BASELINE_LOSS, P_ENTROPY_SUM, P_TOTAL_LOSS = 0, 1, 2, 3
P_SUMSQ_DLOGITS, P_SUMSQ_DVALUES, P_SUM_RHO, P_N_RHO_CLIPPED = 4, 5, 6, 7
P_COUNT = 8
PARTIAL_NAMES = ("pg_loss", "baseline_loss", "entropy_sum", "total_loss", "sumsq_dlogits",
                 "sumsq_dvalues", "sum_rho", "n_rho_clipped")
DATA_ERRORS = {0: "ok", 1: "action", 2: "logits", 3: "reward", 4: "value", 5: "discount"}

EXPORTED_SYMBOLS = ("vtrace_workspace_bytes", "vtrace_workspace_init", "vtrace_from_logits",
                    "vtrace_loss_and_grad", "vtrace_loss_and_grad_from_host",
                    "vtrace_read_device_status", "vtrace_status_string", "vtrace_version",
                    "vtrace_kernel_for", "vtrace_rmsprop_workspace_bytes", "vtrace_rmsprop_step",
                    "vtrace_rmsprop_step_multi", "vtrace_rmsprop_step_learners",
                    "vtrace_output_layer", "vtrace_partials_mailbox_bytes",
                    "vtrace_partials_allreduce", "vtrace_head_workspace_bytes",
                    "vtrace_head_loss_and_grad", "vtrace_rmsprop_norm_mailbox_bytes",
                    "vtrace_rmsprop_step_sharded", "vtrace_grad_push",
                    "vtrace_loss_and_grad_learners", "vtrace_partials_mailbox_bytes_batched",
                    "vtrace_partials_allreduce_batched")


class VtraceError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {status_string(status)} (status {status})")


class _Params(ctypes.Structure):
    _fields_ = [("clip_rho_threshold", ctypes.c_float), ("clip_c_threshold", ctypes.c_float),
                ("clip_pg_rho_threshold", ctypes.c_float), ("lambda_", ctypes.c_float),
                ("reward_mode", ctypes.c_int32), ("correction", ctypes.c_int32),
                ("epsilon", ctypes.c_float), ("q_from_values", ctypes.c_int32),
                ("behaviour_log_probs", ctypes.c_int32), ("overlap_previous", ctypes.c_int32),
                ("kernel", ctypes.c_int32), ("sm_budget", ctypes.c_int32)]


# vt_kernel: which kernel runs a call (0 = automatic; tests / A-B only)
KERNEL_AUTO, KERNEL_COLUMN_BLOCK, KERNEL_LOOKBACK = 0, 1, 2


# vt_correction: Section 5.2.2 off-policy correction variants
CORRECTION_VTRACE, CORRECTION_NONE, CORRECTION_EPSILON, CORRECTION_ONE_STEP_IS = 0, 1, 2, 3


class _RmsParams(ctypes.Structure):  # vt_rmsprop_params
    _fields_ = [("learning_rate", ctypes.c_float), ("decay", ctypes.c_float),
                ("epsilon", ctypes.c_float), ("max_global_norm", ctypes.c_float)]


class _Weights(ctypes.Structure):
    _fields_ = [("baseline_cost", ctypes.c_float), ("entropy_cost", ctypes.c_float)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Loads libvtrace.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run `python -m paper_1802_01561_b200._build` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(path)
    P = ctypes.c_void_p
    i64 = ctypes.c_int64
    lib.vtrace_workspace_bytes.argtypes = [i64, i64, i64, ctypes.c_int]
    lib.vtrace_workspace_bytes.restype = ctypes.c_size_t
    lib.vtrace_workspace_init.argtypes = [P, ctypes.c_size_t, P]
    lib.vtrace_workspace_init.restype = ctypes.c_int
    lib.vtrace_from_logits.argtypes = [i64, i64, i64, ctypes.c_int] + [P] * 7 + [
        ctypes.POINTER(_Params)] + [P] * 5 + [P, ctypes.c_size_t, P]
    lib.vtrace_from_logits.restype = ctypes.c_int
    lib.vtrace_loss_and_grad.argtypes = [i64, i64, i64, ctypes.c_int] + [P] * 7 + [
        ctypes.POINTER(_Params), ctypes.POINTER(_Weights)] + [P] * 5 + [P, ctypes.c_size_t, P]
    lib.vtrace_loss_and_grad.restype = ctypes.c_int
    lib.vtrace_loss_and_grad_learners.argtypes = [i64, i64, i64, ctypes.c_int] + [P] * 7 + [
        ctypes.POINTER(_Params), ctypes.POINTER(_Weights)] + [P] * 5 + [
        P, ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32, ctypes.c_int32, P]
    lib.vtrace_loss_and_grad_learners.restype = ctypes.c_int
    lib.vtrace_loss_and_grad_from_host.argtypes = [i64, i64, i64, ctypes.c_int] + [P] * 14 + [
        ctypes.POINTER(_Params), ctypes.POINTER(_Weights)] + [P] * 4 + [P, ctypes.c_size_t, P]
    lib.vtrace_loss_and_grad_from_host.restype = ctypes.c_int
    lib.vtrace_read_device_status.argtypes = [P, ctypes.POINTER(ctypes.c_int32),
                                              ctypes.POINTER(ctypes.c_int64), P]
    lib.vtrace_read_device_status.restype = ctypes.c_int
    lib.vtrace_status_string.argtypes = [ctypes.c_int]
    lib.vtrace_status_string.restype = ctypes.c_char_p
    lib.vtrace_version.argtypes = []
    lib.vtrace_version.restype = ctypes.c_int32
    lib.vtrace_kernel_for.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int]
    lib.vtrace_kernel_for.restype = ctypes.c_char_p
    lib.vtrace_rmsprop_workspace_bytes.argtypes = [i64]
    lib.vtrace_rmsprop_workspace_bytes.restype = ctypes.c_size_t
    lib.vtrace_rmsprop_step.argtypes = [i64, P, P, P, ctypes.POINTER(_RmsParams), P, P,
                                        ctypes.c_size_t, P]
    lib.vtrace_rmsprop_step.restype = ctypes.c_int
    lib.vtrace_rmsprop_step_multi.argtypes = [i64, P, P, ctypes.POINTER(ctypes.c_void_p),
                                              ctypes.c_int32, ctypes.POINTER(_RmsParams), P, P,
                                              ctypes.c_size_t, P]
    lib.vtrace_rmsprop_step_multi.restype = ctypes.c_int
    lib.vtrace_rmsprop_step_learners.argtypes = [i64, P, P, ctypes.POINTER(ctypes.c_void_p),
                                                 ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32,
                                                 ctypes.c_int32, ctypes.POINTER(_RmsParams), P, P,
                                                 ctypes.c_size_t, P]
    lib.vtrace_rmsprop_step_learners.restype = ctypes.c_int
    lib.vtrace_output_layer.argtypes = [i64, ctypes.c_int32, ctypes.c_int32, P, P, P, P, P, P]
    lib.vtrace_output_layer.restype = ctypes.c_int
    lib.vtrace_partials_mailbox_bytes.argtypes = [ctypes.c_int32]
    lib.vtrace_partials_mailbox_bytes.restype = ctypes.c_size_t
    lib.vtrace_partials_allreduce.argtypes = [P, ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32,
                                              ctypes.c_int32, P, P, P]
    lib.vtrace_partials_allreduce.restype = ctypes.c_int
    lib.vtrace_partials_mailbox_bytes_batched.argtypes = [ctypes.c_int32, ctypes.c_int32]
    lib.vtrace_partials_mailbox_bytes_batched.restype = ctypes.c_size_t
    lib.vtrace_partials_allreduce_batched.argtypes = [ctypes.POINTER(ctypes.c_void_p),
                                                      ctypes.c_int32, ctypes.c_int32,
                                                      ctypes.POINTER(ctypes.c_void_p),
                                                      ctypes.c_int32, ctypes.c_int32, P, P]
    lib.vtrace_partials_allreduce_batched.restype = ctypes.c_int
    lib.vtrace_rmsprop_norm_mailbox_bytes.argtypes = [ctypes.c_int32]
    lib.vtrace_rmsprop_norm_mailbox_bytes.restype = ctypes.c_size_t
    lib.vtrace_rmsprop_step_sharded.argtypes = [i64, ctypes.POINTER(ctypes.c_void_p), P,
                                                ctypes.POINTER(ctypes.c_void_p),
                                                ctypes.POINTER(ctypes.c_void_p),
                                                ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32,
                                                ctypes.c_int32, ctypes.POINTER(_RmsParams), P, P,
                                                ctypes.c_size_t, P]
    lib.vtrace_rmsprop_step_sharded.restype = ctypes.c_int
    lib.vtrace_grad_push.argtypes = [P, ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32,
                                     ctypes.c_int32, i64, P]
    lib.vtrace_grad_push.restype = ctypes.c_int
    lib.vtrace_head_workspace_bytes.argtypes = [i64, i64, ctypes.c_int32, ctypes.c_int32]
    lib.vtrace_head_workspace_bytes.restype = ctypes.c_size_t
    lib.vtrace_head_loss_and_grad.argtypes = [i64, i64, ctypes.c_int32, ctypes.c_int32] + [P] * 8 + [
        ctypes.POINTER(_Params), ctypes.POINTER(_Weights)] + [P] * 5 + [ctypes.c_size_t, P]
    lib.vtrace_head_loss_and_grad.restype = ctypes.c_int
    _lib = lib
    return lib


def status_string(status: int) -> str:
    return load_library().vtrace_status_string(int(status)).decode()


def _check(status: int, where: str):
    if status != 0:
        raise VtraceError(status, where)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return VT_FLOAT32
    if t.dtype == torch.bfloat16:
        return VT_BFLOAT16
    raise TypeError(f"logits must be float32 or bfloat16, got {t.dtype}")


def params(rho_bar=1.0, c_bar=1.0, pg_rho_bar=None, lambda_=1.0, reward_mode=0,
           correction=CORRECTION_VTRACE, epsilon=1e-6, q_from_values=0,
           behaviour_log_probs=0, overlap_previous=0, kernel=KERNEL_AUTO,
           sm_budget=0) -> _Params:
    return _Params(float(rho_bar), float(c_bar),
                   float(rho_bar if pg_rho_bar is None else pg_rho_bar), float(lambda_),
                   int(reward_mode), int(correction), float(epsilon), int(q_from_values),
                   int(behaviour_log_probs), int(overlap_previous), int(kernel), int(sm_budget))


def workspace_bytes(T: int, B: int, A: int, dtype_code: int) -> int:
    return int(load_library().vtrace_workspace_bytes(T, B, A, dtype_code))


class Workspace:
    """Device workspace for (T, B, A, dtype): allocated once, initialised once."""

    def __init__(self, T, B, A, dtype_code, device=None):
        n = workspace_bytes(T, B, A, dtype_code)
        if n == 0:
            raise ValueError("bad shape for workspace")
        self.device = torch.device(device if device is not None else "cuda")
        self.nbytes = n
        self.buf = torch.empty(n + 256, dtype=torch.uint8, device=self.device)
        off = (-self.buf.data_ptr()) % 256
        self.tensor = self.buf[off:off + n]
        _check(load_library().vtrace_workspace_init(_ptr(self.tensor), n, _stream(self.device)),
               "vtrace_workspace_init")

    @property
    def ptr(self):
        return _ptr(self.tensor)


def _shapes(behaviour_logits, target_logits, actions, discounts, rewards, values,
            bootstrap_value):
    """(T, B, A, mu_lp) after checking every input's shape, dtype, layout and device
    (the kernels trust these; a wrong dtype or an undersized buffer would be misread).
    The behaviour input is either mu's [T, B, A] logits (the target logits' dtype) or,
    in behaviour-log-prob mode, log mu(a_t) as a [T, B] float32 tensor."""
    if target_logits.dim() != 3:
        raise ValueError("target logits must be [T, B, A]")
    T, B, A = target_logits.shape
    _dtype_code(target_logits)
    if behaviour_logits.dim() == 2:
        if behaviour_logits.shape != (T, B) or behaviour_logits.dtype != torch.float32:
            raise ValueError("behaviour log-probs must be a [T, B] float32 tensor")
        mu_lp = 1
    elif behaviour_logits.shape != target_logits.shape:
        raise ValueError("behaviour and target logits must have equal [T, B, A] shapes")
    elif behaviour_logits.dtype != target_logits.dtype:
        raise ValueError("behaviour and target logits must have the same dtype")
    else:
        mu_lp = 0
    if actions.shape != (T, B) or actions.dtype != torch.int32:
        raise ValueError("actions must be a [T, B] int32 tensor")
    for name, t in (("discounts", discounts), ("rewards", rewards), ("values", values)):
        if t.shape != (T, B) or t.dtype != torch.float32:
            raise ValueError(f"{name} must be a [T, B] float32 tensor")
    if bootstrap_value.shape != (B,) or bootstrap_value.dtype != torch.float32:
        raise ValueError("bootstrap_value must be a [B] float32 tensor")
    _contig(behaviour_logits, target_logits, actions, discounts, rewards, values, bootstrap_value)
    dev = target_logits.device
    for t in (behaviour_logits, actions, discounts, rewards, values, bootstrap_value):
        if t.device != dev:
            raise ValueError("all inputs must be on the same device")
    return T, B, A, mu_lp


def _check_out(out: dict, specs: dict, dev):
    """Caller-supplied outputs: present where required, right dtype, shape, layout, device."""
    for k, (shape, dtype, required) in specs.items():
        t = out.get(k)
        if t is None:
            if required:
                raise ValueError(f"out[{k!r}] is required")
            continue
        if tuple(t.shape) != tuple(shape) or t.dtype != dtype or not t.is_contiguous() or \
                t.device != dev:
            raise ValueError(f"out[{k!r}] must be a contiguous {dtype} tensor of shape "
                             f"{tuple(shape)} on {dev}")


def _contig(*ts):
    for t in ts:
        if t is not None and not t.is_contiguous():
            raise ValueError("all tensors must be contiguous")
        if t is not None and not t.is_cuda:
            raise ValueError("all tensors must be CUDA tensors")


def from_logits(behaviour_logits, target_logits, actions, discounts, rewards, values,
                bootstrap_value, *, rho_bar=1.0, c_bar=1.0, pg_rho_bar=None, lambda_=1.0,
                reward_mode=0, correction=CORRECTION_VTRACE, epsilon=1e-6, q_from_values=0,
                overlap_previous=False, workspace: Workspace | None = None, with_log_probs=True,
                out: dict | None = None, kernel=KERNEL_AUTO, sm_budget=0):
    """vtrace_from_logits.  Returns dict of fp32 [T, B] tensors: vs,
    pg_advantages (+ log_rhos, target_action_log_probs, behaviour_action_log_probs)."""
    lib = load_library()
    T, B, A, mu_lp = _shapes(behaviour_logits, target_logits, actions, discounts, rewards, values,
                             bootstrap_value)
    dt = _dtype_code(target_logits)
    dev = target_logits.device
    ws = workspace if workspace is not None else Workspace(T, B, A, dt, dev)
    if out is None:
        out = {k: torch.empty(T, B, dtype=torch.float32, device=dev) for k in ("vs", "pg_advantages")}
        if with_log_probs:
            for k in ("log_rhos", "target_action_log_probs", "behaviour_action_log_probs"):
                out[k] = torch.empty(T, B, dtype=torch.float32, device=dev)
    else:
        f = torch.float32
        _check_out(out, {"vs": ((T, B), f, True), "pg_advantages": ((T, B), f, True),
                         "log_rhos": ((T, B), f, False), "target_action_log_probs": ((T, B), f, False),
                         "behaviour_action_log_probs": ((T, B), f, False)}, dev)
    p = params(rho_bar, c_bar, pg_rho_bar, lambda_, reward_mode, correction, epsilon, q_from_values,
               mu_lp, int(overlap_previous), kernel, sm_budget)
    st = lib.vtrace_from_logits(
        T, B, A, dt, _ptr(behaviour_logits), _ptr(target_logits), _ptr(actions), _ptr(discounts),
        _ptr(rewards), _ptr(values), _ptr(bootstrap_value), ctypes.byref(p), _ptr(out["vs"]),
        _ptr(out["pg_advantages"]), _ptr(out.get("log_rhos")),
        _ptr(out.get("target_action_log_probs")), _ptr(out.get("behaviour_action_log_probs")),
        ws.ptr, ws.nbytes, _stream(dev))
    _check(st, "vtrace_from_logits")
    return out


def loss_and_grad(behaviour_logits, target_logits, actions, discounts, rewards, values,
                  bootstrap_value, *, rho_bar=1.0, c_bar=1.0, pg_rho_bar=None, lambda_=1.0,
                  reward_mode=0, correction=CORRECTION_VTRACE, epsilon=1e-6, q_from_values=0,
                  baseline_cost=0.5, entropy_cost=0.01, overlap_previous=False,
                  workspace: Workspace | None = None, with_targets=True, out: dict | None = None,
                  kernel=KERNEL_AUTO, sm_budget=0, mailboxes=None, self_index: int = 0):
    """vtrace_loss_and_grad.  Returns dict: grad_target_logits [T,B,A] (logits
    dtype), grad_values [T,B] fp32, partials [8] fp64 (device), and, if
    with_targets, vs and pg_advantages [T,B] fp32.  With ``mailboxes`` (one peer-mapped
    device pointer per learner) it is vtrace_loss_and_grad_learners: ``partials`` is the
    sum over the learners, exchanged inside the kernel (``self_index`` = this learner)."""
    lib = load_library()
    T, B, A, mu_lp = _shapes(behaviour_logits, target_logits, actions, discounts, rewards, values,
                             bootstrap_value)
    dt = _dtype_code(target_logits)
    dev = target_logits.device
    ws = workspace if workspace is not None else Workspace(T, B, A, dt, dev)
    if out is None:
        out = {"grad_target_logits": torch.empty_like(target_logits),
               "grad_values": torch.empty(T, B, dtype=torch.float32, device=dev),
               "partials": torch.empty(P_COUNT, dtype=torch.float64, device=dev)}
        if with_targets:
            out["vs"] = torch.empty(T, B, dtype=torch.float32, device=dev)
            out["pg_advantages"] = torch.empty(T, B, dtype=torch.float32, device=dev)
    else:
        f = torch.float32
        _check_out(out, {"grad_target_logits": ((T, B, A), target_logits.dtype, True),
                         "grad_values": ((T, B), f, True), "partials": ((P_COUNT,), torch.float64, True),
                         "vs": ((T, B), f, False), "pg_advantages": ((T, B), f, False)}, dev)
    p = params(rho_bar, c_bar, pg_rho_bar, lambda_, reward_mode, correction, epsilon, q_from_values,
               mu_lp, int(overlap_previous), kernel, sm_budget)
    w = _Weights(float(baseline_cost), float(entropy_cost))
    if mailboxes is not None:
        mb = _ptr_array([int(m) for m in mailboxes])
        st = lib.vtrace_loss_and_grad_learners(
            T, B, A, dt, _ptr(behaviour_logits), _ptr(target_logits), _ptr(actions),
            _ptr(discounts), _ptr(rewards), _ptr(values), _ptr(bootstrap_value), ctypes.byref(p),
            ctypes.byref(w), _ptr(out["grad_target_logits"]), _ptr(out["grad_values"]),
            _ptr(out["partials"]), _ptr(out.get("vs")), _ptr(out.get("pg_advantages")), ws.ptr,
            ws.nbytes, mb, len(mailboxes), int(self_index), _stream(dev))
        _check(st, "vtrace_loss_and_grad_learners")
        return out
    st = lib.vtrace_loss_and_grad(
        T, B, A, dt, _ptr(behaviour_logits), _ptr(target_logits), _ptr(actions), _ptr(discounts),
        _ptr(rewards), _ptr(values), _ptr(bootstrap_value), ctypes.byref(p), ctypes.byref(w),
        _ptr(out["grad_target_logits"]), _ptr(out["grad_values"]), _ptr(out["partials"]),
        _ptr(out.get("vs")), _ptr(out.get("pg_advantages")), ws.ptr, ws.nbytes, _stream(dev))
    _check(st, "vtrace_loss_and_grad")
    return out


def loss_and_grad_from_host(host: dict, dev_in: dict, out: dict, workspace: Workspace,
                            partials_host: torch.Tensor, *, rho_bar=1.0, c_bar=1.0,
                            pg_rho_bar=None, lambda_=1.0, reward_mode=0,
                            correction=CORRECTION_VTRACE, epsilon=1e-6, q_from_values=0,
                            baseline_cost=0.5, entropy_cost=0.01):
    """vtrace_loss_and_grad_from_host: ``host`` holds pinned CPU tensors of the
    seven inputs, ``dev_in`` same-shaped device staging tensors, ``out`` the
    device outputs (grad_target_logits, grad_values, partials);
    ``partials_host`` a pinned float64 [8] tensor filled asynchronously."""
    lib = load_library()
    T, B, A = host["target_logits"].shape
    dt = _dtype_code(host["target_logits"])
    dev = dev_in["target_logits"].device
    names = ("behaviour_logits", "target_logits", "actions", "discounts", "rewards", "values",
             "bootstrap_value")
    mu_lp = 1 if host["behaviour_logits"].dim() == 2 else 0  # log mu(a_t) [T, B] mode
    p = params(rho_bar, c_bar, pg_rho_bar, lambda_, reward_mode, correction, epsilon, q_from_values,
               mu_lp, 0)  # (its inputs come from the copies just before)
    w = _Weights(float(baseline_cost), float(entropy_cost))
    st = lib.vtrace_loss_and_grad_from_host(
        T, B, A, dt, *[_ptr(host[k]) for k in names], *[_ptr(dev_in[k]) for k in names],
        ctypes.byref(p), ctypes.byref(w), _ptr(out["grad_target_logits"]),
        _ptr(out["grad_values"]), _ptr(out["partials"]), _ptr(partials_host), workspace.ptr,
        workspace.nbytes, _stream(dev))
    _check(st, "vtrace_loss_and_grad_from_host")


def read_device_status(workspace: Workspace):
    """Synchronising read-and-clear of the data-error status: (kind, first_bad_row)."""
    code = ctypes.c_int32(0)
    idx = ctypes.c_int64(-1)
    _check(load_library().vtrace_read_device_status(workspace.ptr, ctypes.byref(code),
                                                     ctypes.byref(idx),
                                                     _stream(workspace.device)),
           "vtrace_read_device_status")
    return int(code.value), int(idx.value)


def version() -> int:
    return int(load_library().vtrace_version())


def kernel_for(T: int, B: int, A: int, dtype) -> str:
    """Name of the kernel a (T, B, A, dtype) call takes (16-byte aligned tensors);
    dtype: torch.float32 / torch.bfloat16 or the library code (0 / 1)."""
    code = dtype if isinstance(dtype, int) else {torch.float32: VT_FLOAT32,
                                                  torch.bfloat16: VT_BFLOAT16}[dtype]
    return load_library().vtrace_kernel_for(int(T), int(B), int(A), int(code)).decode()


# ---------------------------------------------------------------------------
# marshalling of the synthetic workload dicts (numpy, library layout) to tensors

INPUT_NAMES = ("behaviour_logits", "target_logits", "actions", "discounts", "rewards", "values",
               "bootstrap_value")


def tensors_from_workload(inp: dict, device="cuda", pin: bool = False) -> dict:
    """numpy workload dict -> torch tensors (bf16 logits from their uint16 bits).
    If the dict carries ``behaviour_log_probs`` ([T, B] log mu(a_t)), that array is
    the behaviour input (the "behaviour_logits" slot) instead of the logits."""
    out = {}
    for k in INPUT_NAMES:
        a = inp[k]
        if k == "behaviour_logits" and inp.get("behaviour_log_probs") is not None:
            a = np.ascontiguousarray(inp["behaviour_log_probs"], dtype=np.float32)
            t = torch.from_numpy(a)
            out[k] = (t.pin_memory() if pin else t.clone()) if device == "cpu" else t.to(device)
            continue
        if k.endswith("logits") and inp["dtype"] == _wl.DTYPE_BF16:
            t = torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16)
        else:
            t = torch.from_numpy(np.ascontiguousarray(a))
        if device == "cpu":
            out[k] = t.pin_memory() if pin else t.clone()
        else:
            out[k] = t.to(device)
    return out


def call_kwargs(inp: dict) -> dict:
    """Method parameters that a workload dict implies (reward transform)."""
    return {"reward_mode": int(inp.get("reward_mode", 0))}


__all__ = ["workspace_bytes", "Workspace", "from_logits", "loss_and_grad",
           "loss_and_grad_from_host", "read_device_status", "status_string", "version",
           "tensors_from_workload", "VtraceError", "load_library"]


# ---- the learner's parameter update (include/vtrace.h) ----

_RMS_PRM_CACHE: dict = {}
_PTR_ARRAYS: dict = {}


def _ptr_array(ptrs):
    """ctypes array of device pointers, cached by value (same buffers every step)."""
    key = tuple(ptrs)
    arr = _PTR_ARRAYS.get(key)
    if arr is None:
        if len(_PTR_ARRAYS) > 256:
            _PTR_ARRAYS.clear()
        arr = _PTR_ARRAYS.setdefault(key, (ctypes.c_void_p * len(ptrs))(*ptrs))
    return arr


class RmspropWorkspace(Workspace):
    """Device workspace of vtrace_rmsprop_step: allocated once, initialised once."""

    def __init__(self, n: int, device=None):  # noqa: D107 (same layout rules as Workspace)
        nbytes = int(load_library().vtrace_rmsprop_workspace_bytes(int(n)))
        if nbytes == 0:
            raise ValueError("bad size for the rmsprop workspace")
        self.device = torch.device(device if device is not None else "cuda")
        self.nbytes = nbytes
        self.buf = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
        off = (-self.buf.data_ptr()) % 256
        self.tensor = self.buf[off:off + nbytes]
        _check(load_library().vtrace_workspace_init(_ptr(self.tensor), nbytes,
                                                   _stream(self.device)),
               "vtrace_workspace_init")


def rmsprop_step(params, mean_square, grads, learning_rate: float, decay: float,
                 epsilon: float, max_global_norm: float = 40.0, global_norm_out=None,
                 workspace: RmspropWorkspace | None = None, learner_flags=None,
                 self_index: int = 0):
    """Clipped RMSProp step (momentum 0) in place on fp32 CUDA tensors of equal size
    (DESIGN.md r9-r11).  `grads`: one fp32 CUDA tensor, or a list
    of up to 8 gradients -- fp32 CUDA tensors or raw device pointers (ints; e.g. the
    learners' symmetric-memory buffers, peers included) -- summed in list order inside
    the kernel (vtrace_rmsprop_step_multi).  `global_norm_out`: optional float64 CUDA
    tensor of 1 element receiving ||sum of grads||_2 before clipping.  `learner_flags`:
    with a list of learners' buffers, one device pointer per learner to its two
    {ready, done} uint32 words -- the learners then synchronise inside the kernel
    (vtrace_rmsprop_step_learners; `self_index` = this learner's position)."""
    for t in (params, mean_square):
        if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
            raise ValueError("params and mean_square must be contiguous fp32 CUDA tensors")
    n = params.numel()
    multi = isinstance(grads, (list, tuple))
    glist = list(grads) if multi else [grads]
    if not 1 <= len(glist) <= 8:
        raise ValueError("between 1 and 8 gradients")
    ptrs = []
    for g in glist:
        if isinstance(g, int):
            ptrs.append(g)
            continue
        if not (g.is_cuda and g.dtype == torch.float32 and g.is_contiguous()):
            raise ValueError("gradients must be contiguous fp32 CUDA tensors (or device pointers)")
        if g.numel() != n:
            raise ValueError("params, mean_square and grads must have the same size")
        ptrs.append(g.data_ptr())
    if mean_square.numel() != n:
        raise ValueError("params, mean_square and grads must have the same size")
    if global_norm_out is not None and not (global_norm_out.is_cuda and
                                            global_norm_out.dtype == torch.float64):
        raise ValueError("global_norm_out must be a float64 CUDA tensor")
    if learner_flags is not None and workspace is None:
        # the in-kernel learner sync counts calls in the workspace: a fresh one per call
        # would restart the count and let learners read peers' buffers early
        raise ValueError("learner_flags needs a persistent RmspropWorkspace (one per learner, "
                         "reused every step)")
    ws = workspace if workspace is not None else RmspropWorkspace(n, params.device)
    key = (float(learning_rate), float(decay), float(epsilon), float(max_global_norm))
    prm = _RMS_PRM_CACHE.get(key)
    if prm is None:  # (argument marshalling is cached: a learner calls this every step)
        prm = _RMS_PRM_CACHE.setdefault(key, _RmsParams(*key))
    lib = load_library()
    if not multi:
        st = lib.vtrace_rmsprop_step(n, _ptr(params), _ptr(mean_square), ctypes.c_void_p(ptrs[0]),
                                     ctypes.byref(prm), _ptr(global_norm_out), ws.ptr, ws.nbytes,
                                     _stream(params.device))
        _check(st, "vtrace_rmsprop_step")
        return
    arr = _ptr_array(ptrs)
    if learner_flags is not None:
        if len(learner_flags) != len(ptrs):
            raise ValueError("one flag pointer per learner buffer")
        fl = _ptr_array([int(f) for f in learner_flags])
        st = lib.vtrace_rmsprop_step_learners(n, _ptr(params), _ptr(mean_square), arr, fl,
                                              len(ptrs), int(self_index), ctypes.byref(prm),
                                              _ptr(global_norm_out), ws.ptr, ws.nbytes,
                                              _stream(params.device))
        _check(st, "vtrace_rmsprop_step_learners")
        return
    st = lib.vtrace_rmsprop_step_multi(n, _ptr(params), _ptr(mean_square), arr, len(ptrs),
                                       ctypes.byref(prm), _ptr(global_norm_out), ws.ptr,
                                       ws.nbytes, _stream(params.device))
    _check(st, "vtrace_rmsprop_step_multi")


def rmsprop_norm_mailbox_bytes(num_learners: int) -> int:
    return int(load_library().vtrace_rmsprop_norm_mailbox_bytes(int(num_learners)))


def rmsprop_step_sharded(params_ptrs, mean_square, grads_ptrs, learning_rate: float,
                         decay: float, epsilon: float, max_global_norm: float, *, flags,
                         norm_mailboxes, self_index: int, n: int, workspace: RmspropWorkspace,
                         global_norm_out=None):
    """vtrace_rmsprop_step_sharded: the learners' update sharded over the learners (each
    updates 1/N of the parameters from the summed gradients and writes the new values into
    every learner's params).  ``params_ptrs``, ``grads_ptrs``, ``flags``, ``norm_mailboxes``:
    one device pointer per learner (peer-mapped); ``mean_square`` this learner's fp32
    tensor of n elements.  Marshalling only."""
    if not (mean_square.is_cuda and mean_square.dtype == torch.float32 and
            mean_square.is_contiguous() and mean_square.numel() == n):
        raise ValueError("mean_square must be a contiguous fp32 CUDA tensor of n elements")
    N = len(params_ptrs)
    if not (len(grads_ptrs) == len(flags) == len(norm_mailboxes) == N):
        raise ValueError("one params / grads / flags / mailbox pointer per learner")
    key = (float(learning_rate), float(decay), float(epsilon), float(max_global_norm))
    prm = _RMS_PRM_CACHE.get(key)
    if prm is None:
        prm = _RMS_PRM_CACHE.setdefault(key, _RmsParams(*key))
    st = load_library().vtrace_rmsprop_step_sharded(
        int(n), _ptr_array([int(p) for p in params_ptrs]), _ptr(mean_square),
        _ptr_array([int(p) for p in grads_ptrs]), _ptr_array([int(p) for p in flags]),
        _ptr_array([int(p) for p in norm_mailboxes]), N, int(self_index), ctypes.byref(prm),
        _ptr(global_norm_out), workspace.ptr, workspace.nbytes, _stream(mean_square.device))
    _check(st, "vtrace_rmsprop_step_sharded")


def grad_push(grad: torch.Tensor, recv_ptrs, self_index: int):
    """vtrace_grad_push: this learner's fp32 gradient into slot ``self_index`` of every
    learner's receive buffer (``recv_ptrs``: one device pointer per learner, each buffer
    num_learners * n floats).  Marshalling only."""
    if not (grad.is_cuda and grad.dtype == torch.float32 and grad.is_contiguous()):
        raise ValueError("grad must be a contiguous fp32 CUDA tensor")
    st = load_library().vtrace_grad_push(_ptr(grad), _ptr_array([int(p) for p in recv_ptrs]),
                                         len(recv_ptrs), int(self_index), grad.numel(),
                                         _stream(grad.device))
    _check(st, "vtrace_grad_push")


def output_layer(hidden: torch.Tensor, w_t: torch.Tensor, bias: torch.Tensor | None = None,
                 logits_out: torch.Tensor | None = None, values_out: torch.Tensor | None = None):
    """NEXT #3 (reading r12): ``[z^pi | V] = h W + b`` on the tensor cores.
    ``hidden`` [T, B, H] (or [M, H]) bf16, ``w_t`` = W^T [A+1, H] bf16, ``bias`` [A+1] fp32
    or None.  Returns (logits [.., A] fp32, values [..] fp32) -- the layouts
    :func:`loss_and_grad` reads.  Marshalling only: vtrace_output_layer does the work."""
    if hidden.dtype != torch.bfloat16 or w_t.dtype != torch.bfloat16:
        raise TypeError("output_layer: hidden and w_t must be bfloat16")
    lead = tuple(hidden.shape[:-1])
    H = int(hidden.shape[-1])
    A = int(w_t.shape[0]) - 1
    if w_t.dim() != 2 or int(w_t.shape[1]) != H:
        raise ValueError("output_layer: w_t must be [A+1, H]")
    M = 1
    for d in lead:
        M *= int(d)
    _contig(hidden, w_t)
    dev = hidden.device
    if w_t.device != dev:
        raise ValueError("output_layer: hidden and w_t must be on the same device")
    if bias is not None:
        if bias.numel() != A + 1:
            raise ValueError(f"output_layer: bias must have A + 1 = {A + 1} elements "
                             "(policy logits then the baseline)")
        bias = bias.to(device=dev, dtype=torch.float32).contiguous()
    if logits_out is None:
        logits_out = torch.empty(lead + (A,), dtype=torch.float32, device=dev)
    elif not (logits_out.dtype == torch.float32 and logits_out.is_contiguous() and
              logits_out.numel() == M * A and logits_out.device == dev):
        raise ValueError("output_layer: logits_out must be a contiguous fp32 tensor of M * A "
                         "elements on hidden's device")
    if values_out is None:
        values_out = torch.empty(lead, dtype=torch.float32, device=dev)
    elif not (values_out.dtype == torch.float32 and values_out.is_contiguous() and
              values_out.numel() == M and values_out.device == dev):
        raise ValueError("output_layer: values_out must be a contiguous fp32 tensor of M "
                         "elements on hidden's device")
    st = load_library().vtrace_output_layer(M, H, A, _ptr(hidden), _ptr(w_t), _ptr(bias),
                                            _ptr(logits_out), _ptr(values_out), _stream(dev))
    _check(st, "vtrace_output_layer")
    return logits_out, values_out


# ---- a13 over NVLink peer memory (include/vtrace.h vtrace_partials_allreduce) ----

def partials_mailbox_bytes(num_learners: int) -> int:
    """Bytes of one learner's mailbox for vtrace_partials_allreduce (0: out of range)."""
    return int(load_library().vtrace_partials_mailbox_bytes(int(num_learners)))


def partials_allreduce(partials: torch.Tensor, mailbox_ptrs, self_index: int,
                       counter: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Sum of the learners' [8] fp64 partials over NVLink peer memory (row a13):
    ``mailbox_ptrs`` are the learners' mailbox device pointers (zero-initialised once,
    peer-mapped, e.g. symmetric memory), ``counter`` this learner's int64 call counter
    (zero-initialised once).  Every learner makes the same sequence of calls; the sums
    are bitwise identical.  Marshalling only: the kernel does the exchange."""
    if partials.dtype != torch.float64 or partials.numel() != 8 or not partials.is_contiguous():
        raise ValueError("partials_allreduce: partials must be a contiguous float64 tensor of 8")
    if counter.dtype != torch.int64 or counter.numel() != 1 or counter.device != partials.device:
        raise ValueError("partials_allreduce: counter must be one int64 on partials' device")
    if out is None:
        out = partials
    elif out.dtype != torch.float64 or out.numel() != 8 or not out.is_contiguous() or \
            out.device != partials.device:
        raise ValueError("partials_allreduce: out must be a contiguous float64 tensor of 8")
    ptrs = [int(p) for p in mailbox_ptrs]
    arr = _ptr_array(ptrs)
    st = load_library().vtrace_partials_allreduce(_ptr(partials), arr, len(ptrs), int(self_index),
                                                  _ptr(counter), _ptr(out),
                                                  _stream(partials.device))
    _check(st, "vtrace_partials_allreduce")
    return out


# ---- NEXT #3 second half: the head fused with the path and its backward ----

class HeadWorkspace:
    """Device workspace of vtrace_head_loss_and_grad (a grid-barrier word pair and the
    per-CTA partials): zero-initialised once here, left ready by every call."""

    def __init__(self, T: int, B: int, H: int, A: int, device=None):
        self.nbytes = int(load_library().vtrace_head_workspace_bytes(T, B, H, A))
        if self.nbytes == 0:
            raise ValueError("head workspace: bad shape")
        dev = torch.device(device) if device is not None else torch.device("cuda")
        self.buf = torch.zeros(self.nbytes + 256, dtype=torch.uint8, device=dev)
        off = (-self.buf.data_ptr()) % 256
        self.ptr = ctypes.c_void_p(self.buf.data_ptr() + off)


def head_loss_and_grad(hidden, w_t, bias, behaviour_logits, actions, discounts, rewards,
                       bootstrap_value, *, rho_bar=1.0, c_bar=1.0, pg_rho_bar=None,
                       lambda_=1.0, reward_mode=0, correction=CORRECTION_VTRACE,
                       epsilon=1e-6, q_from_values=0, baseline_cost=0.5, entropy_cost=0.01,
                       workspace: HeadWorkspace | None = None, out: dict | None = None):
    """vtrace_head_loss_and_grad (NEXT #3, P:173-174 + Section 4): the output layer
    ``[z^pi | V] = h W + b`` with the V-trace loss and gradients as its epilogue and the
    head's backward.  hidden [T,B,H] bf16, w_t = W^T [A+1,H] bf16, bias [A+1] fp32 or None,
    behaviour_logits [T,B,A] fp32, actions/discounts/rewards [T,B], bootstrap_value [B].
    Returns dict grad_hidden [T,B,H] bf16, grad_w_t [A+1,H] fp32, grad_bias [A+1] fp32,
    partials [8] fp64.  Marshalling only: the two kernels do the work."""
    lib = load_library()
    if hidden.dtype != torch.bfloat16 or w_t.dtype != torch.bfloat16:
        raise TypeError("head_loss_and_grad: hidden and w_t must be bfloat16")
    if hidden.dim() != 3 or w_t.dim() != 2:
        raise ValueError("head_loss_and_grad: hidden [T,B,H], w_t [A+1,H]")
    T, B, H = (int(x) for x in hidden.shape)
    A = int(w_t.shape[0]) - 1
    dev = hidden.device
    if int(w_t.shape[1]) != H:
        raise ValueError("head_loss_and_grad: w_t must be [A+1, H]")
    want = {"behaviour_logits": (behaviour_logits, (T, B, A), torch.float32),
            "actions": (actions, (T, B), torch.int32), "discounts": (discounts, (T, B), torch.float32),
            "rewards": (rewards, (T, B), torch.float32),
            "bootstrap_value": (bootstrap_value, (B,), torch.float32)}
    for name, (t, shp, dt) in want.items():
        if tuple(t.shape) != shp or t.dtype != dt or t.device != dev:
            raise ValueError(f"head_loss_and_grad: {name} must be {dt} {shp} on {dev}")
    _contig(hidden, w_t, behaviour_logits, actions, discounts, rewards, bootstrap_value)
    if bias is not None:
        if bias.numel() != A + 1:
            raise ValueError(f"head_loss_and_grad: bias must have A + 1 = {A + 1} elements")
        bias = bias.to(device=dev, dtype=torch.float32).contiguous()
    ws = workspace if workspace is not None else HeadWorkspace(T, B, H, A, dev)
    if out is None:
        out = {"grad_hidden": torch.empty_like(hidden),
               "grad_w_t": torch.empty(A + 1, H, dtype=torch.float32, device=dev),
               "grad_bias": torch.empty(A + 1, dtype=torch.float32, device=dev),
               "partials": torch.empty(P_COUNT, dtype=torch.float64, device=dev)}
    else:
        _check_out(out, {"grad_hidden": ((T, B, H), torch.bfloat16, True),
                         "grad_w_t": ((A + 1, H), torch.float32, True),
                         "grad_bias": ((A + 1,), torch.float32, True),
                         "partials": ((P_COUNT,), torch.float64, True)}, dev)
    p = params(rho_bar, c_bar, pg_rho_bar, lambda_, reward_mode, correction, epsilon,
               q_from_values, 0, 0)
    w = _Weights(float(baseline_cost), float(entropy_cost))
    st = lib.vtrace_head_loss_and_grad(
        T, B, H, A, _ptr(hidden), _ptr(w_t), _ptr(bias), _ptr(behaviour_logits), _ptr(actions),
        _ptr(discounts), _ptr(rewards), _ptr(bootstrap_value), ctypes.byref(p), ctypes.byref(w),
        _ptr(out["grad_hidden"]), _ptr(out["grad_w_t"]), _ptr(out["grad_bias"]),
        _ptr(out["partials"]), ws.ptr, ws.nbytes, _stream(dev))
    _check(st, "vtrace_head_loss_and_grad")
    return out


def partials_mailbox_bytes_batched(num_learners: int, batch: int) -> int:
    return int(load_library().vtrace_partials_mailbox_bytes_batched(int(num_learners), int(batch)))


def partials_allreduce_batched(partials_list, mailbox_ptrs, self_index: int,
                               counter: torch.Tensor, batch_max: int = 32):
    """Sum over the learners of several steps' [8] fp64 partials, in place, one kernel
    (vtrace_partials_allreduce_batched).  Marshalling only."""
    if not 1 <= len(partials_list) <= 32:
        raise ValueError("partials_allreduce_batched: 1..32 partials tensors")
    dev = partials_list[0].device
    for t in partials_list:
        if t.dtype != torch.float64 or t.numel() != 8 or not t.is_contiguous() or t.device != dev:
            raise ValueError("partials_allreduce_batched: contiguous float64 tensors of 8")
    if counter.dtype != torch.int64 or counter.numel() != 1 or counter.device != dev:
        raise ValueError("partials_allreduce_batched: counter must be one int64 on the device")
    pa = _ptr_array([t.data_ptr() for t in partials_list])
    mb = _ptr_array([int(p) for p in mailbox_ptrs])
    st = load_library().vtrace_partials_allreduce_batched(pa, len(partials_list), int(batch_max), mb,
                                                          len(mailbox_ptrs), int(self_index),
                                                          _ptr(counter), _stream(dev))
    _check(st, "vtrace_partials_allreduce_batched")
