"""CPU oracle for the IMPALA V-trace learner hot path (arxiv 1802.01561, Section 4).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_1802_01561_b200`` never imports it and
shares no code with it.

This module is argument marshalling (numpy <-> ctypes) around ``liboracle.so``
(``vtrace_oracle.cpp``: plain fp64 loops).  See ``vtrace_oracle.h`` for what each
function computes and the paper passages it follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "vtrace_oracle.cpp")

DTYPE_F32 = 0
DTYPE_BF16 = 1

REWARD_NONE = 0
REWARD_CLIP_UNIT = 1
REWARD_ASYM_TANH = 2

DATA_ERRORS = {1: "action", 2: "logits", 3: "reward", 4: "value", 5: "discount"}


def build(force: bool = False) -> str:
    """Compile liboracle.so with g++ (plain -O2, no fast-math)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "vtrace_oracle.h"))
    ):
        subprocess.check_call(
            ["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-fno-fast-math",
             "-ffp-contract=off", "-o", _SO, _SRC]
        )
    return _SO


class _Params(ctypes.Structure):
    _fields_ = [("rho_bar", ctypes.c_double), ("c_bar", ctypes.c_double),
                ("pg_rho_bar", ctypes.c_double), ("lambda_", ctypes.c_double),
                ("reward_mode", ctypes.c_int32), ("correction", ctypes.c_int32),
                ("epsilon", ctypes.c_double), ("q_from_values", ctypes.c_int32),
                ("behaviour_log_probs", ctypes.c_int32)]


# Section 5.2.2 off-policy correction variants
CORR_VTRACE, CORR_NONE, CORR_EPSILON, CORR_ONE_STEP_IS = 0, 1, 2, 3


class _Weights(ctypes.Structure):
    _fields_ = [("baseline_cost", ctypes.c_double), ("entropy_cost", ctypes.c_double)]


_lib = None


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        _lib.vtrace_oracle_from_logits.argtypes = [i64, i64, i64, ctypes.c_int32] + [P] * 7 + [
            ctypes.POINTER(_Params)] + [P] * 5 + [ctypes.POINTER(i64)]
        _lib.vtrace_oracle_loss_and_grad.argtypes = [i64, i64, i64, ctypes.c_int32] + [P] * 7 + [
            ctypes.POINTER(_Params), ctypes.POINTER(_Weights)] + [P] * 5 + [ctypes.POINTER(i64)]
        _lib.vtrace_oracle_vs_eq1.argtypes = [i64, i64] + [P] * 5 + [ctypes.POINTER(_Params), P]
        _lib.vtrace_oracle_vs_recursion.argtypes = [i64, i64] + [P] * 5 + [
            ctypes.POINTER(_Params), P, P]
        _lib.vtrace_oracle_reward_transform.argtypes = [ctypes.c_double, ctypes.c_int32]
        _lib.vtrace_oracle_reward_transform.restype = ctypes.c_double
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code, bad_index=-1):
        self.code = code
        self.bad_index = bad_index
        super().__init__(f"oracle status {code} (bad index {bad_index})")


def _params(rho_bar=1.0, c_bar=1.0, pg_rho_bar=None, lambda_=1.0, reward_mode=REWARD_NONE,
            correction=CORR_VTRACE, epsilon=1e-6, q_from_values=0, behaviour_log_probs=0):
    return _Params(float(rho_bar), float(c_bar),
                   float(rho_bar if pg_rho_bar is None else pg_rho_bar), float(lambda_),
                   int(reward_mode), int(correction), float(epsilon), int(q_from_values),
                   int(behaviour_log_probs))


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _logits_array(x, dtype):
    """fp32 logits -> float32 array; bf16 logits -> uint16 raw bits."""
    if dtype == DTYPE_F32:
        return np.ascontiguousarray(x, dtype=np.float32)
    x = np.ascontiguousarray(x)
    if x.dtype != np.uint16:
        raise TypeError("bf16 logits must be passed as uint16 bit patterns")
    return x


def _inputs(inp):
    """The seven input arrays.  With inp["behaviour_log_probs"] (a [T, B] array of
    log mu(a_t)), that array replaces the behaviour logits (behaviour_log_probs=1)."""
    T, B, A = inp["T"], inp["B"], inp["A"]
    dt = inp["dtype"]
    if inp.get("behaviour_log_probs") is not None:
        mu = np.ascontiguousarray(inp["behaviour_log_probs"], dtype=np.float32)
        assert mu.size == T * B
    else:
        mu = _logits_array(inp["behaviour_logits"], dt)
    pi = _logits_array(inp["target_logits"], dt)
    a = np.ascontiguousarray(inp["actions"], dtype=np.int32)
    g = np.ascontiguousarray(inp["discounts"], dtype=np.float32)
    r = np.ascontiguousarray(inp["rewards"], dtype=np.float32)
    V = np.ascontiguousarray(inp["values"], dtype=np.float32)
    boot = np.ascontiguousarray(inp["bootstrap_value"], dtype=np.float32)
    assert pi.size == T * B * A and a.size == T * B
    assert boot.size == B
    return T, B, A, dt, (mu, pi, a, g, r, V, boot)


def _mu_mode(inp, params):
    if inp.get("behaviour_log_probs") is not None:
        return dict(params, behaviour_log_probs=1)
    return params


def from_logits(inp, check=True, **params):
    """V-trace targets from logits.  ``inp``: dict with T, B, A, dtype and the
    seven input arrays (see paper_1802_01561_b200.workload).  Returns a dict of
    float64 [T, B] arrays: vs, pg_advantages, log_rhos, target_action_log_probs,
    behaviour_action_log_probs; plus status and bad_index."""
    lib = _load()
    T, B, A, dt, arrs = _inputs(inp)
    out = {k: np.zeros((T, B), np.float64) for k in
           ("vs", "pg_advantages", "log_rhos", "target_action_log_probs",
            "behaviour_action_log_probs")}
    bad = ctypes.c_int64(-1)
    p = _params(**_mu_mode(inp, params))
    st = lib.vtrace_oracle_from_logits(
        T, B, A, dt, *[_ptr(x) for x in arrs], ctypes.byref(p),
        _ptr(out["vs"]), _ptr(out["pg_advantages"]), _ptr(out["log_rhos"]),
        _ptr(out["target_action_log_probs"]), _ptr(out["behaviour_action_log_probs"]),
        ctypes.byref(bad))
    if check and st != 0:
        raise OracleError(st, bad.value)
    out["status"] = st
    out["bad_index"] = bad.value
    return out


def loss_and_grad(inp, baseline_cost=0.5, entropy_cost=0.01, check=True, **params):
    """Summed losses and gradients.  Returns dict with grad_target_logits
    [T,B,A] f64, grad_values [T,B] f64, partials [8] f64, vs, pg_advantages."""
    lib = _load()
    T, B, A, dt, arrs = _inputs(inp)
    gz = np.zeros((T, B, A), np.float64)
    gv = np.zeros((T, B), np.float64)
    parts = np.zeros(8, np.float64)
    vs = np.zeros((T, B), np.float64)
    adv = np.zeros((T, B), np.float64)
    bad = ctypes.c_int64(-1)
    p = _params(**_mu_mode(inp, params))
    w = _Weights(float(baseline_cost), float(entropy_cost))
    st = lib.vtrace_oracle_loss_and_grad(
        T, B, A, dt, *[_ptr(x) for x in arrs], ctypes.byref(p), ctypes.byref(w),
        _ptr(gz), _ptr(gv), _ptr(parts), _ptr(vs), _ptr(adv), ctypes.byref(bad))
    if check and st != 0:
        raise OracleError(st, bad.value)
    return {"grad_target_logits": gz, "grad_values": gv, "partials": parts, "vs": vs,
            "pg_advantages": adv, "status": st, "bad_index": bad.value}


def _f64(x):
    return np.ascontiguousarray(x, dtype=np.float64)


def vs_eq1(log_rhos, discounts, rewards, values, bootstrap, **params):
    """Eq.(1) explicit double sum from log ratios; [T,B] float64."""
    lib = _load()
    lr, g, r, V, boot = map(_f64, (log_rhos, discounts, rewards, values, bootstrap))
    T, B = lr.shape
    vs = np.zeros((T, B), np.float64)
    p = _params(**params)
    st = lib.vtrace_oracle_vs_eq1(T, B, _ptr(lr), _ptr(g), _ptr(r), _ptr(V), _ptr(boot),
                                  ctypes.byref(p), _ptr(vs))
    if st:
        raise OracleError(st)
    return vs


def vs_recursion(log_rhos, discounts, rewards, values, bootstrap, **params):
    """Remark-1 recursion from log ratios; returns (vs, pg_adv)."""
    lib = _load()
    lr, g, r, V, boot = map(_f64, (log_rhos, discounts, rewards, values, bootstrap))
    T, B = lr.shape
    vs = np.zeros((T, B), np.float64)
    adv = np.zeros((T, B), np.float64)
    p = _params(**params)
    st = lib.vtrace_oracle_vs_recursion(T, B, _ptr(lr), _ptr(g), _ptr(r), _ptr(V),
                                        _ptr(boot), ctypes.byref(p), _ptr(vs), _ptr(adv))
    if st:
        raise OracleError(st)
    return vs, adv


def reward_transform(r, mode):
    return _load().vtrace_oracle_reward_transform(float(r), int(mode))
