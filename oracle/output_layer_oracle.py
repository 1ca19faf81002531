"""CPU oracle of the output layer in front of the V-trace path.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may use it.  Plain numpy,
fp64 matmuls, no blocking or reordering beyond the definitions below.

What the paper fixes:
  * the learner applies the network to all T*B steps of the batch at once, the
    time dimension folded into the batch dimension, and the LSTM output
    feeds a linear policy head and a linear baseline head (Fig. 3);
  * the loss whose gradients the path computes, summed over batch
    and time, with v_s, q_s, pg_adv and rho held constant (the
    stop-gradients of reading c10).
Readings (DESIGN.md r12):
  * one fused head: ``[z^pi | V] = h @ W + b`` with ``W`` [H, A+1] (the first A
    columns the policy logits, the last the baseline), ``h`` [T, B, H];
  * the head's outputs reach the V-trace path as fp32 (the tensor-core kernel's
    accumulator type), so the oracle rounds z and V to fp32 before
    ``oracle.loss_and_grad`` and applies the chain rule in fp64:
        dZ = [dL/dz^pi | dL/dV]   [T*B, A+1]
        dh = dZ @ W^T,  dW = h^T @ dZ,  db = sum_rows dZ.

Pins (tests/test_output_layer_oracle_pins.py): the identity head reduces to the
bare path; central differences of the paper's loss with the stop-gradient
quantities frozen, on an exact dyadic grid, for every entry of h, W and b;
linearity of dW in the batch (summed loss).
"""
from __future__ import annotations

import numpy as np

import oracle


def output_layer(h, W, b):
    """logits and baseline of every folded step.  h [T,B,H], W [H,A+1],
    b [A+1] -> (z [T,B,A] f64, V [T,B] f64)."""
    h = np.asarray(h, np.float64)
    W = np.asarray(W, np.float64)
    b = np.asarray(b, np.float64)
    T, B, H = h.shape
    Z = h.reshape(T * B, H) @ W + b
    A = W.shape[1] - 1
    return Z[:, :A].reshape(T, B, A), Z[:, A].reshape(T, B)


def loss_and_grad_from_hidden(inp, h, W, b, baseline_cost=0.5, entropy_cost=0.01, **params):
    """The V-trace loss of the head's outputs and its gradients w.r.t. h, W, b.
    ``inp``: a workload dict (fp32 logits layout) whose behaviour logits/log-probs,
    actions, discounts, rewards and bootstrap are used; its target logits and values
    are replaced by the head's.  Returns the dict of ``oracle.loss_and_grad`` plus
    grad_hidden [T,B,H], grad_W [H,A+1], grad_b [A+1] (f64), target_logits and
    values (the fp32-rounded head outputs)."""
    z, V = output_layer(h, W, b)
    T, B, H = np.shape(h)
    A = np.shape(W)[1] - 1
    assert inp["T"] == T and inp["B"] == B and inp["A"] == A
    assert inp["dtype"] == oracle.DTYPE_F32
    run = dict(inp)
    run["target_logits"] = z.astype(np.float32)
    run["values"] = V.astype(np.float32)
    out = oracle.loss_and_grad(run, baseline_cost=baseline_cost,
                               entropy_cost=entropy_cost, **params)
    dZ = np.concatenate([out["grad_target_logits"].reshape(T * B, A),
                         out["grad_values"].reshape(T * B, 1)], axis=1)
    h2 = np.asarray(h, np.float64).reshape(T * B, H)
    out["grad_hidden"] = (dZ @ np.asarray(W, np.float64).T).reshape(T, B, H)
    out["grad_W"] = h2.T @ dZ
    out["grad_b"] = dZ.sum(axis=0)
    out["target_logits"] = run["target_logits"]
    out["values"] = run["values"]
    return out
