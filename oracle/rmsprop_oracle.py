"""CPU oracle of the learner's parameter update.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may use it.  Plain numpy,
fp64 throughout, no blocking or reordering beyond the definitions below.

What the paper fixes:
  * the optimiser is RMSProp with momentum 0 and a regularisation epsilon
    (epsilon swept over {1e-1, 1e-3, 1e-5, 1e-7});
  * the global gradient norm is clipped at 40;
  * the loss is summed over batch and time, and the learners update
    synchronously, so the gradient of the whole batch is the SUM of
    the learners' gradients (reading r11).
What it does not fix, and the readings taken (DESIGN.md r9, r10):
  * the RMSProp formula: the TensorFlow form (the paper's implementation is TF,
    P:178), with epsilon inside the square root:
        ms    <- decay * ms + (1 - decay) * g^2
        theta <- theta - lr * g / sqrt(ms + epsilon)
    `decay` is a parameter (not given by the paper) and the mean-square state
    `ms` is owned and initialised by the caller;
  * the clip: g <- g * c / max(||g||_2, c) over ALL parameters (the global norm
    of the concatenated gradient), i.e. unchanged when ||g||_2 <= c.

Pins (tests/test_oracle_pins.py): a 3-4-5 norm, exact power-of-two clip scales,
the closed form of the mean square under a constant gradient, the fixed point
ms = g^2, the zero-gradient step, scale invariance of a clipped update.
"""
from __future__ import annotations

import numpy as np


def global_norm(grads) -> float:
    """||g||_2 over every parameter, fp64 ("global gradient norm")."""
    g = np.asarray(grads, dtype=np.float64).ravel()
    return float(np.sqrt(np.sum(g * g)))


def clip_by_global_norm(grads, max_norm: float):
    """g * c / max(||g||, c) (reading r10); max_norm <= 0 disables the clip.
    Returns (clipped fp64 gradient, the norm before clipping)."""
    g = np.asarray(grads, dtype=np.float64).ravel()
    norm = global_norm(g)
    if max_norm > 0 and norm > max_norm:
        g = g * (max_norm / norm)
    return g, norm


def rmsprop_step(params, mean_square, grads, learning_rate: float, decay: float,
                 epsilon: float, max_global_norm: float):
    """One synchronous update (momentum 0): clip, then RMSProp
    (reading r9).  Returns (new params, new mean square, global norm),
    all fp64."""
    theta = np.asarray(params, dtype=np.float64).ravel()
    ms = np.asarray(mean_square, dtype=np.float64).ravel()
    g, norm = clip_by_global_norm(grads, max_global_norm)
    ms_new = decay * ms + (1.0 - decay) * g * g
    theta_new = theta - learning_rate * g / np.sqrt(ms_new + epsilon)
    return theta_new, ms_new, norm


def sum_learner_grads(grads_per_learner):
    """The whole batch's gradient from the learners' shard gradients: their sum
    (the loss is a sum over the batch; reading r11)."""
    out = None
    for g in grads_per_learner:
        g = np.asarray(g, dtype=np.float64)
        out = g.copy() if out is None else out + g
    return out
