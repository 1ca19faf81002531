"""Seeded synthetic trajectory batches shaped like the paper's learner inputs.

This module is the ONE piece shared by the oracle tests and the CUDA path: it
draws inputs and holds none of the method's arithmetic (no softmax, no
importance weights, no targets, no reward transform).  Everything is drawn on
the CPU with a seeded ``torch.Generator`` so any process (test, bench rank,
oracle leg) reproduces identical bits.

Recipe:
  * target logits  z_pi ~ N(0, 1.5^2) iid per element,
  * behaviour logits z_mu = z_pi + N(0, 0.3^2)  (policy lag, P:152 / P:158),
    both rounded to the config's logits dtype (bf16: round-to-nearest-even),
  * actions sampled from mu = softmax(z_mu) by the Gumbel-max trick
    a = argmax_j (z_mu_j + G_j), G_j = -log(-log U_j)   (actors act with mu),
  * values V(x_t) and bootstrap V(x_T) ~ N(0, 1),
  * raw rewards: 0 w.p. 0.9, else +1 / +10 / -1 w.p. 0.6 / 0.2 / 0.2
    (the config's reward_mode transform is applied by the method, not here),
  * discounts = 0.99 * (1 - done), done ~ Bernoulli(p_done).
"""
from __future__ import annotations

import dataclasses

import numpy as np
import torch

DTYPE_F32 = 0
DTYPE_BF16 = 1
REWARD_NONE = 0
REWARD_CLIP_UNIT = 1
REWARD_ASYM_TANH = 2


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    T: int
    B: int
    A: int
    dtype: int
    reward_mode: int
    p_done: float
    index: int          # position in BASELINE.json "configs"; seed = 1802 + index
    paper: str          # where the shape comes from

    @property
    def seed(self) -> int:
        return 1802 + self.index


CONFIGS = {
    "toy": Config("toy", 5, 2, 3, DTYPE_F32, REWARD_NONE, 0.0, 0,
                  "hand-built worked example (SURVEY 8(c)); gamma=0.99 (P:836)"),
    "atari": Config("atari", 20, 32, 18, DTYPE_F32, REWARD_CLIP_UNIT, 0.05, 1,
                    "n=20 (P:945), batch 32 (P:946), 18 actions (P:926), clip[-1,1] (P:944)"),
    "dmlab": Config("dmlab", 100, 32, 9, DTYPE_BF16, REWARD_ASYM_TANH, 0.001, 2,
                    "n=100 (P:832), batch 32 (P:326), 9 actions (P:796-811), asym clip (P:819)"),
    "large": Config("large", 100, 8192, 18, DTYPE_BF16, REWARD_CLIP_UNIT, 0.01, 3,
                    "n=100 (P:832), 18 actions (P:926), batch beyond the paper's 128 (P:320)"),
    "stress": Config("stress", 2000, 1024, 9, DTYPE_F32, REWARD_ASYM_TANH, 0.001, 4,
                     "long unroll exercising the affine scan; asym clip (P:819)"),
}

GAMMA = 0.99
BASELINE_COST = 0.5
ENTROPY_COST = 0.01
RHO_BAR = 1.0
C_BAR = 1.0


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round fp32 to bf16 (nearest-even) and return the raw uint16 bits."""
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16)
    return t.view(torch.int16).numpy().view(np.uint16).copy()


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    """Exact decode of bf16 bit patterns (for sampling only)."""
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def toy_inputs() -> dict:
    """The hand-built T=5 B=2 A=3 example of SURVEY.md section 8(c) (config 1),
    with exactly one terminal step at (t=2, b=0)."""
    zp = np.array([[[1, 0, -1], [0, 1, 2]], [[0, 0, 0], [1, 1, 0]], [[2, 1, 0], [0, -1, 0]],
                   [[0, 1, 0], [3, 0, 0]], [[-1, 0, 1], [0, 0, 0]]], np.float32)
    zm = np.array([[[0, 0, 0], [0, 1, 2]], [[1, 0, -1], [0, 0, 0]], [[2, 1, 0], [1, 0, 0]],
                   [[0, 0, 1], [0, 0, 3]], [[0, 0, 0], [0, 0, 1]]], np.float32)
    a = np.array([[0, 2], [2, 0], [1, 1], [1, 0], [2, 1]], np.int32)
    r = np.array([[0, 1], [1, 0], [0, 0], [-1, 0], [1, 1]], np.float32)
    V = np.array([[.5, 1], [.25, .5], [-.5, -.25], [1, .75], [0, .125]], np.float32)
    boot = np.array([2.0, -1.0], np.float32)
    g = np.full((5, 2), GAMMA, np.float32)
    g[2, 0] = 0.0
    return dict(T=5, B=2, A=3, dtype=DTYPE_F32, reward_mode=REWARD_NONE,
                target_logits=zp, behaviour_logits=zm, actions=a, rewards=r, values=V,
                bootstrap_value=boot, discounts=g)


def make_inputs(config, seed: int | None = None, B: int | None = None, T: int | None = None,
                A: int | None = None, dtype: int | None = None, spread: float = 1.5,
                lag: float = 0.3, p_done: float | None = None) -> dict:
    """Seeded synthetic batch for ``config`` (a name or a Config).

    Returns a dict of numpy arrays in the library's layout: logits [T,B,A]
    (float32, or uint16 bf16 bits), actions int32 [T,B], rewards / values /
    discounts float32 [T,B], bootstrap_value float32 [B]; plus T, B, A, dtype,
    reward_mode.  Shape overrides keep the config's distributions; ``spread`` / ``lag``
    (std of z_pi and of z_mu - z_pi) and ``p_done`` override them for stress tests
    (p_done = 0: no episode end at all)."""
    cfg = CONFIGS[config] if isinstance(config, str) else config
    T = cfg.T if T is None else T
    B = cfg.B if B is None else B
    A = cfg.A if A is None else A
    dtype = cfg.dtype if dtype is None else dtype
    seed = cfg.seed if seed is None else seed
    g = torch.Generator().manual_seed(int(seed))
    zp = torch.randn(T, B, A, generator=g) * spread
    zm = zp + torch.randn(T, B, A, generator=g) * lag
    if dtype == DTYPE_BF16:
        zp_s = f32_to_bf16_bits(zp.numpy())
        zm_s = f32_to_bf16_bits(zm.numpy())
        zm_val = torch.from_numpy(bf16_bits_to_f32(zm_s))
    else:
        zp_s = zp.numpy().astype(np.float32)
        zm_s = zm.numpy().astype(np.float32)
        zm_val = torch.from_numpy(zm_s)
    u = torch.rand(T, B, A, generator=g).clamp_(min=1e-12)
    gumbel = -torch.log(-torch.log(u))
    actions = torch.argmax(zm_val + gumbel, dim=-1).to(torch.int32)
    V = torch.randn(T, B, generator=g)
    boot = torch.randn(B, generator=g)
    ur = torch.rand(T, B, generator=g)
    rew = torch.zeros(T, B)
    rew = torch.where(ur >= 0.90, torch.full_like(rew, 1.0), rew)
    rew = torch.where(ur >= 0.96, torch.full_like(rew, 10.0), rew)
    rew = torch.where(ur >= 0.98, torch.full_like(rew, -1.0), rew)
    pd = cfg.p_done if p_done is None else p_done
    done = torch.rand(T, B, generator=g) < pd
    if pd > 0 and not bool(done.any()):
        done[T // 2, 0] = True     # at least one episode end in the batch
    disc = torch.where(done, torch.zeros(T, B), torch.full((T, B), GAMMA))
    return dict(T=T, B=B, A=A, dtype=dtype, reward_mode=cfg.reward_mode,
                target_logits=zp_s, behaviour_logits=zm_s,
                actions=actions.numpy().astype(np.int32),
                rewards=rew.numpy().astype(np.float32), values=V.numpy().astype(np.float32),
                bootstrap_value=boot.numpy().astype(np.float32),
                discounts=disc.numpy().astype(np.float32))


def inputs_for(name: str, seed: int | None = None, **kw) -> dict:
    """``toy`` -> the hand-built example; other names -> make_inputs."""
    if name == "toy" and seed is None and not kw:
        return toy_inputs()
    return make_inputs(name, seed=seed, **kw)


def column_slice(inp: dict, b0: int, b1: int) -> dict:
    """Columns [b0, b1) of a batch (a learner's shard), as contiguous arrays."""
    out = dict(inp)
    out["B"] = b1 - b0
    for k in ("target_logits", "behaviour_logits"):
        out[k] = np.ascontiguousarray(inp[k][:, b0:b1])
    for k in ("actions", "rewards", "values", "discounts", "behaviour_log_probs"):
        if inp.get(k) is not None:
            out[k] = np.ascontiguousarray(inp[k][:, b0:b1])
    out["bootstrap_value"] = np.ascontiguousarray(inp["bootstrap_value"][b0:b1])
    return out


# ---- inputs of the learner's parameter update -------------
# The paper's networks have 1.2 M (shallow) and 1.6 M (deep) parameters;
# there is no network here, so the gradient is synthetic: per-parameter N(0, s^2)
# with s chosen so the global norm is `norm` (default 80: above the clip of 40,
# P:953), parameters N(0, 0.05^2), mean squares U(0.5, 1.5) (a run in progress).
UPDATE_SIZES = {"shallow": 1_200_000, "deep": 1_600_000}


def update_inputs(n: int, seed: int = 0, norm: float = 80.0, learners: int = 1) -> dict:
    """fp32 numpy params [n], mean_square [n] and one gradient [n] per learner
    (their sum has global norm ~`norm`)."""
    rng = np.random.default_rng(seed)
    params = rng.normal(0.0, 0.05, size=n).astype(np.float32)
    ms = rng.uniform(0.5, 1.5, size=n).astype(np.float32)
    s = norm / np.sqrt(max(n, 1) * learners)
    grads = [rng.normal(0.0, s, size=n).astype(np.float32) for _ in range(learners)]
    return {"n": n, "params": params, "mean_square": ms, "grads": grads}
