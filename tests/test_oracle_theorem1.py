"""Statistical pin of the oracle against the paper's Theorem 1 (App. A.1;
the fixed point stated in Section 4.1): under behaviour mu, the n-step V-trace operator has
the unique fixed point V^{pi_rho_bar}, the value of the policy

    pi_rho_bar(a|x) = min(rho_bar mu(a|x), pi(a|x)) / sum_b min(rho_bar mu(b|x), pi(b|x)),

for any n (here the unroll T) when c_bar <= rho_bar.  So on a small tabular MDP, with V set
to V^{pi_rho_bar} (solved exactly by linear algebra, independently of the oracle), the
oracle's v_s over trajectories sampled from mu must equal V(x_s) in expectation: the sample
mean of v_0 - V(x_0) is zero within its standard error.  With V = V^pi instead (a value that
is NOT the fixed point when rho_bar truncates) the same statistic must be far from zero --
the test has the power to see a wrong fixed point.  Pure CPU (the C oracle), seeded."""
import numpy as np
import pytest

import oracle

S, A, GAMMA = 4, 3, 0.9


def _mdp(seed):
    rng = np.random.default_rng(seed)
    P = rng.dirichlet(np.ones(S), size=(S, A))           # P[x, a, x']
    R = rng.normal(size=(S, A))                          # r(x, a), deterministic
    z_pi = rng.normal(scale=1.5, size=(S, A))            # target logits per state
    z_mu = z_pi + rng.normal(scale=1.0, size=(S, A))     # behaviour logits per state
    return P, R, z_pi, z_mu


def _softmax(z):
    e = np.exp(z - z.max(axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


def _value(P, R, pol):
    """V of a stationary policy: (I - gamma P_pol)^-1 r_pol (exact linear solve)."""
    P_pol = np.einsum("xa,xay->xy", pol, P)
    r_pol = np.einsum("xa,xa->x", pol, R)
    return np.linalg.solve(np.eye(S) - GAMMA * P_pol, r_pol)


def _sample(P, R, z_pi, z_mu, T, N, rng):
    """N trajectories of length T under mu, started uniformly over the states, in the
    oracle's [T, B] layout (fp32 logits), plus the visited states [T + 1, N]."""
    mu = _softmax(z_mu)
    x = np.zeros((T + 1, N), np.int64)
    a = np.zeros((T, N), np.int64)
    x[0] = rng.integers(0, S, size=N)
    cum_mu = np.cumsum(mu, axis=-1)
    cum_P = np.cumsum(P, axis=-1)
    for t in range(T):
        u = rng.random(N)[:, None]
        a[t] = np.minimum((u > cum_mu[x[t]]).sum(axis=-1), A - 1)
        u2 = rng.random(N)[:, None]
        x[t + 1] = np.minimum((u2 > cum_P[x[t], a[t]]).sum(axis=-1), S - 1)
    inp = dict(T=T, B=N, A=A, dtype=oracle.DTYPE_F32,
               target_logits=z_pi[x[:T]].astype(np.float32),
               behaviour_logits=z_mu[x[:T]].astype(np.float32),
               actions=a.astype(np.int32), rewards=R[x[:T], a].astype(np.float32),
               discounts=np.full((T, N), GAMMA, np.float32),
               values=np.zeros((T, N), np.float32), bootstrap_value=np.zeros(N, np.float32))
    return inp, x


def _bias(inp, x, V, rho_bar):
    run = dict(inp)
    run["values"] = V[x[:-1]].astype(np.float32)
    run["bootstrap_value"] = V[x[-1]].astype(np.float32)
    out = oracle.from_logits(run, rho_bar=rho_bar, c_bar=min(1.0, rho_bar))
    d = out["vs"][0] - run["values"][0].astype(np.float64)  # v_0 - V(x_0)
    return float(d.mean()), float(d.std(ddof=1) / np.sqrt(d.size))


@pytest.mark.parametrize("rho_bar,T", [(1.0, 3), (1.0, 8), (0.5, 4), (2.0, 5)])
def test_fixed_point_is_v_of_pi_rho_bar(rho_bar, T):
    P, R, z_pi, z_mu = _mdp(7)
    pi, mu = _softmax(z_pi), _softmax(z_mu)
    pi_rb = np.minimum(rho_bar * mu, pi)
    pi_rb /= pi_rb.sum(axis=-1, keepdims=True)
    V_rb, V_pi = _value(P, R, pi_rb), _value(P, R, pi)
    rng = np.random.default_rng(100 + T)
    inp, x = _sample(P, R, z_pi, z_mu, T, 400_000, rng)
    m, se = _bias(inp, x, V_rb, rho_bar)
    assert abs(m) < 5 * se, (m, se)
    # power: V^pi is not the fixed point when rho_bar truncates pi/mu on this MDP
    m2, se2 = _bias(inp, x, V_pi, rho_bar)
    assert abs(m2) > 20 * se2, (m2, se2)
