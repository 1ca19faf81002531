"""Pins for the CPU oracle (oracle/): each test ties an oracle output to something
other than the oracle itself -- a value printed in SPEC.md / SURVEY.md, a closed
form from the paper, a second formula from the paper (brute-force Eq.(1)), a
finite difference, or an invariant.  Citations: P:n = PAPER.md line n."""
import json
import math
import os

import numpy as np
import pytest

import oracle
from paper_1802_01561_b200 import workload as wl

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def _batch(T, B, A, seed, p_done=0.2, dtype=wl.DTYPE_F32, spread=1.5, lag=0.3):
    """Small random batch in the library layout (fp32 logits unless bf16)."""
    rng = np.random.default_rng(seed)
    zp = (rng.normal(size=(T, B, A)) * spread).astype(np.float32)
    zm = (zp + rng.normal(size=(T, B, A)) * lag).astype(np.float32)
    if dtype == wl.DTYPE_BF16:
        zp, zm = wl.f32_to_bf16_bits(zp), wl.f32_to_bf16_bits(zm)
    done = rng.random((T, B)) < p_done
    return dict(T=T, B=B, A=A, dtype=dtype,
                target_logits=zp, behaviour_logits=zm,
                actions=rng.integers(0, A, size=(T, B)).astype(np.int32),
                rewards=rng.normal(size=(T, B)).astype(np.float32),
                values=rng.normal(size=(T, B)).astype(np.float32),
                bootstrap_value=rng.normal(size=B).astype(np.float32),
                discounts=np.where(done, 0.0, 0.99).astype(np.float32))


def _logits_for_ratios(ratios):
    """A=2 rows whose pi/mu at action 0 equals `ratio` (mu uniform):
    pi = (ratio/2, 1 - ratio/2), requires ratio < 2."""
    T = len(ratios)
    zp = np.zeros((T, 1, 2), np.float32)
    zm = np.zeros((T, 1, 2), np.float32)
    for t, q in enumerate(ratios):
        p0 = q / 2.0
        zp[t, 0] = [math.log(p0), math.log(1 - p0)]
    return zp, zm


# --------------------------------------------------------------------------
# SURVEY toy fixture (config 1) and hand checks


def test_toy_fixture_matches_survey():
    g = _load("toy_survey.json")
    inp = wl.toy_inputs()
    o = oracle.from_logits(inp)
    lg = oracle.loss_and_grad(inp, baseline_cost=0.5, entropy_cost=0.01)
    for b in (0, 1):
        key = f"b{b}"
        np.testing.assert_allclose(o["log_rhos"][:, b], g["log_rhos"][key], rtol=1e-6, atol=1e-8)
        np.testing.assert_allclose(o["vs"][:, b], g["vs"][key], rtol=1e-6, atol=1e-7)
        np.testing.assert_allclose(o["pg_advantages"][:, b], g["pg_advantages"][key],
                                   rtol=1e-6, atol=1e-7)
        np.testing.assert_allclose(lg["grad_values"][:, b], g["grad_values"][key],
                                   rtol=1e-6, atol=1e-7)
    P = lg["partials"]
    gp = g["partials"]
    np.testing.assert_allclose(P[0], gp["pg_loss"], rtol=1e-6)
    np.testing.assert_allclose(P[1], gp["baseline_loss"], rtol=1e-6)
    np.testing.assert_allclose(P[2], gp["entropy_sum"], rtol=1e-6)
    np.testing.assert_allclose(P[3], gp["total_loss"], rtol=1e-6)
    np.testing.assert_allclose(P[4], gp["sumsq_dlogits"], rtol=1e-6)
    np.testing.assert_allclose(P[5], gp["sumsq_dvalues"], rtol=1e-6)
    # the rho diagnostics (readings r2, r6): counting ratios >= rho_bar
    # instead of > rho_bar gives 9, not 7 (log rho = 0 exactly at two steps)
    np.testing.assert_allclose(P[6], gp["sum_rho"], rtol=1e-9)
    assert P[7] == gp["n_rho_clipped"]
    np.testing.assert_allclose(lg["grad_target_logits"][0, 0], g["grad_target_logits"]["t0_b0"],
                               rtol=1e-6, atol=1e-8)
    np.testing.assert_allclose(lg["grad_target_logits"][4, 1], g["grad_target_logits"]["t4_b1"],
                               rtol=1e-6, atol=1e-8)


def test_rho_diagnostics_chosen_ratios():
    """Partials 6-7 (Sum rho, #clipped; P:196 rho_t = min(rho_bar, pi/mu), readings
    r2/r6) on rows whose ratio pi/mu at the taken action is chosen: A=2, mu uniform,
    pi = (q/2, 1 - q/2).  With c_bar < rho_bar and lambda = 1/2, a sum of
    c = lambda min(c_bar, q) (2.35) instead of rho (5.9), or clipping at c_bar
    (4 clipped, not 2), give different numbers.  The strict '>' of the count is
    pinned by the toy fixture (log rho = 0 exactly at two steps)."""
    ratios = [0.25, 0.5, 0.9, 1.1, 1.5, 1.75, 0.75]
    rho_bar, c_bar = 1.2, 0.8
    zp, zm = _logits_for_ratios(ratios)
    n = len(ratios)
    inp = dict(T=n, B=1, A=2, dtype=0, target_logits=zp, behaviour_logits=zm,
               actions=np.zeros((n, 1), np.int32), rewards=np.ones((n, 1), np.float32),
               values=np.zeros((n, 1), np.float32), bootstrap_value=np.zeros(1, np.float32),
               discounts=np.full((n, 1), 0.5, np.float32))
    P = oracle.loss_and_grad(inp, rho_bar=rho_bar, c_bar=c_bar, lambda_=0.5)["partials"]
    # the ratios pass through fp32 logits (log(q/2) rounded): compare at 1e-6
    np.testing.assert_allclose(P[6], 0.25 + 0.5 + 0.9 + 1.1 + 1.2 + 1.2 + 0.75, rtol=1e-6)
    assert P[7] == 2  # 1.5 and 1.75 exceed rho_bar = 1.2


def test_toy_column0_by_hand():
    """Column b0 has pi/mu >= 1 at every step, so rho = c = 1 and v_s is the
    discounted return with the episode cut at t=2 (Eq.(2); c1)."""
    inp = wl.toy_inputs()
    o = oracle.from_logits(inp)
    g = float(np.float32(0.99))
    r = [0, 1, 0, -1, 1]
    boot = 2.0
    # t=2 is terminal: gamma_2 = 0 cuts both the bootstrap and the trace.
    v4 = r[4] + g * boot
    v3 = r[3] + g * v4
    v2 = r[2]
    v1 = r[1] + g * v2
    v0 = r[0] + g * v1
    np.testing.assert_allclose(o["vs"][:, 0], [v0, v1, v2, v3, v4], rtol=1e-12, atol=1e-12)
    assert np.all(o["log_rhos"][:, 0] >= 0)


# --------------------------------------------------------------------------
# SPEC worked examples


def test_spec_weights_examples():
    """compute_weights examples: through vs of a T=1 column,
    v_0 = V_0 + rho (r + g*boot - V_0), so rho is read back exactly; c is read
    back from a T=2 column: v_0 - V_0 - delta_0 = g c_0 (v_1 - V_1)."""
    for ex in _load("spec_examples.json")["weights"]:
        ratio = ex["pi"] / ex["mu"]
        lr = np.array([[math.log(ratio)], [0.0]])
        g = np.array([[0.5], [0.5]])
        r = np.array([[1.0], [2.0]])
        V = np.array([[0.25], [0.5]])
        boot = np.array([1.0])
        vs, _ = oracle.vs_recursion(lr, g, r, V, boot, rho_bar=ex["rho_bar"],
                                    c_bar=ex["c_bar"], lambda_=ex["lambda"])
        lam = ex["lambda"]
        v1 = V[1, 0] + min(1.0, 1.0) * (r[1, 0] + g[1, 0] * boot[0] - V[1, 0])
        rho0_expected = ex["rho"]
        delta0 = rho0_expected * (r[0, 0] + g[0, 0] * V[1, 0] - V[0, 0])
        c0 = (vs[0, 0] - V[0, 0] - delta0) / (g[0, 0] * (v1 - V[1, 0]))
        assert abs(vs[1, 0] - v1) < 1e-12
        assert abs(c0 - ex["c"]) < 1e-12, (ex, c0, lam)


@pytest.mark.parametrize("via_logits", [False, True])
def test_spec_target_examples(via_logits):
    for ex in _load("spec_examples.json")["targets"]:
        n = len(ex["rewards"])
        g = np.full((n, 1), ex["gamma"])
        r = np.array(ex["rewards"], float).reshape(n, 1)
        V = np.array(ex["values"], float).reshape(n, 1)
        boot = np.array([ex["bootstrap"]], float)
        if not via_logits:
            lr = np.log(np.array(ex["ratios"], float)).reshape(n, 1)
            vs, adv = oracle.vs_recursion(lr, g, r, V, boot)
        else:
            zp, zm = _logits_for_ratios(ex["ratios"])
            inp = dict(T=n, B=1, A=2, dtype=0, target_logits=zp, behaviour_logits=zm,
                       actions=np.zeros((n, 1), np.int32), rewards=r.astype(np.float32),
                       values=V.astype(np.float32), bootstrap_value=boot.astype(np.float32),
                       discounts=g.astype(np.float32))
            o = oracle.from_logits(inp)
            vs, adv = o["vs"], o["pg_advantages"]
        tol = 1e-12 if not via_logits else 2e-7   # fp32 inputs (gamma 0.9 is inexact)
        np.testing.assert_allclose(vs[:, 0], ex["vs"], rtol=tol, atol=tol)
        if "pg_advantages" in ex:
            np.testing.assert_allclose(adv[:, 0], ex["pg_advantages"], rtol=tol, atol=tol)


def test_spec_softmax_examples():
    for ex in _load("spec_examples.json")["softmax"]:
        A = len(ex["logits"])
        for a in range(A):
            z = np.array(ex["logits"], np.float32).reshape(1, 1, A)
            inp = dict(T=1, B=1, A=A, dtype=0, target_logits=z, behaviour_logits=np.zeros_like(z),
                       actions=np.array([[a]], np.int32), rewards=np.zeros((1, 1), np.float32),
                       values=np.zeros((1, 1), np.float32),
                       bootstrap_value=np.zeros(1, np.float32),
                       discounts=np.full((1, 1), 0.99, np.float32))
            o = oracle.from_logits(inp)
            np.testing.assert_allclose(o["target_action_log_probs"][0, 0],
                                       math.log(ex["probs"][a]), rtol=0, atol=1e-7)
            np.testing.assert_allclose(o["behaviour_action_log_probs"][0, 0],
                                       -math.log(A), rtol=0, atol=1e-15)


def test_spec_reward_transform_examples():
    for ex in _load("spec_examples.json")["reward_transform"]:
        assert abs(oracle.reward_transform(ex["r"], ex["mode"]) - ex["out"]) < 1e-9
    assert oracle.reward_transform(-3.0, 1) == -1.0
    assert oracle.reward_transform(0.25, 1) == 0.25
    assert oracle.reward_transform(0.0, 2) == 0.0
    assert oracle.reward_transform(7.5, 0) == 7.5


# --------------------------------------------------------------------------
# Closed forms and the two formulas of the paper


def _eq1_python(lr, g, r, V, boot, rho_bar, c_bar, lam):
    """Eq.(1) in Python, O(T^2): v_s = V_s + sum_t (prod gamma_i)(prod c_i) delta_t."""
    T, B = lr.shape
    out = np.zeros((T, B))
    ratio = np.exp(lr)
    rho = np.minimum(rho_bar, ratio)
    c = lam * np.minimum(c_bar, ratio)
    Vn = np.concatenate([V, boot[None]], 0)
    for b in range(B):
        for s in range(T):
            acc = 0.0
            for t in range(s, T):
                w = 1.0
                for i in range(s, t):
                    w *= g[i, b] * c[i, b]
                acc += w * rho[t, b] * (r[t, b] + g[t, b] * Vn[t + 1, b] - V[t, b])
            out[s, b] = V[s, b] + acc
    return out


@pytest.mark.parametrize("seed", range(40))
def test_recursion_equals_eq1_bruteforce(seed):
    """Remark 1 recursion == Eq.(1) explicit sum on tiny inputs,
    random terminals, rho_bar in {0.5,1,2,inf}, c_bar <= rho_bar, lambda in {0,.5,1}."""
    rng = np.random.default_rng(1000 + seed)
    T = int(rng.integers(1, 7))
    B = 3
    rho_bar = [0.5, 1.0, 2.0, math.inf][seed % 4]
    c_bar = min(rho_bar, [0.3, 1.0, 1.7][seed % 3])
    lam = [0.0, 0.5, 1.0][(seed // 4) % 3]
    lr = rng.normal(size=(T, B)) * 0.8
    g = np.where(rng.random((T, B)) < 0.25, 0.0, rng.uniform(0.5, 1.0, (T, B)))
    r = rng.normal(size=(T, B))
    V = rng.normal(size=(T, B))
    boot = rng.normal(size=B)
    kw = dict(rho_bar=rho_bar, c_bar=c_bar, lambda_=lam, pg_rho_bar=rho_bar)
    rec, _ = oracle.vs_recursion(lr, g, r, V, boot, **kw)
    eq1_c = oracle.vs_eq1(lr, g, r, V, boot, **kw)
    eq1_py = _eq1_python(lr, g, r, V, boot, rho_bar, c_bar, lam)
    np.testing.assert_allclose(rec, eq1_py, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(eq1_c, eq1_py, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("seed", range(10))
def test_on_policy_is_nstep_bellman(seed):
    """pi = mu, c_bar >= 1 => v_s = sum_{t>=s} (prod_{i<t} gamma_i) r_t
    + (prod gamma) V(x_T) (Eq.(2)), log rho == 0 bitwise."""
    rng = np.random.default_rng(seed)
    inp = _batch(int(rng.integers(1, 12)), 4, 5, seed, p_done=0.15)
    inp["behaviour_logits"] = inp["target_logits"].copy()
    for rho_bar, c_bar in [(1.0, 1.0), (3.0, 1.5), (math.inf, 1.0)]:
        o = oracle.from_logits(inp, rho_bar=rho_bar, c_bar=c_bar)
        assert np.all(o["log_rhos"] == 0.0)
        T, B = inp["T"], inp["B"]
        g = inp["discounts"].astype(np.float64)
        r = inp["rewards"].astype(np.float64)
        boot = inp["bootstrap_value"].astype(np.float64)
        ref = np.zeros((T, B))
        for b in range(B):
            for s in range(T):
                acc, w = 0.0, 1.0
                for t in range(s, T):
                    acc += w * r[t, b]
                    w *= g[t, b]
                ref[s, b] = acc + w * boot[b]
        np.testing.assert_allclose(o["vs"], ref, rtol=1e-12, atol=1e-12)


def test_lambda_zero_is_one_step_target():
    """lambda = 0 => v_s = V(x_s) + delta_s V (Remark 2 P:225)."""
    inp = _batch(8, 5, 4, 3)
    o = oracle.from_logits(inp, lambda_=0.0)
    T, B = 8, 5
    rho = np.minimum(1.0, np.exp(o["log_rhos"]))
    V = inp["values"].astype(np.float64)
    Vn = np.concatenate([V[1:], inp["bootstrap_value"][None].astype(np.float64)], 0)
    delta = rho * (inp["rewards"] + inp["discounts"].astype(np.float64) * Vn - V)
    np.testing.assert_allclose(o["vs"], V + delta, rtol=1e-12, atol=1e-12)


def test_q_and_advantage_definition():
    """pg_adv_s = rho_s (r_s + gamma_s v_{s+1} - V(x_s)), v_T = V(x_T)."""
    inp = _batch(9, 6, 3, 4)
    o = oracle.from_logits(inp, rho_bar=2.0, c_bar=1.0)
    rho = np.minimum(2.0, np.exp(o["log_rhos"]))
    vn = np.concatenate([o["vs"][1:], inp["bootstrap_value"][None].astype(np.float64)], 0)
    q = inp["rewards"] + inp["discounts"].astype(np.float64) * vn
    np.testing.assert_allclose(o["pg_advantages"], rho * (q - inp["values"]), rtol=1e-12,
                               atol=1e-12)


def test_terminal_cut_invariance_bitwise():
    """Changing anything after a terminal step t* leaves v_{s<=t*} unchanged,
    bitwise (reading c1)."""
    inp = _batch(10, 4, 5, 5, p_done=0.0)
    inp["discounts"][4, :] = 0.0
    o1 = oracle.from_logits(inp)
    rng = np.random.default_rng(9)
    inp2 = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in inp.items()}
    inp2["rewards"][5:] = rng.normal(size=inp2["rewards"][5:].shape)
    inp2["values"][5:] = rng.normal(size=inp2["values"][5:].shape)
    inp2["target_logits"][5:] += 1.0
    inp2["bootstrap_value"][:] = 123.0
    o2 = oracle.from_logits(inp2)
    assert np.array_equal(o1["vs"][:5], o2["vs"][:5])
    assert np.array_equal(o1["pg_advantages"][:5], o2["pg_advantages"][:5])


def test_logit_shift_invariance():
    inp = _batch(6, 4, 7, 6)
    o1 = oracle.loss_and_grad(inp)
    inp2 = dict(inp)
    inp2["target_logits"] = (inp["target_logits"] + np.float32(4.0)).astype(np.float32)
    inp2["behaviour_logits"] = (inp["behaviour_logits"] - np.float32(2.0)).astype(np.float32)
    o2 = oracle.loss_and_grad(inp2)
    np.testing.assert_allclose(o1["grad_target_logits"], o2["grad_target_logits"], atol=1e-6)
    np.testing.assert_allclose(o1["vs"], o2["vs"], atol=1e-5)


def test_monotone_truncation():
    """Larger rho_bar gives elementwise larger-or-equal rho."""
    inp = _batch(12, 8, 4, 7)
    prev = None
    for rb in [0.25, 0.5, 1.0, 2.0, 8.0]:
        o = oracle.loss_and_grad(inp, rho_bar=rb, c_bar=0.25)
        s = o["partials"][6]
        if prev is not None:
            assert s >= prev
        prev = s


# --------------------------------------------------------------------------
# Gradients


def _total_loss(inp, **kw):
    return oracle.loss_and_grad(inp, **kw)["partials"][3]


@pytest.mark.parametrize("seed", range(4))
def test_grad_logits_finite_difference(seed):
    """dL/dz^pi against central differences of the oracle's own total loss.
    With rho_bar = c_bar = pg_rho_bar tiny, every truncated weight equals the
    threshold in a neighbourhood of the base point, so v, q and pg_adv are
    locally constant and the stop-gradient (reading c10) is exact."""
    rng = np.random.default_rng(seed)
    T = int(rng.integers(1, 5))
    inp = _batch(T, 3, 4, 50 + seed, lag=0.5)
    # Logits on a 2^-8 grid so z +- h (h = 2^-10) is exact in fp32.
    inp["target_logits"] = (np.round(inp["target_logits"] * 256) / 256).astype(np.float32)
    kw = dict(rho_bar=1e-3, c_bar=1e-3, pg_rho_bar=1e-3, baseline_cost=0.5,
              entropy_cost=0.3)
    base = inp
    grad = oracle.loss_and_grad(base, **kw)["grad_target_logits"]
    h = 2.0 ** -10
    zf = base["target_logits"]
    for idx in np.ndindex(zf.shape):
        zp = zf.copy(); zp[idx] += np.float32(h)
        zm = zf.copy(); zm[idx] -= np.float32(h)
        ip, im = dict(base), dict(base)
        ip["target_logits"], im["target_logits"] = zp, zm
        fd = (_total_loss(ip, **kw) - _total_loss(im, **kw)) / (2 * h)
        assert abs(fd - grad[idx]) < 2e-6 * max(1.0, abs(grad[idx])), (idx, fd, grad[idx])


def test_grad_values_is_baseline_residual():
    """dL/dV_s = c_v (V_s - v_s): the gradient of c_v/2 (v - V)^2 with v frozen
    (readings c7, c10); central difference on the frozen loss."""
    inp = _batch(5, 4, 3, 11)
    o = oracle.loss_and_grad(inp, baseline_cost=0.5)
    v = o["vs"]
    V = inp["values"].astype(np.float64)
    h = 1e-6
    fd = (0.5 * 0.5 * ((v - (V + h)) ** 2) - 0.5 * 0.5 * ((v - (V - h)) ** 2)) / (2 * h)
    np.testing.assert_allclose(o["grad_values"], fd, rtol=1e-7, atol=1e-9)


def test_entropy_gradient_zero_at_uniform_and_rowsum():
    """Uniform logits: entropy gradient is 0, so dz_j =
    pg_adv (1/A - 1[j=a]); every gradient row sums to 0."""
    inp = _batch(4, 3, 5, 12)
    inp["target_logits"] = np.zeros_like(inp["target_logits"])
    o = oracle.loss_and_grad(inp, entropy_cost=0.7)
    A = 5
    onehot = np.eye(A)[inp["actions"]]
    ref = o["pg_advantages"][..., None] * (1.0 / A - onehot)
    np.testing.assert_allclose(o["grad_target_logits"], ref, atol=1e-15)
    np.testing.assert_allclose(o["partials"][2], 4 * 3 * math.log(A), rtol=1e-14)
    inp2 = _batch(6, 5, 7, 13)
    o2 = oracle.loss_and_grad(inp2)
    assert np.abs(o2["grad_target_logits"].sum(-1)).max() < 1e-15


def test_loss_is_summed_not_averaged():
    """The loss is summed over batch and time: doubling the batch by
    repeating columns doubles every partial."""
    inp = _batch(5, 3, 4, 14)
    o1 = oracle.loss_and_grad(inp)
    inp2 = dict(inp)
    for k in ("target_logits", "behaviour_logits", "actions", "rewards", "values", "discounts"):
        inp2[k] = np.ascontiguousarray(np.concatenate([inp[k], inp[k]], axis=1))
    inp2["bootstrap_value"] = np.concatenate([inp["bootstrap_value"]] * 2)
    inp2["B"] = 6
    o2 = oracle.loss_and_grad(inp2)
    np.testing.assert_allclose(o2["partials"], 2 * o1["partials"], rtol=1e-13)


# --------------------------------------------------------------------------
# Input decoding, errors


def test_bf16_decoding_is_exact():
    """bf16 bit patterns decode to the same doubles as the equal fp32 values."""
    inp = _batch(5, 4, 6, 15)
    bits_p = wl.f32_to_bf16_bits(inp["target_logits"])
    bits_m = wl.f32_to_bf16_bits(inp["behaviour_logits"])
    inp16 = dict(inp, dtype=1, target_logits=bits_p, behaviour_logits=bits_m)
    inp32 = dict(inp, dtype=0, target_logits=wl.bf16_bits_to_f32(bits_p),
                 behaviour_logits=wl.bf16_bits_to_f32(bits_m))
    a = oracle.loss_and_grad(inp16)
    b = oracle.loss_and_grad(inp32)
    for k in ("grad_target_logits", "grad_values", "partials", "vs", "pg_advantages"):
        assert np.array_equal(a[k], b[k]), k


def test_data_errors_are_reported_with_first_row():
    inp = _batch(4, 3, 5, 16)
    bad = dict(inp, actions=inp["actions"].copy())
    bad["actions"][2, 1] = 5
    o = oracle.from_logits(bad, check=False)
    assert o["status"] == 101 and o["bad_index"] == 2 * 3 + 1
    bad = dict(inp, rewards=inp["rewards"].copy(), discounts=inp["discounts"].copy())
    bad["rewards"][3, 0] = np.nan
    bad["discounts"][1, 2] = 1.5
    o = oracle.from_logits(bad, check=False)
    assert o["status"] == 105 and o["bad_index"] == 1 * 3 + 2
    bad = dict(inp, bootstrap_value=inp["bootstrap_value"].copy())
    bad["bootstrap_value"][2] = np.inf
    o = oracle.from_logits(bad, check=False)
    assert o["status"] == 104 and o["bad_index"] == 4 * 3 + 2
    bad = dict(inp, target_logits=inp["target_logits"].copy())
    bad["target_logits"][0, 2, 3] = -np.inf
    o = oracle.from_logits(bad, check=False)
    assert o["status"] == 102 and o["bad_index"] == 2


def test_param_errors():
    inp = _batch(3, 2, 3, 17)
    with pytest.raises(oracle.OracleError) as e:
        oracle.from_logits(inp, rho_bar=1.0, c_bar=2.0)   # c_bar > rho_bar
    assert e.value.code == 4
    with pytest.raises(oracle.OracleError):
        oracle.from_logits(inp, lambda_=1.5)


# --------------------------------------------------------------------------
# Section 5.2.2 correction variants and the App. E.3 q estimate


def _col_inputs(ex):
    n = len(ex["rewards"])
    g = np.full((n, 1), ex["gamma"])
    r = np.array(ex["rewards"], float).reshape(n, 1)
    V = np.array(ex["values"], float).reshape(n, 1)
    boot = np.array([ex["bootstrap"]], float)
    lr = np.log(np.array(ex["ratios"], float)).reshape(n, 1)
    return lr, g, r, V, boot


def test_spec_variant_examples():
    """SPEC.md:90-91 worked examples: no-correction and 1-step IS on the same column."""
    for ex in _load("spec_examples.json")["variants"]:
        lr, g, r, V, boot = _col_inputs(ex)
        vs, adv = oracle.vs_recursion(lr, g, r, V, boot, correction=ex["correction"])
        np.testing.assert_allclose(vs[:, 0], ex["vs"], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(adv[:, 0], ex["pg_advantages"], rtol=1e-12, atol=1e-12)
        vs1 = oracle.vs_eq1(lr, g, r, V, boot, correction=ex["correction"])
        np.testing.assert_allclose(vs1[:, 0], ex["vs"], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("seed", range(6))
def test_uncorrected_variants_are_nstep_bellman(seed):
    """No-correction, epsilon-correction and 1-step IS use rho = c = 1 for the value
    targets: v_s is the n-step Bellman target Eq.(2), written
    out here, whatever the importance ratios; the V-trace targets differ off-policy."""
    rng = np.random.default_rng(300 + seed)
    inp = _batch(int(rng.integers(2, 10)), 4, 5, 300 + seed, p_done=0.15, lag=0.8)
    T, B = inp["T"], inp["B"]
    g = inp["discounts"].astype(np.float64)
    r = inp["rewards"].astype(np.float64)
    boot = inp["bootstrap_value"].astype(np.float64)
    ref = np.zeros((T, B))
    for b in range(B):
        for s in range(T):
            acc, w = 0.0, 1.0
            for t in range(s, T):
                acc += w * r[t, b]
                w *= g[t, b]
            ref[s, b] = acc + w * boot[b]
    for corr in (oracle.CORR_NONE, oracle.CORR_EPSILON, oracle.CORR_ONE_STEP_IS):
        o = oracle.from_logits(inp, correction=corr)
        np.testing.assert_allclose(o["vs"], ref, rtol=1e-12, atol=1e-12)
    assert np.max(np.abs(oracle.from_logits(inp)["vs"] - ref)) > 1e-3


def test_variant_advantages_closed_forms():
    """pg_adv per variant from its definition: no-/epsilon-correction the plain
    advantage q - V; 1-step IS the same times min(pg_rho_bar, pi/mu); with
    q_from_values, q_s = r_s + gamma_s V(x_{s+1}) for every variant."""
    inp = _batch(9, 6, 4, 77, p_done=0.2, lag=0.8)
    V = inp["values"].astype(np.float64)
    Vn = np.concatenate([V[1:], inp["bootstrap_value"][None].astype(np.float64)], 0)
    g = inp["discounts"].astype(np.float64)
    r = inp["rewards"].astype(np.float64)
    ratio = np.exp(oracle.from_logits(inp)["log_rhos"])
    none = oracle.from_logits(inp, correction=oracle.CORR_NONE)
    vs_next = np.concatenate([none["vs"][1:], inp["bootstrap_value"][None].astype(np.float64)], 0)
    np.testing.assert_allclose(none["pg_advantages"], r + g * vs_next - V, rtol=1e-12, atol=1e-12)
    eps = oracle.from_logits(inp, correction=oracle.CORR_EPSILON)
    np.testing.assert_allclose(eps["pg_advantages"], none["pg_advantages"], rtol=0, atol=0)
    for pg_bar in (1.0, 2.0):
        one = oracle.from_logits(inp, correction=oracle.CORR_ONE_STEP_IS, pg_rho_bar=pg_bar)
        np.testing.assert_allclose(one["pg_advantages"],
                                   np.minimum(pg_bar, ratio) * none["pg_advantages"],
                                   rtol=1e-12, atol=1e-12)
    for corr in (0, 1, 2, 3):
        q = oracle.from_logits(inp, correction=corr, q_from_values=1)
        w = np.minimum(1.0, ratio) if corr in (0, 3) else 1.0
        np.testing.assert_allclose(q["pg_advantages"], w * (r + g * Vn - V), rtol=1e-12,
                                   atol=1e-12)
        # the targets themselves do not depend on the q estimate
        np.testing.assert_allclose(q["vs"], oracle.from_logits(inp, correction=corr)["vs"],
                                   rtol=0, atol=0)


def test_on_policy_all_variants_agree():
    """pi = mu: every variant gives the same targets and advantages."""
    inp = _batch(7, 5, 6, 91)
    inp["behaviour_logits"] = inp["target_logits"].copy()
    ref = oracle.from_logits(inp)
    for corr in (1, 2, 3):
        o = oracle.from_logits(inp, correction=corr)
        np.testing.assert_allclose(o["vs"], ref["vs"], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(o["pg_advantages"], ref["pg_advantages"], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("seed", range(3))
def test_epsilon_correction_gradient_finite_difference(seed):
    """epsilon-correction loss -pg_adv log(pi(a) + eps) (reading c11): its logit
    gradient against central differences.  rho = c = 1 under this variant, so v and
    pg_adv do not depend on pi at all and the differences are exact up to rounding.
    A large eps (0.05) makes the pi/(pi + eps) factor visible."""
    rng = np.random.default_rng(seed)
    inp = _batch(int(rng.integers(1, 4)), 3, 4, 70 + seed, lag=0.5)
    inp["target_logits"] = (np.round(inp["target_logits"] * 256) / 256).astype(np.float32)
    kw = dict(correction=oracle.CORR_EPSILON, epsilon=0.05, baseline_cost=0.5, entropy_cost=0.3)
    grad = oracle.loss_and_grad(inp, **kw)["grad_target_logits"]
    plain = oracle.loss_and_grad(inp, **dict(kw, correction=oracle.CORR_NONE))["grad_target_logits"]
    assert np.max(np.abs(grad - plain)) > 1e-4
    h = 2.0 ** -10
    zf = inp["target_logits"]
    for idx in np.ndindex(zf.shape):
        zp = zf.copy(); zp[idx] += np.float32(h)
        zm = zf.copy(); zm[idx] -= np.float32(h)
        ip, im = dict(inp), dict(inp)
        ip["target_logits"], im["target_logits"] = zp, zm
        fd = (_total_loss(ip, **kw) - _total_loss(im, **kw)) / (2 * h)
        assert abs(fd - grad[idx]) < 2e-6 * max(1.0, abs(grad[idx])), (idx, fd, grad[idx])


def test_epsilon_to_zero_is_no_correction():
    inp = _batch(5, 4, 6, 12)
    a = oracle.loss_and_grad(inp, correction=oracle.CORR_EPSILON, epsilon=1e-300)
    b = oracle.loss_and_grad(inp, correction=oracle.CORR_NONE)
    np.testing.assert_allclose(a["grad_target_logits"], b["grad_target_logits"], rtol=1e-12,
                               atol=1e-15)
    np.testing.assert_allclose(a["partials"], b["partials"], rtol=1e-12)


def test_variant_partials_and_param_checks():
    """rho partials count the rho_t the variant uses (1 off V-trace, reading r6)."""
    inp = _batch(6, 5, 4, 5, lag=0.8)
    for corr in (1, 2, 3):
        p = oracle.loss_and_grad(inp, correction=corr)["partials"]
        assert p[6] == inp["T"] * inp["B"] and p[7] == 0
    p = oracle.loss_and_grad(inp)["partials"]
    assert p[6] < inp["T"] * inp["B"] and p[7] > 0
    for bad in (dict(correction=4), dict(correction=-1), dict(correction=2, epsilon=0.0),
                dict(correction=2, epsilon=float("nan")), dict(q_from_values=2)):
        with pytest.raises(oracle.OracleError):
            oracle.from_logits(inp, **bad)


# --------------------------------------------------------------------------
# behaviour given as log mu(a_t) [T, B]


def test_spec_target_examples_with_behaviour_log_probs():
    """SPEC.md:74-76 worked targets with mu(a_t) given directly: pi(a) = ratio / 2 on a
    2-action row with pi = (ratio/2, 1 - ratio/2), and log mu(a) = log(1/2)."""
    for ex in _load("spec_examples.json")["targets"]:
        n = len(ex["rewards"])
        zp, _ = _logits_for_ratios(ex["ratios"])
        g = np.full((n, 1), ex["gamma"], np.float32)
        inp = dict(T=n, B=1, A=2, dtype=0, target_logits=zp,
                   behaviour_log_probs=np.full((n, 1), math.log(0.5), np.float32),
                   actions=np.zeros((n, 1), np.int32),
                   rewards=np.array(ex["rewards"], np.float32).reshape(n, 1),
                   values=np.array(ex["values"], np.float32).reshape(n, 1),
                   bootstrap_value=np.array([ex["bootstrap"]], np.float32), discounts=g)
        o = oracle.from_logits(inp)
        np.testing.assert_allclose(o["vs"][:, 0], ex["vs"], rtol=2e-7, atol=2e-7)
        np.testing.assert_allclose(o["behaviour_action_log_probs"][:, 0], math.log(0.5), rtol=1e-7)
        if "pg_advantages" in ex:
            np.testing.assert_allclose(o["pg_advantages"][:, 0], ex["pg_advantages"], rtol=2e-7,
                                       atol=2e-7)


@pytest.mark.parametrize("seed", range(4))
def test_behaviour_log_probs_match_logits_mode(seed):
    """Given log mu(a_t) computed from the behaviour logits by an independent
    (numpy, fp64) log-softmax and rounded to fp32, every output matches the
    logits-mode oracle to the fp32 rounding of log mu."""
    inp = _batch(7, 5, 6, 700 + seed, lag=0.6)
    zm = inp["behaviour_logits"].astype(np.float64)
    lse = np.log(np.sum(np.exp(zm - zm.max(-1, keepdims=True)), -1)) + zm.max(-1)
    a = inp["actions"]
    lmu = (np.take_along_axis(zm, a[..., None], -1)[..., 0] - lse).astype(np.float32)
    lp_inp = dict(inp, behaviour_log_probs=lmu)
    for corr in (0, 3):
        ref = oracle.loss_and_grad(inp, correction=corr)
        got = oracle.loss_and_grad(lp_inp, correction=corr)
        for k in ("vs", "pg_advantages", "grad_values", "grad_target_logits"):
            np.testing.assert_allclose(got[k], ref[k], rtol=1e-6, atol=1e-6)
        # (the total loss is a difference of the other terms: absolute tolerance)
        np.testing.assert_allclose(got["partials"][:6], ref["partials"][:6], rtol=1e-6, atol=2e-5)
    o = oracle.from_logits(lp_inp)
    np.testing.assert_array_equal(o["behaviour_action_log_probs"], lmu.astype(np.float64))


def test_behaviour_log_probs_data_error():
    inp = _batch(4, 3, 5, 7)
    lmu = np.full((4, 3), -1.0, np.float32)
    lmu[2, 1] = np.nan
    o = oracle.from_logits(dict(inp, behaviour_log_probs=lmu), check=False)
    assert o["status"] == 100 + 2 and o["bad_index"] == 2 * 3 + 1
