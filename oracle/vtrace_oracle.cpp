// vtrace_oracle.cpp -- plain, slow, fp64 CPU ORACLE (test infrastructure only).
//
// Every function follows the paper (arxiv 1802.01561, PAPER.md) step by step
// in its own order and notation; nothing is blocked, fused or reordered.
// Citations are PAPER.md line numbers ("P:n") with the section / equation.
// Readings where the paper is silent are DESIGN.md section "Readings" (c1..c18).
//
// Parity pins (tests/test_oracle_pins.py) tie every function below to
// something other than itself: SPEC worked examples, Eq.(2) closed form,
// Eq.(1) brute force, finite differences, softmax/entropy closed forms,
// the SURVEY toy fixture.  Nothing here is "parity unpinned".
#include "vtrace_oracle.h"

#include <cmath>
#include <cstring>
#include <limits>
#include <vector>

namespace {

// Exact decode of one logit to double: fp32 as is; bf16 = upper 16 bits of an fp32.
double decode_logit(const void* base, int32_t dtype, int64_t i) {
  if (dtype == 0) return (double)((const float*)base)[i];
  uint32_t bits = (uint32_t)((const uint16_t*)base)[i] << 16;
  float f;
  std::memcpy(&f, &bits, 4);
  return (double)f;
}

bool params_ok(const vto_params* p) {
  if (!p) return false;
  if (std::isnan(p->rho_bar) || std::isnan(p->c_bar) || std::isnan(p->pg_rho_bar) ||
      std::isnan(p->lambda_))
    return false;
  if (!(p->rho_bar > 0) || !(p->c_bar > 0) || !(p->pg_rho_bar > 0)) return false;
  if (p->c_bar > p->rho_bar) return false;  // "we assume rho_bar >= c_bar", reading c6
  if (p->lambda_ < 0 || p->lambda_ > 1) return false;  // Remark 2, lambda in [0,1]
  if (p->reward_mode < 0 || p->reward_mode > 2) return false;
  if (p->correction < VTO_CORR_VTRACE || p->correction > VTO_CORR_ONE_STEP_IS) return false;
  if (p->correction == VTO_CORR_EPSILON && !(p->epsilon > 0 && std::isfinite(p->epsilon)))
    return false;
  if (p->q_from_values != 0 && p->q_from_values != 1) return false;
  if (p->behaviour_log_probs != 0 && p->behaviour_log_probs != 1) return false;
  return true;
}

// The weights each variant uses at one step, from the importance ratio pi/mu
// (Section 5.2.2; readings r5-r7 in DESIGN.md):
//   V-trace (4):        rho = min(rho_bar, ratio), c = lambda min(c_bar, ratio),
//                       rho_pg = min(pg_rho_bar, ratio)
//   No-correction (1):  "No off-policy correction": rho = 1, c = lambda, rho_pg = 1
//   epsilon-corr. (2):  as no-correction (the epsilon enters the log in the PG term)
//   1-step IS (3):      "No off-policy correction when optimising V(x)": rho = 1,
//                       c = lambda; "multiply the advantage at each time step by the
//                       corresponding importance weight": rho_pg = min(pg_rho_bar, ratio)
void variant_weights(const vto_params* p, double ratio, double* rho, double* c,
                     double* rho_pg) {
  if (p->correction == VTO_CORR_VTRACE) {
    *rho = std::min(p->rho_bar, ratio);
    *c = p->lambda_ * std::min(p->c_bar, ratio);
    *rho_pg = std::min(p->pg_rho_bar, ratio);
  } else {
    *rho = 1.0;
    *c = p->lambda_;
    *rho_pg = (p->correction == VTO_CORR_ONE_STEP_IS) ? std::min(p->pg_rho_bar, ratio) : 1.0;
  }
}

// Records the data error with the smallest (row, kind).
struct BadTracker {
  int64_t row = std::numeric_limits<int64_t>::max();
  int kind = 0;
  void hit(int64_t r, int k) {
    if (r < row || (r == row && k < kind)) { row = r; kind = k; }
  }
};

// Log-softmax of one row, written as its definition:
//   log pi(j|x) = z_j - log sum_k exp(z_k)
// evaluated as z_j - m - log sum_k exp(z_k - m) with m = max_k z_k (m is only
// for range; any m gives the same value, reading c14).
void log_softmax_row(const void* logits, int32_t dtype, int64_t row, int64_t A,
                     std::vector<double>& logp) {
  std::vector<double> z(A);
  for (int64_t j = 0; j < A; ++j) z[j] = decode_logit(logits, dtype, row * A + j);
  double m = z[0];
  for (int64_t j = 1; j < A; ++j) m = std::max(m, z[j]);
  double S = 0.0;
  for (int64_t j = 0; j < A; ++j) S += std::exp(z[j] - m);
  double logS = std::log(S);
  for (int64_t j = 0; j < A; ++j) logp[j] = z[j] - m - logS;
}

bool row_logits_finite(const void* logits, int32_t dtype, int64_t row, int64_t A) {
  for (int64_t j = 0; j < A; ++j)
    if (!std::isfinite(decode_logit(logits, dtype, row * A + j))) return false;
  return true;
}

// Per-column V-trace given log importance ratios, per Section 4.1:
//   rho_t = min(rho_bar, pi/mu), c_t = lambda * min(c_bar, pi/mu)
//   (or the weights of a Section 5.2.2 variant, variant_weights above)
//   delta_t V = rho_t (r_t + gamma_t V(x_{t+1}) - V(x_t))
//   v_s = V(x_s) + delta_s V + gamma_s c_s (v_{s+1} - V(x_{s+1}))     (Remark 1)
//   with v_T = V(x_T) = bootstrap (reading c2), gamma_t = discounts[t] (reading c1).
//   q_s = r_s + gamma_s v_{s+1}; pg_adv_s = rho^pg_s (q_s - V(x_s))
void vtrace_column(int64_t T, int64_t B, int64_t b, const double* lr, const double* g,
                   const double* r, const double* V, double boot, const vto_params* p,
                   double* vs_col, double* adv_col, double* rho_col) {
  std::vector<double> rho(T), c(T), rho_pg(T), Vn(T + 1);
  for (int64_t t = 0; t < T; ++t) {
    double ratio = std::exp(lr[t]);
    variant_weights(p, ratio, &rho[t], &c[t], &rho_pg[t]);
    Vn[t] = V[t];
  }
  Vn[T] = boot;
  std::vector<double> v(T + 1);
  v[T] = boot;  // v_{s+n} = V(x_{s+n})
  for (int64_t t = T - 1; t >= 0; --t) {
    double delta = rho[t] * (r[t] + g[t] * Vn[t + 1] - Vn[t]);
    v[t] = Vn[t] + delta + g[t] * c[t] * (v[t + 1] - Vn[t + 1]);
  }
  for (int64_t t = 0; t < T; ++t) {
    // q_s = r_s + gamma_s v_{s+1}, or r_s + gamma_s V(x_{s+1}) (App. E.3)
    double q = r[t] + g[t] * (p->q_from_values ? Vn[t + 1] : v[t + 1]);
    vs_col[t] = v[t];
    adv_col[t] = rho_pg[t] * (q - Vn[t]);
    if (rho_col) rho_col[t] = rho[t];
  }
  (void)B;
  (void)b;
}

// Shared driver: per column b, per row t.  Fills log ratios and log probs,
// then the Remark-1 recursion.  Returns 0 or 100+kind.
int run_targets(int64_t T, int64_t B, int64_t A, int32_t dtype, const void* mu_logits,
                const void* pi_logits, const int32_t* actions, const float* discounts,
                const float* rewards, const float* values, const float* bootstrap,
                const vto_params* p, std::vector<double>& vs, std::vector<double>& adv,
                std::vector<double>& lr, std::vector<double>& lp, std::vector<double>& lm,
                std::vector<double>& rho, std::vector<double>& rew, int64_t* bad_index) {
  BadTracker bad;
  const int64_t N = T * B;
  vs.assign(N, 0.0); adv.assign(N, 0.0); lr.assign(N, 0.0); lp.assign(N, 0.0);
  lm.assign(N, 0.0); rho.assign(N, 0.0); rew.assign(N, 0.0);
  std::vector<double> logp(A), logm(A);
  for (int64_t t = 0; t < T; ++t)
    for (int64_t b = 0; b < B; ++b) {
      const int64_t row = t * B + b;
      int32_t a = actions[row];
      if (a < 0 || a >= A) bad.hit(row, VTO_DATA_ACTION);
      const bool mu_lp = p->behaviour_log_probs != 0;  // mu given as log mu(a_t) [T][B]
      if (!row_logits_finite(pi_logits, dtype, row, A) ||
          (mu_lp ? !std::isfinite(((const float*)mu_logits)[row])
                 : !row_logits_finite(mu_logits, dtype, row, A)))
        bad.hit(row, VTO_DATA_LOGITS);
      if (!std::isfinite(rewards[row])) bad.hit(row, VTO_DATA_REWARD);
      if (!std::isfinite(values[row])) bad.hit(row, VTO_DATA_VALUE);
      if (!std::isfinite(discounts[row]) || discounts[row] < 0.f || discounts[row] > 1.f)
        bad.hit(row, VTO_DATA_DISCOUNT);
      int32_t ac = a < 0 ? 0 : (a >= A ? (int32_t)(A - 1) : a);
      log_softmax_row(pi_logits, dtype, row, A, logp);
      lp[row] = logp[ac];                 // log pi(a_t|x_t)
      if (mu_lp) {
        lm[row] = (double)((const float*)mu_logits)[row];  // log mu(a_t|x_t), given
      } else {
        log_softmax_row(mu_logits, dtype, row, A, logm);
        lm[row] = logm[ac];               // log mu(a_t|x_t)
      }
      lr[row] = lp[row] - lm[row];        // log(pi/mu)
      rew[row] = vtrace_oracle_reward_transform((double)rewards[row], p->reward_mode);
    }
  for (int64_t b = 0; b < B; ++b)
    if (!std::isfinite(bootstrap[b])) bad.hit(N + b, VTO_DATA_VALUE);

  std::vector<double> clr(T), cg(T), cr(T), cV(T), cvs(T), cadv(T), crho(T);
  for (int64_t b = 0; b < B; ++b) {
    for (int64_t t = 0; t < T; ++t) {
      const int64_t row = t * B + b;
      clr[t] = lr[row]; cg[t] = discounts[row]; cr[t] = rew[row]; cV[t] = values[row];
    }
    vtrace_column(T, B, b, clr.data(), cg.data(), cr.data(), cV.data(), (double)bootstrap[b],
                  p, cvs.data(), cadv.data(), crho.data());
    for (int64_t t = 0; t < T; ++t) {
      vs[t * B + b] = cvs[t]; adv[t * B + b] = cadv[t]; rho[t * B + b] = crho[t];
    }
  }
  if (bad.kind) {
    if (bad_index) *bad_index = bad.row;
    return 100 + bad.kind;
  }
  if (bad_index) *bad_index = -1;
  return 0;
}

int check_common(int64_t T, int64_t B, int64_t A, int32_t dtype, const void* mu,
                 const void* pi, const int32_t* actions, const float* discounts,
                 const float* rewards, const float* values, const float* bootstrap,
                 const vto_params* p) {
  if (!mu || !pi || !actions || !discounts || !rewards || !values || !bootstrap || !p)
    return VTO_ERR_INVALID_ARG;
  if (T <= 0 || B <= 0 || A <= 0) return VTO_ERR_SHAPE;
  if (dtype != 0 && dtype != 1) return VTO_ERR_DTYPE;
  if (!params_ok(p)) return VTO_ERR_PARAM;
  return VTO_OK;
}

}  // namespace

extern "C" {

// Reward transforms: clip to [-1, 1] for single tasks and Atari;
// "optimistic asymmetric clipping" 0.3 min(tanh r, 0) + 5.0 max(tanh r, 0) for
// DMLab-30.
double vtrace_oracle_reward_transform(double r, int32_t mode) {
  if (mode == 1) return std::min(1.0, std::max(-1.0, r));
  if (mode == 2) {
    double th = std::tanh(r);
    return 0.3 * std::min(th, 0.0) + 5.0 * std::max(th, 0.0);
  }
  return r;
}

int vtrace_oracle_from_logits(int64_t T, int64_t B, int64_t A, int32_t dtype,
                              const void* behaviour_logits, const void* target_logits,
                              const int32_t* actions, const float* discounts,
                              const float* rewards, const float* values,
                              const float* bootstrap_value, const vto_params* p,
                              double* vs, double* pg_advantages, double* log_rhos,
                              double* target_action_log_probs,
                              double* behaviour_action_log_probs, int64_t* bad_index) {
  int st = check_common(T, B, A, dtype, behaviour_logits, target_logits, actions, discounts,
                        rewards, values, bootstrap_value, p);
  if (st) return st;
  if (!vs || !pg_advantages) return VTO_ERR_INVALID_ARG;
  std::vector<double> v, adv, lr, lp, lm, rho, rew;
  st = run_targets(T, B, A, dtype, behaviour_logits, target_logits, actions, discounts, rewards,
                   values, bootstrap_value, p, v, adv, lr, lp, lm, rho, rew, bad_index);
  const int64_t N = T * B;
  for (int64_t i = 0; i < N; ++i) {
    vs[i] = v[i];
    pg_advantages[i] = adv[i];
    if (log_rhos) log_rhos[i] = lr[i];
    if (target_action_log_probs) target_action_log_probs[i] = lp[i];
    if (behaviour_action_log_probs) behaviour_action_log_probs[i] = lm[i];
  }
  return st;
}

// Section 4.2 "V-trace actor-critic algorithm".  The three update
// directions are, for one step s:
//   value:   (v_s - V(x_s)) grad V(x_s)
//   policy:  rho_s grad log pi(a_s|x_s) (r_s + gamma v_{s+1} - V(x_s))
//   entropy: -grad sum_a pi(a|x_s) log pi(a|x_s)
// "summing these three gradients rescaled by appropriate coefficients",
// with the loss summed over batch and time.  We return the loss whose
// negative gradient is that sum (readings c7, c8, c10):
//   L = -sum pg_adv log pi(a) + c_v * 1/2 sum (v - V)^2 - c_e * sum H,
//   H_s = -sum_j pi_j log pi_j,
//   dL/dz_j = pg_adv (pi_j - 1[j = a]) + c_e pi_j (log pi_j + H_s),
//   dL/dV_s = c_v (V_s - v_s);  v, q, pg_adv, rho are constants (stop-gradient).
int vtrace_oracle_loss_and_grad(int64_t T, int64_t B, int64_t A, int32_t dtype,
                                const void* behaviour_logits, const void* target_logits,
                                const int32_t* actions, const float* discounts,
                                const float* rewards, const float* values,
                                const float* bootstrap_value, const vto_params* p,
                                const vto_weights* w, double* grad_target_logits,
                                double* grad_values, double* partials, double* vs,
                                double* pg_advantages, int64_t* bad_index) {
  int st = check_common(T, B, A, dtype, behaviour_logits, target_logits, actions, discounts,
                        rewards, values, bootstrap_value, p);
  if (st) return st;
  if (!w || !grad_target_logits || !grad_values || !partials) return VTO_ERR_INVALID_ARG;
  if (!std::isfinite(w->baseline_cost) || !std::isfinite(w->entropy_cost))
    return VTO_ERR_PARAM;
  std::vector<double> v, adv, lr, lp, lm, rho, rew;
  st = run_targets(T, B, A, dtype, behaviour_logits, target_logits, actions, discounts, rewards,
                   values, bootstrap_value, p, v, adv, lr, lp, lm, rho, rew, bad_index);
  double L_pg = 0, L_v = 0, H_sum = 0, sq_dz = 0, sq_dv = 0, sum_rho = 0, n_clip = 0;
  std::vector<double> logp(A);
  for (int64_t t = 0; t < T; ++t)
    for (int64_t b = 0; b < B; ++b) {
      const int64_t row = t * B + b;
      int32_t a = actions[row];
      int32_t ac = a < 0 ? 0 : (a >= A ? (int32_t)(A - 1) : a);
      log_softmax_row(target_logits, dtype, row, A, logp);
      double H = 0;
      for (int64_t j = 0; j < A; ++j) H -= std::exp(logp[j]) * logp[j];
      // epsilon-correction: log(pi(a) + eps) in the policy-gradient term (reading
      // c11); its logit gradient is the plain one scaled by pi(a) / (pi(a) + eps)
      const bool eps_corr = p->correction == VTO_CORR_EPSILON;
      const double pa = std::exp(logp[ac]);
      const double logpa = eps_corr ? std::log(pa + p->epsilon) : logp[ac];
      const double wpg = eps_corr ? pa / (pa + p->epsilon) : 1.0;
      L_pg += -adv[row] * logpa;
      double res = v[row] - (double)values[row];
      L_v += 0.5 * res * res;
      H_sum += H;
      for (int64_t j = 0; j < A; ++j) {
        double pj = std::exp(logp[j]);
        double dz = adv[row] * wpg * (pj - (j == ac ? 1.0 : 0.0)) +
                    w->entropy_cost * pj * (logp[j] + H);
        grad_target_logits[row * A + j] = dz;
        sq_dz += dz * dz;
      }
      double dv = w->baseline_cost * ((double)values[row] - v[row]);
      grad_values[row] = dv;
      sq_dv += dv * dv;
      // the rho_t the variant uses in delta_t V; truncations counted for V-trace only (r6)
      sum_rho += rho[row];
      if (p->correction == VTO_CORR_VTRACE && std::exp(lr[row]) > p->rho_bar) n_clip += 1.0;
      if (vs) vs[row] = v[row];
      if (pg_advantages) pg_advantages[row] = adv[row];
    }
  partials[VTO_P_PG_LOSS] = L_pg;
  partials[VTO_P_BASELINE_LOSS] = L_v;
  partials[VTO_P_ENTROPY_SUM] = H_sum;
  partials[VTO_P_TOTAL_LOSS] = L_pg + w->baseline_cost * L_v - w->entropy_cost * H_sum;
  partials[VTO_P_SUMSQ_DLOGITS] = sq_dz;
  partials[VTO_P_SUMSQ_DVALUES] = sq_dv;
  partials[VTO_P_SUM_RHO] = sum_rho;
  partials[VTO_P_N_RHO_CLIPPED] = n_clip;
  return st;
}

// Eq.(1), literally:
//   v_s = V(x_s) + sum_{t=s}^{s+n-1} gamma^{t-s} (prod_{i=s}^{t-1} c_i) delta_t V
// with per-step discounts gamma_i (reading c1: gamma^{t-s} -> prod_{i=s}^{t-1} gamma_i)
// and the horizon of each s running to the end of the unroll (reading c2).
int vtrace_oracle_vs_eq1(int64_t T, int64_t B, const double* log_rhos, const double* discounts,
                         const double* rewards, const double* values,
                         const double* bootstrap_value, const vto_params* p, double* vs) {
  if (!log_rhos || !discounts || !rewards || !values || !bootstrap_value || !p || !vs)
    return VTO_ERR_INVALID_ARG;
  if (T <= 0 || B <= 0) return VTO_ERR_SHAPE;
  if (!params_ok(p)) return VTO_ERR_PARAM;
  for (int64_t b = 0; b < B; ++b)
    for (int64_t s = 0; s < T; ++s) {
      double sum = 0.0;
      for (int64_t t = s; t < T; ++t) {
        double disc_prod = 1.0, c_prod = 1.0;
        for (int64_t i = s; i < t; ++i) {
          double rho_i, c_i, pg_i;
          variant_weights(p, std::exp(log_rhos[i * B + b]), &rho_i, &c_i, &pg_i);
          disc_prod *= discounts[i * B + b];
          c_prod *= c_i;
        }
        double rho_t, c_t, pg_t;
        variant_weights(p, std::exp(log_rhos[t * B + b]), &rho_t, &c_t, &pg_t);
        double V_next = (t + 1 < T) ? values[(t + 1) * B + b] : bootstrap_value[b];
        double delta = rho_t * (rewards[t * B + b] + discounts[t * B + b] * V_next -
                                values[t * B + b]);
        sum += disc_prod * c_prod * delta;
      }
      vs[s * B + b] = values[s * B + b] + sum;
    }
  return VTO_OK;
}

int vtrace_oracle_vs_recursion(int64_t T, int64_t B, const double* log_rhos,
                               const double* discounts, const double* rewards,
                               const double* values, const double* bootstrap_value,
                               const vto_params* p, double* vs, double* pg_advantages) {
  if (!log_rhos || !discounts || !rewards || !values || !bootstrap_value || !p || !vs)
    return VTO_ERR_INVALID_ARG;
  if (T <= 0 || B <= 0) return VTO_ERR_SHAPE;
  if (!params_ok(p)) return VTO_ERR_PARAM;
  std::vector<double> clr(T), cg(T), cr(T), cV(T), cvs(T), cadv(T);
  for (int64_t b = 0; b < B; ++b) {
    for (int64_t t = 0; t < T; ++t) {
      clr[t] = log_rhos[t * B + b]; cg[t] = discounts[t * B + b];
      cr[t] = rewards[t * B + b]; cV[t] = values[t * B + b];
    }
    vtrace_column(T, B, b, clr.data(), cg.data(), cr.data(), cV.data(), bootstrap_value[b], p,
                  cvs.data(), cadv.data(), nullptr);
    for (int64_t t = 0; t < T; ++t) {
      vs[t * B + b] = cvs[t];
      if (pg_advantages) pg_advantages[t * B + b] = cadv[t];
    }
  }
  return VTO_OK;
}

}  // extern "C"
