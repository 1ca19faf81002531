/* vtrace_oracle.h -- CPU ORACLE for the IMPALA V-trace learner hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_1802_01561_b200/) never links, imports or calls it.
 * It shares no code, header, constant or helper with the CUDA path.
 *
 * What it computes: arxiv 1802.01561 (Espeholt et al., "IMPALA"), Section 4,
 * written out as the plain definitions, column by column, in fp64:
 *   - log-softmax of target (pi) and behaviour (mu) logits
 *   - truncated IS weights rho_t, c_t (Remark 2 lambda)
 *   - V-trace targets v_s by the Remark-1 recursion
 *     (and, separately, by the explicit Eq.(1) double sum)
 *   - q_s = r_s + gamma_s v_{s+1}, pg advantage rho_s(q_s - V_s)
 *   - baseline L2 loss, policy-gradient loss, entropy bonus,
 *     summed over batch and time, and their gradients w.r.t. the
 *     target logits and the values
 *   - reward transforms clip[-1,1] and optimistic asymmetric
 *   - the off-policy correction variants of Section 5.2.2
 *     (no-correction, epsilon-correction, 1-step IS) and the
 *     q_s = r_s + gamma V(x_{s+1}) estimate of App. E.3
 *
 * Layout: time-major.  Logits are [T][B][A] (A fastest), per-step arrays are
 * [T][B], bootstrap is [B].  Logits are given as fp32 (dtype 0) or as raw
 * bfloat16 bit patterns (dtype 1, uint16_t); each input is decoded exactly to
 * double before any arithmetic.  All outputs are double.  Host pointers only.
 * Optional outputs may be NULL.
 *
 * Parity pins: see tests/test_oracle_pins.py (closed forms, brute force,
 * finite differences, SPEC worked examples, the SURVEY toy fixture).
 */
#ifndef VTRACE_ORACLE_H_
#define VTRACE_ORACLE_H_
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes.  0 = ok; 1..7 = argument errors (nothing written);
 * 100+k = data error k (see below), first offending row in *bad_index. */
#define VTO_OK 0
#define VTO_ERR_INVALID_ARG 1
#define VTO_ERR_SHAPE 2
#define VTO_ERR_DTYPE 3
#define VTO_ERR_PARAM 4
/* data error kinds (k) */
#define VTO_DATA_ACTION 1      /* a_t not in [0, A)                 */
#define VTO_DATA_LOGITS 2      /* a non-finite logit in the row      */
#define VTO_DATA_REWARD 3      /* non-finite reward                  */
#define VTO_DATA_VALUE 4       /* non-finite value or bootstrap      */
#define VTO_DATA_DISCOUNT 5    /* discount non-finite or not in [0,1] */

/* Off-policy correction variants of Section 5.2.2. */
#define VTO_CORR_VTRACE 0      /* 4. V-trace (Section 4)                          */
#define VTO_CORR_NONE 1        /* 1. No-correction: rho = c = 1, unweighted PG    */
#define VTO_CORR_EPSILON 2     /* 2. epsilon-correction: as 1, PG uses log(pi+eps) */
#define VTO_CORR_ONE_STEP_IS 3 /* 3. 1-step IS: as 1 for V, PG weighted by rho_pg  */

typedef struct {
  double rho_bar;     /* truncation of rho_t; +inf = none          */
  double c_bar;       /* truncation of c_t; must be <= rho_bar     */
  double pg_rho_bar;  /* truncation of the rho_s in the PG term    */
  double lambda_;     /* Remark 2, in [0, 1]                       */
  int32_t reward_mode;/* 0 none, 1 clip[-1,1], 2 asym tanh */
  int32_t correction; /* VTO_CORR_* (P:410-416); 0 = V-trace               */
  double epsilon;     /* epsilon-correction constant (1e-6)         */
  int32_t q_from_values; /* 0: q_s = r_s + gamma v_{s+1};
                            1: q_s = r_s + gamma V(x_{s+1}) (App. E.3) */
  int32_t behaviour_log_probs; /* 0: behaviour_logits is [T][B][A] mu logits;
                                  1: it is log mu(a_t|x_t) [T][B] fp32 (the actors'
                                  "policy distributions" reduced to the taken action,
                                  P:152)                        */
} vto_params;

typedef struct {
  double baseline_cost; /* 0.5 */
  double entropy_cost;  /* 0.01        */
} vto_weights;

/* partials[8] */
#define VTO_P_PG_LOSS 0
#define VTO_P_BASELINE_LOSS 1
#define VTO_P_ENTROPY_SUM 2
#define VTO_P_TOTAL_LOSS 3
#define VTO_P_SUMSQ_DLOGITS 4
#define VTO_P_SUMSQ_DVALUES 5
#define VTO_P_SUM_RHO 6
#define VTO_P_N_RHO_CLIPPED 7

/* Targets and advantages (the paper's Section 4.1 / 4.2 quantities). */
int vtrace_oracle_from_logits(int64_t T, int64_t B, int64_t A, int32_t dtype,
                              const void* behaviour_logits, const void* target_logits,
                              const int32_t* actions, const float* discounts,
                              const float* rewards, const float* values,
                              const float* bootstrap_value, const vto_params* p,
                              double* vs, double* pg_advantages, double* log_rhos,
                              double* target_action_log_probs,
                              double* behaviour_action_log_probs, int64_t* bad_index);

/* Summed losses and their gradients (Section 4.2 update directions, negated:
 * the gradient of the loss to minimise). grad_target_logits [T][B][A],
 * grad_values [T][B], partials[8]. */
int vtrace_oracle_loss_and_grad(int64_t T, int64_t B, int64_t A, int32_t dtype,
                                const void* behaviour_logits, const void* target_logits,
                                const int32_t* actions, const float* discounts,
                                const float* rewards, const float* values,
                                const float* bootstrap_value, const vto_params* p,
                                const vto_weights* w, double* grad_target_logits,
                                double* grad_values, double* partials, double* vs,
                                double* pg_advantages, int64_t* bad_index);

/* V-trace targets by the explicit Eq.(1) double sum, O(T^2) per
 * column, from given log importance ratios (no logits).  For tiny inputs. */
int vtrace_oracle_vs_eq1(int64_t T, int64_t B, const double* log_rhos,
                         const double* discounts, const double* rewards,
                         const double* values, const double* bootstrap_value,
                         const vto_params* p, double* vs);

/* Same Remark-1 recursion as the main path, from given log ratios. */
int vtrace_oracle_vs_recursion(int64_t T, int64_t B, const double* log_rhos,
                               const double* discounts, const double* rewards,
                               const double* values, const double* bootstrap_value,
                               const vto_params* p, double* vs, double* pg_advantages);

/* Reward transform of one value (P:944 / P:819). */
double vtrace_oracle_reward_transform(double r, int32_t mode);

#ifdef __cplusplus
}
#endif
#endif
