/* vtrace.h -- C ABI of the B200-native IMPALA V-trace learner hot path.
 *
 * Implements, on one NVIDIA B200 (sm_100a), the learner-side computation of
 * Espeholt et al., "IMPALA: Scalable Distributed Deep-RL with Importance
 * Weighted Actor-Learner Architectures", arxiv 1802.01561, Section 4:
 *
 *   log pi(a_t|x_t), log mu(a_t|x_t) from full logits rows
 *   rho_t = min(rho_bar, pi/mu), c_t = lambda min(c_bar, pi/mu)  P:196 (Eq.1), P:225 (Remark 2)
 *   delta_t V = rho_t (r_t + gamma_t V(x_{t+1}) - V(x_t))
 *   v_s = V(x_s) + delta_s V + gamma_s c_s (v_{s+1} - V(x_{s+1})) P:222 (Remark 1)
 *   q_s = r_s + gamma_s v_{s+1};  pg_adv_s = rho_s (q_s - V(x_s)) P:242
 *   L = -sum pg_adv log pi(a) + c_v 1/2 sum (v - V)^2 - c_e sum H
 *   dL/dz^pi and dL/dV (v, q, pg_adv, rho held constant)
 *
 * Notation follows Section 4: t in [0,T) is time, b in [0,B) is the trajectory
 * (batch column), j in [0,A) the action.  The episode-end convention (the paper
 * is silent) is gamma_t = gamma (1 - done_t): a discount of 0 cuts both the
 * bootstrap term of delta_t and the trace (reading c1).  v_T is the
 * bootstrap value V(x_T) (reading c2).  All sums run over batch AND time.
 *
 * Conventions for every call:
 *  - All array pointers are CUDA DEVICE pointers, C-contiguous, time-major:
 *    logits [T][B][A] (A fastest), per-step arrays [T][B], bootstrap [B].
 *  - Every call is asynchronous on `stream`, allocates nothing, never
 *    synchronises the host (except vtrace_read_device_status), and is CUDA-graph
 *    capturable.  The caller owns all memory; outputs must not alias inputs.
 *  - Host-checkable problems are reported by the return value before anything
 *    is launched or written.  Problems in the DATA (bad action index, non-finite
 *    values, discount outside [0,1]) cannot be seen by the host: the kernel
 *    records the smallest offending row (t*B + b, or T*B + b for bootstrap[b])
 *    with its kind in the workspace status word, keeps every memory access in
 *    bounds (the action index is clamped for the gather), and leaves the
 *    outputs of bad rows unspecified.  Read it with vtrace_read_device_status.
 *  - The workspace (size from vtrace_workspace_bytes) must be initialised once
 *    with vtrace_workspace_init before its first use; it carries the decoupled
 *    look-back flags, per-tile partial sums and the status word across calls
 *    (epoch-tagged: no per-call memset).  Calls that may run concurrently need
 *    distinct workspaces.
 *  - Requires an sm_100 device (B200).  No CPU fallback exists.
 */
#ifndef VTRACE_B200_H_
#define VTRACE_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* vt_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
  VT_OK = 0,
  VT_ERR_INVALID_ARG = 1, /* a required pointer is NULL                                 */
  VT_ERR_SHAPE = 2,       /* T, B or A <= 0, A > VT_MAX_ACTIONS, or T*B*A overflows     */
  VT_ERR_DTYPE = 3,       /* logits dtype not VT_FLOAT32 / VT_BFLOAT16                   */
  VT_ERR_PARAM = 4,       /* thresholds <= 0 or NaN, c_bar > rho_bar, lambda not
                             in [0,1], unknown reward mode, non-finite costs      */
  VT_ERR_ALIGNMENT = 5,   /* a pointer is not aligned to its element size               */
  VT_ERR_WORKSPACE = 6,   /* workspace NULL, too small, or not 256-byte aligned         */
  VT_ERR_CUDA = 7,        /* a CUDA runtime call or launch failed                        */
  VT_ERR_DEVICE = 8       /* current device is not compute capability 10.0 (sm_100)    */
} vt_status;

typedef enum { VT_FLOAT32 = 0, VT_BFLOAT16 = 1 } vt_dtype;

/* Reward transform applied to r_t before use (P:834 / P:944: clip to [-1,1];
 * P:819 / P:835: optimistic asymmetric clipping for DMLab-30). */
typedef enum {
  VT_REWARD_NONE = 0,
  VT_REWARD_CLIP_UNIT = 1, /* min(1, max(-1, r))                          */
  VT_REWARD_ASYM_TANH = 2  /* 0.3 min(tanh r, 0) + 5.0 max(tanh r, 0)       */
} vt_reward_mode;

/* Data-error kinds recorded in the device status word. */
typedef enum {
  VT_DATA_OK = 0,
  VT_DATA_ACTION = 1,   /* a_t outside [0, A)                              */
  VT_DATA_LOGITS = 2,   /* a non-finite logit in the row (either policy)   */
  VT_DATA_REWARD = 3,   /* non-finite reward                               */
  VT_DATA_VALUE = 4,    /* non-finite V(x_t) or bootstrap                  */
  VT_DATA_DISCOUNT = 5  /* discount non-finite or outside [0, 1]           */
} vt_data_error;

#define VT_MAX_ACTIONS 1024

/* Off-policy correction (Section 5.2.2; readings r5-r7).
 * Per step, from the importance ratio pi(a_t)/mu(a_t):
 *   V-trace          rho = min(rho_bar, ratio), c = lambda min(c_bar, ratio),
 *                    rho_pg = min(pg_rho_bar, ratio)                 (Section 4)
 *   no-correction    rho = 1, c = lambda, rho_pg = 1
 *   epsilon          as no-correction; the policy-gradient term uses
 *                    log(pi(a) + epsilon)
 *   1-step IS        rho = 1, c = lambda, rho_pg = min(pg_rho_bar, ratio) */
typedef enum {
  VT_CORRECTION_VTRACE = 0,
  VT_CORRECTION_NONE = 1,
  VT_CORRECTION_EPSILON = 2,
  VT_CORRECTION_ONE_STEP_IS = 3
} vt_correction;

/* A zero-initialised struct with the three thresholds and lambda set is plain
 * V-trace with q_s = r_s + gamma_s v_{s+1}. */
typedef struct {
  float clip_rho_threshold;    /* rho_bar; +INFINITY = no truncation         */
  float clip_c_threshold;      /* c_bar; must be <= clip_rho_threshold       */
  float clip_pg_rho_threshold; /* truncation of the rho_s in the PG term;
                                  the paper uses rho_bar (reading c4)                */
  float lambda_;               /* Remark 2, in [0, 1]; 1 = plain V-trace     */
  int32_t reward_mode;         /* vt_reward_mode                                     */
  int32_t correction;          /* vt_correction; 0 = V-trace                         */
  float epsilon;               /* epsilon of VT_CORRECTION_EPSILON (1e-6);
                                  must be finite and > 0 with that correction        */
  int32_t q_from_values;       /* 0: q_s = r_s + gamma_s v_{s+1};
                                  1: q_s = r_s + gamma_s V(x_{s+1}) (App. E.3) */
  int32_t behaviour_log_probs; /* 0: behaviour_policy_logits is mu's [T][B][A] logits;
                                  1: it is log mu(a_t|x_t) [T][B] fp32 (the actors ship
                                  only the taken action's log-probability; SURVEY 8(f)
                                  NEXT #2), 4-byte aligned; logits_dtype still gives
                                  the target logits' dtype                           */
  int32_t overlap_previous;    /* 1: this call's inputs are not outputs of the previous
                                  kernel on `stream` (e.g. consecutive learner steps on
                                  fresh trajectories).  The wide-batch kernel is then
                                  launched as a programmatic dependent: its prologue
                                  (input loads, the first chunk's statistics) overlaps
                                  the previous kernel's tail, and it waits for that
                                  kernel before its first global write.  0 = plain
                                  stream order (always safe)                         */
  int32_t kernel;              /* vt_kernel: which kernel runs the call; 0 = automatic
                                  (a pure function of the shape and pointer alignment,
                                  vtrace_kernel_for).  A forced kernel that cannot take
                                  the shape returns VT_ERR_SHAPE.  Tests / A-B only    */
  int32_t sm_budget;           /* > 0: the column-block kernel plans for at most this
                                  many SMs (e.g. leave SMs to a concurrent per-step
                                  collective); 0 = every SM        */
} vt_vtrace_params;

/* Kernel choice (vt_vtrace_params.kernel). */
typedef enum {
  VT_KERNEL_AUTO = 0,
  VT_KERNEL_COLUMN_BLOCK = 1, /* vtrace_cb_kernel: one CTA per SM owns a block of
                                 trajectories over the whole unroll (TMA ring)       */
  VT_KERNEL_LOOKBACK = 2      /* vtrace_fused_kernel: (8 trajectories x Tc steps)
                                 units, decoupled look-back across time chunks       */
} vt_kernel;

typedef struct {
  float baseline_cost; /* c_v: "baseline loss scaling" 0.5 */
  float entropy_cost;  /* c_e: entropy regulariser 0.01           */
} vt_loss_weights;

/* Indices into the double partials[VT_P_COUNT] output (sums over this call's
 * batch and time; shards of one global batch add up elementwise). */
enum {
  VT_P_PG_LOSS = 0,       /* -sum pg_adv_t log pi(a_t|x_t)                       */
  VT_P_BASELINE_LOSS = 1, /* 1/2 sum (v_t - V(x_t))^2                            */
  VT_P_ENTROPY_SUM = 2,   /* sum_t H_t, H = -sum_j pi_j log pi_j                 */
  VT_P_TOTAL_LOSS = 3,    /* PG + c_v BASELINE - c_e ENTROPY                    */
  VT_P_SUMSQ_DLOGITS = 4, /* sum of squared dL/dz^pi (fp32 values before the
                             store rounding)                                     */
  VT_P_SUMSQ_DVALUES = 5, /* sum of squared dL/dV                                */
  VT_P_SUM_RHO = 6,       /* sum of truncated rho_t                              */
  VT_P_N_RHO_CLIPPED = 7, /* number of steps with pi/mu > rho_bar                */
  VT_P_COUNT = 8
};

/* Bytes of device workspace needed for a (T, B, A, dtype) problem.  0 on bad
 * arguments.  The size depends only on these four numbers. */
size_t vtrace_workspace_bytes(int64_t T, int64_t B, int64_t A, vt_dtype logits_dtype);

/* One-time initialisation of a workspace (stream-ordered memset). */
vt_status vtrace_workspace_init(void* workspace, size_t workspace_bytes, vt_stream_t stream);

/* V-trace targets and policy-gradient advantages (Section 4.1-4.2).
 *   behaviour_policy_logits  z^mu [T][B][A]  logits of the actors' policy mu
 *   target_policy_logits     z^pi [T][B][A]  logits of the learner's policy pi
 *   actions                  a_t  [T][B]     int32 in [0, A)
 *   discounts                gamma_t [T][B]  fp32 in [0,1]; gamma (1 - done_t)
 *   rewards                  r_t  [T][B]     fp32, raw (p->reward_mode applied here)
 *   values                   V(x_t) [T][B]   fp32
 *   bootstrap_value          V(x_T) [B]      fp32
 * Outputs (fp32 [T][B]): vs = v_t (required), pg_advantages (required),
 *   log_rhos = log(pi/mu)(a_t), target_action_log_probs, behaviour_action_log_probs
 *   (each nullable).  Logits are fp32 or bf16 (bf16 values are used exactly).
 *   Pointers must be aligned to their element size. */
vt_status vtrace_from_logits(int64_t T, int64_t B, int64_t A, vt_dtype logits_dtype,
                             const void* behaviour_policy_logits,
                             const void* target_policy_logits, const int32_t* actions,
                             const float* discounts, const float* rewards,
                             const float* values, const float* bootstrap_value,
                             const vt_vtrace_params* params, float* vs, float* pg_advantages,
                             float* log_rhos, float* target_action_log_probs,
                             float* behaviour_action_log_probs, void* workspace,
                             size_t workspace_bytes, vt_stream_t stream);

/* Fused V-trace + actor-critic loss + gradients (Section 4.2, summed per P:789).
 * Same seven inputs as vtrace_from_logits.  Outputs:
 *   grad_target_logits [T][B][A] in the logits dtype (bf16: round-to-nearest-even)
 *       dL/dz^pi_j = pg_adv (pi_j - 1[j=a_t]) + c_e pi_j (log pi_j + H_t)
 *   grad_values [T][B] fp32: dL/dV(x_t) = c_v (V(x_t) - v_t)
 *   partials [VT_P_COUNT] double (device): this call's sums (deterministic:
 *       fixed-order reduction, bitwise reproducible run to run)
 *   vs, pg_advantages [T][B] fp32: nullable.
 * No gradient flows to z^mu, the bootstrap value or the rewards (reading c10). */
vt_status vtrace_loss_and_grad(int64_t T, int64_t B, int64_t A, vt_dtype logits_dtype,
                               const void* behaviour_policy_logits,
                               const void* target_policy_logits, const int32_t* actions,
                               const float* discounts, const float* rewards,
                               const float* values, const float* bootstrap_value,
                               const vt_vtrace_params* params, const vt_loss_weights* weights,
                               void* grad_target_logits, float* grad_values, double* partials,
                               float* vs, float* pg_advantages, void* workspace,
                               size_t workspace_bytes, vt_stream_t stream);

/* vtrace_loss_and_grad for one of num_learners synchronous learners (SURVEY
 * 8(a) a13) with the learners' sum of the partials INSIDE the kernel: the column-block
 * kernel's last CTA stores this learner's 8 partials into its slot of every learner's
 * mailbox (NVLink stores into peer memory), waits for every learner's slot of this call in
 * its own mailbox and writes the sum in learner order to `partials` -- bitwise the same on
 * every learner; no separate collective.  The call's tag is the workspace's call count, so
 * every learner must make the same sequence of calls on workspaces initialised together,
 * and a mailbox serves one such sequence.  mailboxes: host array of num_learners device
 * pointers (16-byte aligned) to each learner's mailbox of
 * vtrace_partials_mailbox_bytes(num_learners) bytes, zero-initialised once, peer-mapped.
 * Shapes that do not take the column-block kernel: VT_ERR_SHAPE (use vtrace_loss_and_grad
 * + vtrace_partials_allreduce).  A learner that never calls leaves the others waiting at
 * most 20 s, then its terms read NaN.  Other arguments and errors as vtrace_loss_and_grad. */
vt_status vtrace_loss_and_grad_learners(
    int64_t T, int64_t B, int64_t A, vt_dtype logits_dtype, const void* behaviour_policy_logits,
    const void* target_policy_logits, const int32_t* actions, const float* discounts,
    const float* rewards, const float* values, const float* bootstrap_value,
    const vt_vtrace_params* params, const vt_loss_weights* weights, void* grad_target_logits,
    float* grad_values, double* partials, float* vs, float* pg_advantages, void* workspace,
    size_t workspace_bytes, double* const* mailboxes, int32_t num_learners, int32_t self,
    vt_stream_t stream);

/* End-to-end variant for inputs that live in HOST memory (the actors' queue):
 * copies the seven host inputs (pinned memory recommended) into the caller's
 * device staging buffers with cudaMemcpyAsync, runs vtrace_loss_and_grad, and
 * copies the partials back to host `partials_host`.  Gradients stay on the
 * device (they feed the network backward).  Asynchronous on `stream`; the host
 * values are valid after the stream is synchronised.  d_* are device buffers of
 * the inputs' sizes. */
vt_status vtrace_loss_and_grad_from_host(
    int64_t T, int64_t B, int64_t A, vt_dtype logits_dtype, const void* h_behaviour_logits,
    const void* h_target_logits, const int32_t* h_actions, const float* h_discounts,
    const float* h_rewards, const float* h_values, const float* h_bootstrap_value,
    void* d_behaviour_logits, void* d_target_logits, int32_t* d_actions, float* d_discounts,
    float* d_rewards, float* d_values, float* d_bootstrap_value,
    const vt_vtrace_params* params, const vt_loss_weights* weights, void* grad_target_logits,
    float* grad_values, double* partials_device, double* partials_host, void* workspace,
    size_t workspace_bytes, vt_stream_t stream);

/* Reads and clears the device status word: *code = vt_data_error of the
 * smallest offending row (VT_DATA_OK if none), *first_bad_flat_index = that
 * row (-1 if none).  Synchronises `stream` (the only call that does). */
vt_status vtrace_read_device_status(void* workspace, int32_t* code,
                                    int64_t* first_bad_flat_index, vt_stream_t stream);

/* Static, NUL-terminated description of a status code. */
const char* vtrace_status_string(vt_status status);

/* Library ABI version (major*10000 + minor*100 + patch). */
int32_t vtrace_version(void);

/* Name of the kernel a call with this shape takes when every pointer is 16-byte
 * aligned (as torch / cudaMalloc allocations are): "vtrace_ctb_kernel" (wide
 * batches, one 16-warp CTA per SM: one warp per 4 trajectories, the remainder
 * cut into time segments to balance the SM sub-partitions; needs the current
 * device's SM count), "vtrace_ct_kernel" (wide batches, one-warp CTAs),
 * "vtrace_fused_kernel" (look-back kernel, TMA staging) or
 * "vtrace_fused_kernel (plain loads)".  Host-only (at most a device-attribute
 * query, no launch); static string.  Used by bench.py to name the kernel its
 * roofline line describes. */
const char* vtrace_kernel_for(int64_t T, int64_t B, int64_t A, vt_dtype logits_dtype);

/* ---- The learner's parameter update -------------------
 * The step after the network backward: clip the global gradient norm at
 * max_global_norm (40), then RMSProp with momentum 0.
 * The paper gives no formula; the TensorFlow form is used (its implementation is
 * TF), epsilon inside the square root (readings r9, r10):
 *     g'    = g * c / max(||g||_2, c)          (||.|| over all n parameters)
 *     ms    <- decay * ms + (1 - decay) * g'^2
 *     theta <- theta - lr * g' / sqrt(ms + epsilon)
 * With several learners the caller first SUM-all-reduces the
 * gradient (the loss is summed over the batch; reading r11), then every
 * learner applies the same update to its replica. */
typedef struct {
  float learning_rate;   /* > 0; the paper anneals it linearly to 0, caller's job */
  float decay;           /* RMSProp mean-square decay, in [0, 1) (not given by the paper)  */
  float epsilon;         /* > 0, inside the square root (0.01; sweep P:786)        */
  float max_global_norm; /* > 0: clip threshold c (40); 0: no clipping             */
} vt_rmsprop_params;

/* Workspace bytes for vtrace_rmsprop_step (initialise once with
 * vtrace_workspace_init; not shared with a V-trace call or a concurrent update). */
size_t vtrace_rmsprop_workspace_bytes(int64_t n);

/* One clipped RMSProp step over n fp32 parameters, in place.
 *   params       theta [n]  fp32 device, updated in place
 *   mean_square  ms    [n]  fp32 device, updated in place (the caller initialises it)
 *   grads        g     [n]  fp32 device, read only (the batch's summed gradient)
 *   global_norm_out         optional fp64 device scalar: ||g||_2 before clipping
 * The three arrays must not overlap; 4-byte alignment is required, 16-byte
 * alignment of all three takes the vector path.  n = 0 is a no-op (norm 0).
 * Non-finite gradients propagate (the norm reports them).  Errors: VT_ERR_INVALID_ARG
 * (NULL array), VT_ERR_SHAPE (n < 0), VT_ERR_PARAM (see the struct), VT_ERR_ALIGNMENT,
 * VT_ERR_WORKSPACE, VT_ERR_DEVICE, VT_ERR_CUDA.  One cooperative launch (one CTA
 * per SM) on `stream`; deterministic (fixed reduction order). */
vt_status vtrace_rmsprop_step(int64_t n, float* params, float* mean_square, const float* grads,
                              const vt_rmsprop_params* prm, double* global_norm_out,
                              void* workspace, size_t workspace_bytes, vt_stream_t stream);

/* The same step on the SUM of num_grads (1..8) gradient buffers, added in index order
 * in fp32 inside the kernel: `grads` is a HOST array of DEVICE pointers, which may
 * be other GPUs' memory reachable over NVLink (peer / symmetric-memory buffers).
 * Learners that pass the same buffers in the same order compute bitwise-identical
 * norms and updates, so the gradient all-reduce (reading r11) happens in
 * this kernel.  The caller orders the accesses: every buffer is complete before
 * the call, and no buffer is overwritten before every learner's call has finished
 * (e.g. a barrier on both sides).  Errors as vtrace_rmsprop_step; num_grads out of
 * range or a NULL entry: VT_ERR_INVALID_ARG. */
vt_status vtrace_rmsprop_step_multi(int64_t n, float* params, float* mean_square,
                                    const float* const* grads, int32_t num_grads,
                                    const vt_rmsprop_params* prm, double* global_norm_out,
                                    void* workspace, size_t workspace_bytes,
                                    vt_stream_t stream);

/* The multi-learner step with the learners' synchronisation inside the kernel (no
 * separate barrier).  grads[j] (host array of device pointers) is learner j's
 * gradient buffer and flags[j] its two zero-initialised uint32 words {ready, done}
 * (8-byte aligned), all in memory every learner can reach (e.g. symmetric memory
 * over NVLink); `self` is the caller's index.  Call k of every learner (counted by
 * its workspace) publishes ready = k + 1 when its kernel starts -- the caller's own
 * buffer must be complete by then (earlier work on `stream`) -- waits for every
 * ready >= k + 1 before reading the buffers, and ends only after every learner has
 * published done >= k + 1, so each buffer may be refilled after the call returns on
 * the stream.  Every learner must make the same sequence of calls with the same
 * buffer order (the sums, norms and updates are then bitwise identical); a learner
 * that does not call leaves the others waiting.  Errors: as
 * vtrace_rmsprop_step_multi; flags NULL, a NULL entry or self out of range:
 * VT_ERR_INVALID_ARG. */
vt_status vtrace_rmsprop_step_learners(int64_t n, float* params, float* mean_square,
                                       const float* const* grads, uint32_t* const* flags,
                                       int32_t num_learners, int32_t self,
                                       const vt_rmsprop_params* prm, double* global_norm_out,
                                       void* workspace, size_t workspace_bytes,
                                       vt_stream_t stream);

/* The learners' update sharded over the learners (a reduce-scatter / all-gather inside
 * one kernel per learner): learner `self` owns the float4 units
 * [U*self/N, U*(self+1)/N) of the n parameters (U = n/4; the n % 4 tail belongs to the
 * last learner).  For its units it sums every learner's gradient (learner order, NVLink
 * reads), adds its shard's sum of squares to the others' through the peer-mapped norm
 * mailboxes (learner order: the same norm, bitwise, on every learner), clips, applies
 * RMSProp to its own mean_square, and stores the new theta into EVERY learner's params
 * (NVLink stores), so the replicas stay bitwise equal while each learner reads 1/N of
 * the peers' gradients.  mean_square: each learner's entries outside its shard are not
 * read or written (each owns its shard's state).
 *   params          host array of num_learners device pointers, each learner's params
 *                   (peer-mapped, 16-byte aligned); params[self] is this learner's
 *   grads, flags    as vtrace_rmsprop_step_learners
 *   norm_mailboxes  host array of num_learners device pointers: learner j's mailbox of
 *                   vtrace_rmsprop_norm_mailbox_bytes(num_learners) bytes, zero-initialised
 *                   once, peer-mapped, 16-byte aligned
 * Arrays must be 16-byte aligned (else VT_ERR_ALIGNMENT) and a shard must fit the
 * register-resident form (148 x 512 x 6 float4 units; else VT_ERR_SHAPE).  Other errors
 * and the call discipline as vtrace_rmsprop_step_learners. */
size_t vtrace_rmsprop_norm_mailbox_bytes(int32_t num_learners);

/* The push half of a push-based gradient all-gather: learner `self` stores its
 * gradient into slot `self` of every learner's receive buffer (NVLink stores into peer
 * memory; posted writes instead of the peers' remote reads), then fences at system scope, so
 * that a following vtrace_rmsprop_step_learners on the same stream -- given the LOCAL slots
 * recv[0..N-1] of this learner's own receive buffer as its gradients -- may publish ready and
 * every learner reads only local memory.  The learners' ready / done protocol of that call is
 * what makes a slot safe to read and to refill.
 *   grad         float[n] device (16-byte aligned): this learner's gradient
 *   recv         host array of num_learners device pointers (16-byte aligned): learner r's
 *                receive buffer of num_learners * n floats, slot j at recv[r] + j * n
 *                (peer-mapped, e.g. symmetric memory)
 * Errors: VT_ERR_INVALID_ARG (NULL, num_learners or self out of range), VT_ERR_SHAPE (n < 0 or
 * n % 4 != 0), VT_ERR_ALIGNMENT, VT_ERR_DEVICE, VT_ERR_CUDA.  One launch on `stream`. */
vt_status vtrace_grad_push(const float* grad, float* const* recv, int32_t num_learners,
                           int32_t self, int64_t n, vt_stream_t stream);
vt_status vtrace_rmsprop_step_sharded(int64_t n, float* const* params, float* mean_square,
                                      const float* const* grads, uint32_t* const* flags,
                                      double* const* norm_mailboxes, int32_t num_learners,
                                      int32_t self, const vt_rmsprop_params* prm,
                                      double* global_norm_out, void* workspace,
                                      size_t workspace_bytes, vt_stream_t stream);

/* ---- SURVEY.md 8(a) a13 over NVLink peer memory ----
 * The sum of the synchronous learners' partials (every learner computes the
 * loss of its own trajectories and the losses add, summed loss P:789) in one 32-thread
 * kernel per step instead of a collective-library call: learner `self` stores its
 * VT_P_COUNT partials (value, then a call tag with release semantics) into its slot of
 * every learner's mailbox, waits until every learner's slot of this call has landed in
 * its own mailbox, and adds them in learner order (bitwise identical on every learner).
 *   partials      double[VT_P_COUNT] device, 8-byte aligned: this learner's partials
 *   mailboxes     host array of num_learners device pointers (16-byte aligned): learner
 *                 j's mailbox of vtrace_partials_mailbox_bytes(num_learners) bytes,
 *                 zero-initialised once, reachable from this GPU (peer-mapped, e.g.
 *                 symmetric memory over NVLink); mailboxes[self] is this learner's own
 *   num_learners  1..16;  self  0..num_learners-1
 *   counter       device uint64, zero-initialised once: this learner's call count
 *   out           double[VT_P_COUNT] device: the sum over learners (may alias partials)
 * Every learner must make the same sequence of calls; a learner that does not call
 * leaves the others waiting inside the kernel (as with any collective) -- for at most
 * 20 s, after which the missing learner's terms read as NaN (no hang).  Errors:
 * VT_ERR_INVALID_ARG (NULL pointer, num_learners or self out of range),
 * VT_ERR_ALIGNMENT, VT_ERR_DEVICE, VT_ERR_CUDA.  One launch on `stream`; capturable. */
size_t vtrace_partials_mailbox_bytes(int32_t num_learners);
vt_status vtrace_partials_allreduce(const double* partials, double* const* mailboxes,
                                   int32_t num_learners, int32_t self, uint64_t* counter,
                                   double* out, vt_stream_t stream);

/* The same sum for `batch` steps at once: partials[m] (host array of device pointers,
 * 8-byte aligned) is step m's double[VT_P_COUNT], replaced in place by the sum over the
 * learners.  One launch per `batch` steps: in a CUDA graph the side stream's per-step launch
 * costs the learners' kernel chain ~2.5 us a step at N = 4.  Mailboxes
 * of vtrace_partials_mailbox_bytes_batched(num_learners, batch_max) bytes (batch_max 1..32),
 * zero-initialised once; every call passes that batch_max and a batch of 1..batch_max steps;
 * every learner makes the same sequence of calls with the same batch sizes; a mailbox serves
 * one such sequence.  Errors as vtrace_partials_allreduce (batch or batch_max out of range:
 * VT_ERR_INVALID_ARG). */
size_t vtrace_partials_mailbox_bytes_batched(int32_t num_learners, int32_t batch_max);
vt_status vtrace_partials_allreduce_batched(double* const* partials, int32_t batch,
                                           int32_t batch_max, double* const* mailboxes,
                                           int32_t num_learners, int32_t self, uint64_t* counter,
                                           vt_stream_t stream);

/* ---- NEXT #3, first half: the output layer in front of the path ----
 * [z^pi | V] = h W + b over all M = T*B time-folded steps (time folded into the
 * batch; Fig. 3: linear policy and baseline heads on the LSTM output; DESIGN.md
 * reading r12), on the tcgen05 tensor cores (bf16 in, fp32 accumulate, fp32 out).
 *   M           rows = T*B (time-major, row t*B + b); M = 0 is a no-op
 *   H           hidden width: 64, 128, 192 or 256
 *   A           actions, 1 <= A <= 31 (A + 1 <= 32 head columns)
 *   hidden      h   [M, H]   bf16 device, row-major, 16-byte aligned
 *   w_t         W^T [A+1, H] bf16 device, row j = column j of W (rows 0..A-1 the policy
 *               logits, row A the baseline), 16-byte aligned
 *   bias        b   [A+1]    fp32 device, or NULL (no bias)
 *   logits_out  z^pi [M, A]  fp32 device (the layout vtrace_loss_and_grad reads)
 *   values_out  V    [M]     fp32 device
 * Outputs must not overlap the inputs.  Caller owns every buffer.  Errors: VT_ERR_SHAPE
 * (M, H or A out of range), VT_ERR_INVALID_ARG (NULL array), VT_ERR_ALIGNMENT,
 * VT_ERR_DEVICE, VT_ERR_CUDA.  One persistent launch on `stream`; deterministic (fixed
 * accumulation order); capturable in a CUDA graph. */
vt_status vtrace_output_layer(int64_t M, int32_t H, int32_t A, const void* hidden,
                              const void* w_t, const float* bias, float* logits_out,
                              float* values_out, vt_stream_t stream);

/* ---- NEXT #3, second half: the head fused with the whole path and its backward ----
 * One call = the learner's output layer over all T*B folded steps (Fig. 3:
 * [z^pi | V] = h W + b, reading r12), the V-trace targets, loss and gradients of
 * Section 4 (summed over the batch P:789) as the GEMM's
 * epilogue -- z^pi and V never reach HBM -- and the head's backward on the same tile:
 *   dZ = [dL/dz^pi | dL/dV]  (the vtrace_loss_and_grad gradients of that z^pi and V)
 *   grad_hidden = dZ W^T,  grad_w_t = dZ^T h  (= (h^T dZ)^T),  grad_bias = sum_rows dZ.
 *   T, B        unroll length and trajectories; B a multiple of 4
 *   H, A        hidden width 128 or 256; actions A in {3, 4, 6, 9, 18}
 *   hidden      h [T][B][H] bf16 device (time-major, row t*B + b), 16-byte aligned
 *   w_t         W^T [A+1][H] bf16 device (rows 0..A-1 the policy logits, row A the baseline)
 *   bias        b [A+1] fp32 device, or NULL
 *   behaviour_logits  z^mu [T][B][A] fp32 device (the actors' policy)
 *   actions, discounts, rewards  [T][B] (int32 / fp32 / fp32), bootstrap_value [B] fp32
 *               (as vtrace_loss_and_grad; 16-byte aligned except bootstrap_value)
 *   params, weights   as vtrace_loss_and_grad (behaviour_log_probs must be 0;
 *               overlap_previous, kernel and sm_budget are ignored)
 * Outputs (caller-owned, device): grad_hidden [T][B][H] bf16 (round-to-nearest-even of
 *   the fp32 product of dZ, carried as bf16 hi + lo, with W), grad_w_t [A+1][H] fp32,
 *   grad_bias [A+1] fp32, partials [VT_P_COUNT] double (as vtrace_loss_and_grad).
 * Precision: z^pi, V are fp32 tensor-core accumulations of the bf16 h and W; the path
 * then runs as in vtrace_loss_and_grad with fp32 logits; dZ enters both backward
 * products as two bf16 terms (hi + lo: 2^-17 relative), accumulated in fp32, the
 * per-CTA partials of grad_w_t / grad_bias added in fp64 in a fixed order
 * (deterministic).  workspace: vtrace_head_workspace_bytes(T, B, H, A) bytes, 256-byte
 * aligned, zero-initialised once (each call leaves it ready for the next; calls sharing
 * a workspace must be stream-ordered).  Errors: VT_ERR_INVALID_ARG (NULL pointer),
 * VT_ERR_SHAPE (T, B, H, A out of range), VT_ERR_PARAM, VT_ERR_ALIGNMENT,
 * VT_ERR_WORKSPACE, VT_ERR_DEVICE, VT_ERR_CUDA.  One cooperative launch on `stream` (a
 * persistent grid: the per-CTA partials are summed after an in-kernel grid barrier);
 * capturable. */
size_t vtrace_head_workspace_bytes(int64_t T, int64_t B, int32_t H, int32_t A);
vt_status vtrace_head_loss_and_grad(
    int64_t T, int64_t B, int32_t H, int32_t A, const void* hidden, const void* w_t,
    const float* bias, const float* behaviour_logits, const int32_t* actions,
    const float* discounts, const float* rewards, const float* bootstrap_value,
    const vt_vtrace_params* params, const vt_loss_weights* weights, void* grad_hidden,
    float* grad_w_t, float* grad_bias, double* partials, void* workspace,
    size_t workspace_bytes, vt_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* VTRACE_B200_H_ */
