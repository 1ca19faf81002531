// learner_update.cu -- the learner's parameter update after the network backward
// (SURVEY.md 8(f) NEXT #4): global-norm clip and RMSProp with momentum 0
// (P:838), TF form with epsilon inside the square root (DESIGN.md r9):
//     g' = g * c / max(||g||_2, c)            (c = max_global_norm; reading r10)
//     ms <- decay * ms + (1 - decay) * g'^2
//     theta <- theta - lr * g' / sqrt(ms + epsilon)
//
// One cooperative launch, one CTA per SM (co-resident by construction).  Up to
// 148 x 512 x 6 float4 (1.8 M parameters: both of the paper's networks)
// the arrays are register-resident (rmsprop_reg_kernel: every load issued before the
// exchange below, g read once); beyond that, two streaming passes:
//   phase 1  every CTA sums g^2 of its contiguous slice in fp64 (fixed strides, a
//            fixed tree) and publishes it as an epoch-tagged 16-byte record; every
//            CTA then reads all records in index order -> the same ||g|| bitwise in
//            every CTA, no second pass over memory and no atomics on the data path;
//   phase 2  the clip scale and the RMSProp update of the slice (its g re-read hits
//            L2: the slice was streamed moments ago); 1/sqrt by MUFU rsqrt.
// HBM traffic per parameter: g 4 B read, ms 4+4 B, theta 4+4 B = 20 B.
// Data-parallel learners: the caller all-reduces (SUM) the gradient first
// (paper_1802_01561_b200/learner.py, NCCL); every learner then applies the same
// update to its replica (reading r11).

#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <cstddef>

#include "vtrace.h"
#include "vtrace_kernels.cuh"

namespace vtb200 {

constexpr int RMS_THREADS = 512;
constexpr int RMS_MAX_CTAS = 1024;
constexpr size_t RMS_RECS_OFF = 256;
constexpr int RMS_MAX_GRADS = 8;  // gradients summed in the kernel (learners' buffers)

struct RmsHeader {  // workspace bytes [0, 16); vtrace_workspace_init zeroes them
  unsigned int epoch;   // calls completed (tags this call's records with epoch + 1)
  unsigned int ticket;  // CTAs done with phase 1 (the last one bumps the epoch)
  unsigned int done_ticket;  // CTAs done reading (learner sync: the last one signals)
  unsigned int go;           // learner sync: every learner ready for epoch go - 1 (CTA 0)
};
// vtrace_workspace_init zeroes the workspace and then sets the V-trace status word
// (WsHeader::status, bytes [16, 24)) to ~0: the RMSProp header must stay below it, or
// a field initialised to 0xFFFFFFFF would never match a ticket and the learners hang
static_assert(sizeof(RmsHeader) <= offsetof(vtb200::WsHeader, status),
              "RmsHeader overlaps the status word vtrace_workspace_init sets to ~0");

struct NormSlot {  // a learner's shard sum of squares and the call tag that published it
  double v;
  unsigned long long tag;
};

struct RmsArgs {
  long long n;
  float* theta;
  float* ms;
  const float* g[RMS_MAX_GRADS];  // g = g[0] + g[1] + ... (index order), ng of them
  int ng;
  unsigned int* flags[RMS_MAX_GRADS];  // learner sync: learner j's {ready, done} epoch words
  int self;                            // (flags[0] == NULL: no sync; see peers_ready)
  float lr, decay, eps, clip;
  double* norm_out;
  unsigned char* ws;
  // sharded learners (vtrace_rmsprop_step_sharded): this learner updates float4 units
  // [u0, u1) only, writes the new theta of that range into every learner's params, and the
  // learners add their shards' sums of squares through peer-mapped mailboxes
  long long u0, u1;                     // (non-sharded: 0, n / 4)
  int sharded;
  int tail_owner;                       // this learner updates the n % 4 tail
  float* peer_theta[RMS_MAX_GRADS];     // every learner's params (sharded)
  NormSlot* nmail[RMS_MAX_GRADS];       // every learner's norm mailbox [2][ng]
};

#ifdef RMS_TIMING
// timing build only (not part of the ABI): globaltimer stamps of CTA 0 / the last CTA per
// call (ring of 4096 calls): [start, ready published, peers ready seen, norm known,
// updates stored, done published, peers done seen]
__device__ unsigned long long rms_stamps[4096][8];
__device__ __forceinline__ unsigned long long rms_now() {
  unsigned long long g;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
  return g;
}
#define RMS_STAMP(e, k) (rms_stamps[(e) & 4095][k] = rms_now())
#else
#define RMS_STAMP(e, k) ((void)0)
#endif

// The gradient element i: the sum of the ng buffers in index order (fp32), so every
// learner that passes the same buffers in the same order gets the same bits.  The
// buffers may be other GPUs' memory (NVLink peer pointers, e.g. symmetric memory):
// the all-reduce of the learners' gradients then happens inside this kernel.
__device__ __forceinline__ float4 gsum4(const RmsArgs& a, long long i) {
  float4 v[RMS_MAX_GRADS];
#pragma unroll
  for (int j = 0; j < RMS_MAX_GRADS; ++j)
    if (j < a.ng) v[j] = __ldcs(reinterpret_cast<const float4*>(a.g[j]) + i);
  float4 s = v[0];
#pragma unroll
  for (int j = 1; j < RMS_MAX_GRADS; ++j) {
    if (j < a.ng) {
      s.x += v[j].x; s.y += v[j].y; s.z += v[j].z; s.w += v[j].w;
    }
  }
  return s;
}

__device__ __forceinline__ float gsum1(const RmsArgs& a, long long i) {
  float s = __ldcs(a.g[0] + i);
#pragma unroll
  for (int j = 1; j < RMS_MAX_GRADS; ++j)
    if (j < a.ng) s += __ldcs(a.g[j] + i);
  return s;
}

__device__ __forceinline__ void rms_update(float& th, float& m, float gv, float scale,
                                           const RmsArgs& a) {
  const float gg = gv * scale;
  m = fmaf(a.decay, m, (1.f - a.decay) * (gg * gg));
  th = fmaf(-a.lr * gg, rsqrtf(m + a.eps), th);  // MUFU rsqrt: rel. error < 2^-22
}

__device__ __forceinline__ unsigned int ld_acquire_sys(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(unsigned int* p, unsigned int v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned int rms_epoch(const RmsArgs& a) {
  return *reinterpret_cast<volatile unsigned int*>(&reinterpret_cast<RmsHeader*>(a.ws)->epoch);
}

// Learner sync (vtrace_rmsprop_step_learners), so the gradient all-reduce needs no
// separate barrier: call e of every learner publishes ready = e + 1 once its kernel
// has started (its own gradient buffer was completed by earlier work on its stream),
// and every CTA waits for all learners' ready >= e + 1 before reading their buffers.
__device__ __forceinline__ void peers_ready(const RmsArgs& a, unsigned int e) {
  if (a.flags[0] == nullptr) return;
  // (CTA 0 alone polls the other learners' flags over NVLink, then releases a local
  // "go" word that the other CTAs poll in L2: 148 remote pollers per GPU slowed the
  // gradient reads)
  RmsHeader* hdr = reinterpret_cast<RmsHeader*>(a.ws);
  if (threadIdx.x == 0) {
    if (blockIdx.x == 0) {
      RMS_STAMP(e, 0);
      // (no system fence before it: the buffers the peers read were written by earlier
      // kernels on this stream, complete before this one started, and peer reads over
      // NVLink are served by this GPU's memory system -- the fence cost ~1-1.5 us a call,
      // profiles/r2_update_n2_stamps.txt)
#ifdef RMS_SYSFENCE
      __threadfence_system();
#endif
      st_release_sys(a.flags[a.self], e + 1u);
      RMS_STAMP(e, 1);
      for (int j = 0; j < a.ng; ++j) {
        if (j == a.self) continue;
        while ((int)(ld_acquire_sys(a.flags[j]) - (e + 1u)) < 0) {
        }
      }
      RMS_STAMP(e, 2);
      st_release_u32(&hdr->go, e + 1u);
    } else {
      while ((int)(ld_acquire_u32(&hdr->go) - (e + 1u)) < 0) {
      }
    }
  }
  __syncthreads();
}

// ... and, when all of this learner's CTAs are done reading (the last CTA to finish),
// publishes done = e + 1 and returns only once every learner is done with call e, so
// the kernel ends (and the caller may refill its buffer) after all peers' reads.
__device__ __forceinline__ void peers_done(const RmsArgs& a, unsigned int e) {
  if (a.flags[0] == nullptr) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    RmsHeader* hdr = reinterpret_cast<RmsHeader*>(a.ws);
    // (cumulative after the CTA barrier: the CTA's stores -- peer stores of the sharded
    // form included -- before this learner's done)
    if (a.sharded) __threadfence_system();
    else __threadfence();
    const unsigned int prev = atomicAdd(&hdr->done_ticket, 1u);
    if (prev == gridDim.x - 1) {
      hdr->done_ticket = 0u;
      st_release_sys(a.flags[a.self] + 1, e + 1u);
      RMS_STAMP(e, 5);
      for (int j = 0; j < a.ng; ++j) {
        if (j == a.self) continue;
        while ((int)(ld_acquire_sys(a.flags[j] + 1) - (e + 1u)) < 0) {
        }
      }
      RMS_STAMP(e, 6);
    }
  }
}

// ||g||_2 of the whole gradient from every thread's fp64 partial sum `ss`: a fixed
// warp tree, the CTA's warps in order, then every CTA publishes its sum as an
// epoch-tagged 16-byte record and adds ALL CTAs' records in index order (lane l:
// l, l + 32, ..., then a fixed tree) -> the same norm, bitwise, in every CTA.
// Needs all CTAs co-resident (cooperative launch).
__device__ __forceinline__ double grid_norm(double ss, const RmsArgs& a, unsigned int epoch) {
  __shared__ double red[RMS_THREADS / 32];
  __shared__ double s_total;
  RmsHeader* hdr = reinterpret_cast<RmsHeader*>(a.ws);
  TagRec* recs = reinterpret_cast<TagRec*>(a.ws + RMS_RECS_OFF);
  const int S = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, w = tid >> 5;
  const unsigned long long tag = (unsigned long long)epoch + 1ull;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if (lane == 0) red[w] = ss;
  __syncthreads();
#if defined(RMS_ABLATE) && RMS_ABLATE == 1
  if (w == 0 && lane == 0) s_total = red[0];  // timing only: no grid exchange
  if (false) {
#else
  if (w == 0) {
#endif
    double x = lane < RMS_THREADS / 32 ? red[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) st_tag16(recs + cta, x, tag);  // (value, tag) in one 16-byte store
    // (records c = lane + 32 k, up to 8 a lane in flight per poll; same order)
    double tot = 0.0;
    for (int c0 = 0; c0 < S; c0 += 256) {
      double v[8];
      while (true) {
        bool ok = true;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int c = c0 + lane + 32 * k;
          unsigned long long t = tag;
          v[k] = 0.0;
          if (c < S) ld_tag16(recs + c, v[k], t);
          ok = ok && (t == tag);
        }
        if (ok) break;  // (spin: only warp 0 polls, the CTA's other warps wait;
      }                 //  a 100 ns sleep per poll measured 0.7 us slower)
#pragma unroll
      for (int k = 0; k < 8; ++k) tot += v[k];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if (lane == 0) s_total = tot;
  }
  __syncthreads();
  if (tid == 0) {
    // re-arm, off the CTA's critical path: every CTA has published (we read all
    // records), so every CTA has read the epoch; the last to get here starts the
    // next call's epoch
    const unsigned int prev = atomicAdd(&hdr->ticket, 1u);
    if (prev == (unsigned int)(S - 1)) {
      hdr->ticket = 0u;
      hdr->epoch = epoch + 1u;
    }
  }
  return s_total;
}

__device__ __forceinline__ unsigned long long ld_acquire_sys64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// ||g||_2 of the whole gradient: this learner's sum of squares (grid_norm), and, when the
// learners shard the parameters, the sum of every learner's shard sum in learner order
// (mailbox slots [parity][learner] in peer memory, value then tag with release
// semantics; every CTA reads its own learner's mailbox) -- bitwise the same everywhere.
__device__ __forceinline__ double global_norm(double ss, const RmsArgs& a, unsigned int epoch) {
  double tot = grid_norm(ss, a, epoch);
  if (a.sharded) {
    __shared__ double s_all;
    const unsigned long long tag = (unsigned long long)epoch + 1ull;
    const int par = (int)(tag & 1ull);
    if (threadIdx.x == 0) {
      if (blockIdx.x == 0) {
        for (int r = 0; r < a.ng; ++r) {
          NormSlot* d = a.nmail[r] + (par * a.ng + a.self);
          asm volatile("st.relaxed.sys.global.f64 [%0], %1;" ::"l"(&d->v), "d"(tot) : "memory");
          asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(&d->tag), "l"(tag) : "memory");
        }
      }
      double x = 0.0;
      const NormSlot* own = a.nmail[a.self] + par * a.ng;
      for (int r = 0; r < a.ng; ++r) {
        while (ld_acquire_sys64(&own[r].tag) != tag) {
        }
        double v;
        asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(&own[r].v) : "memory");
        x += v;
      }
      s_all = x;
    }
    __syncthreads();
    tot = s_all;
  }
  const double norm = sqrt(tot);
  if (blockIdx.x == 0 && threadIdx.x == 0 && a.norm_out) *a.norm_out = norm;
  return norm;
}

// Register-resident form (16-byte-aligned arrays, n <= S * RMS_THREADS * 4 V, V <= 6): each
// thread owns float4 units gt, gt + G, ..., gt + (V-1) G (G = threads in the grid,
// coalesced) of g, theta and ms; every load is issued before the norm exchange, so
// the parameter and mean-square reads overlap it, and g is read once.
template <int V>
__global__ void __launch_bounds__(RMS_THREADS, 1) rmsprop_reg_kernel(const RmsArgs a) {
  const int tid = threadIdx.x;
  const int G = gridDim.x * RMS_THREADS;  // (32-bit: units <= 148 x 512 x 6 here)
  const int gt = blockIdx.x * RMS_THREADS + tid;
  // this learner's float4 units [u0, u1) (all of them unless the learners shard)
  const int units = (int)(a.u1 - a.u0);
  float4* t4 = reinterpret_cast<float4*>(a.theta) + a.u0;
  float4* m4 = reinterpret_cast<float4*>(a.ms) + a.u0;
  const unsigned int e = rms_epoch(a);
  peers_ready(a, e);
  float4 gv[V], th[V], m[V];
  // g alone first: the norm needs only g; theta and ms are requested once this
  // thread's g has arrived (below), so the whole grid's g is not queued behind them
  // in DRAM and the norm exchange overlaps the theta / ms stream
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const int i = gt + k * G;
    gv[k] = i < units ? gsum4(a, a.u0 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  // the n % 4 tail: the grid's last thread (of the learner that owns it)
  const long long tail0 = (a.n / 4) * 4;
  const bool tail = a.tail_owner && gt == G - 1 && tail0 < a.n;
  float tg[3] = {0.f, 0.f, 0.f};
  if (tail)
    for (long long i = tail0; i < a.n; ++i) tg[i - tail0] = gsum1(a, i);
  double ss = 0.0;
#pragma unroll
  for (int k = 0; k < V; ++k) {
    ss = fma((double)gv[k].x, (double)gv[k].x, ss);
    ss = fma((double)gv[k].y, (double)gv[k].y, ss);
    ss = fma((double)gv[k].z, (double)gv[k].z, ss);
    ss = fma((double)gv[k].w, (double)gv[k].w, ss);
  }
  for (int k = 0; k < 3; ++k) ss = fma((double)tg[k], (double)tg[k], ss);
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const int i = gt + k * G;
    if (i < units) {
      th[k] = __ldcs(t4 + i);
      m[k] = __ldcs(m4 + i);
    }
  }
  const double norm = global_norm(ss, a, e);
  if (blockIdx.x == 0 && tid == 0) RMS_STAMP(e, 3);
  const float scale =
      (a.clip > 0.f && norm > (double)a.clip) ? (float)((double)a.clip / norm) : 1.f;
#pragma unroll
  for (int k = 0; k < V; ++k) {
    const int i = gt + k * G;
    if (i < units) {
      rms_update(th[k].x, m[k].x, gv[k].x, scale, a);
      rms_update(th[k].y, m[k].y, gv[k].y, scale, a);
      rms_update(th[k].z, m[k].z, gv[k].z, scale, a);
      rms_update(th[k].w, m[k].w, gv[k].w, scale, a);
#if defined(RMS_ABLATE) && RMS_ABLATE == 2
      if (th[k].x == 12345.f) {  // timing only: no stores
#else
      {
#endif
        __stcs(m4 + i, m[k]);
        if (a.sharded) {  // the new theta into every learner's replica (NVLink stores)
#pragma unroll
          for (int j = 0; j < RMS_MAX_GRADS; ++j)
            if (j < a.ng) reinterpret_cast<float4*>(a.peer_theta[j])[a.u0 + i] = th[k];
        } else {
          __stcs(t4 + i, th[k]);
        }
      }
    }
  }
  if (tail) {
    for (long long i = tail0; i < a.n; ++i) {
      float t = a.theta[i], mm = a.ms[i];
      rms_update(t, mm, tg[i - tail0], scale, a);
      a.ms[i] = mm;
      if (a.sharded) {
        for (int j = 0; j < a.ng; ++j) a.peer_theta[j][i] = t;
      } else {
        a.theta[i] = t;
      }
    }
  }
  if (blockIdx.x == 0 && tid == 0) RMS_STAMP(e, 4);
  peers_done(a, e);
}

// The push half of a push-based gradient all-gather: slot `self` of every learner's receive
// buffer <- this learner's gradient (float4 stores, NVLink for the peers), then a system-scope
// fence by every thread so that the next kernel's ready flag follows the pushed data.
struct PushArgs {
  const float4* g;
  float4* dst[RMS_MAX_GRADS];  // recv[r] + self * n, as float4
  int ng;
  long long units;
};

__global__ void __launch_bounds__(RMS_THREADS) grad_push_kernel(const PushArgs a) {
  const long long stride = (long long)gridDim.x * RMS_THREADS;
  for (long long i = (long long)blockIdx.x * RMS_THREADS + threadIdx.x; i < a.units; i += stride) {
    const float4 v = __ldcs(a.g + i);
#pragma unroll
    for (int r = 0; r < RMS_MAX_GRADS; ++r)
      if (r < a.ng) a.dst[r][i] = v;
  }
  __threadfence_system();
}

template <bool VEC>
__global__ void __launch_bounds__(RMS_THREADS, 1) rmsprop_kernel(const RmsArgs a) {
  const int S = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
  // the CTA's slice [lo, hi) in units of float4 (VEC) or floats; the n % 4 tail of
  // the vector path belongs to the last CTA
  const long long units = VEC ? a.n / 4 : a.n;
  const long long per = (units + S - 1) / S;
  const long long lo = min(units, (long long)cta * per), hi = min(units, lo + per);
  const long long tail0 = VEC ? units * 4 : a.n;
  const bool has_tail = VEC && cta == S - 1;
  const unsigned int e = rms_epoch(a);
  peers_ready(a, e);

  // ---- phase 1: sum of squares (fp64; "global gradient norm") ----
  double ss = 0.0;
  if constexpr (VEC) {
#pragma unroll 4
    for (long long i = lo + tid; i < hi; i += RMS_THREADS) {
      const float4 v = gsum4(a, i);
      ss = fma((double)v.x, (double)v.x, ss);
      ss = fma((double)v.y, (double)v.y, ss);
      ss = fma((double)v.z, (double)v.z, ss);
      ss = fma((double)v.w, (double)v.w, ss);
    }
  } else {
    for (long long i = lo + tid; i < hi; i += RMS_THREADS) {
      const double v = (double)gsum1(a, i);
      ss = fma(v, v, ss);
    }
  }
  if (has_tail) {
    for (long long i = tail0 + tid; i < a.n; i += RMS_THREADS) {
      const double v = (double)gsum1(a, i);
      ss = fma(v, v, ss);
    }
  }
  const double norm = global_norm(ss, a, e);
  // clip scale c / max(||g||, c) in fp64 (reading r10); 1 when disabled
  const float scale =
      (a.clip > 0.f && norm > (double)a.clip) ? (float)((double)a.clip / norm) : 1.f;

  // ---- phase 2: RMSProp, momentum 0 ----
  if constexpr (VEC) {
    float4* t4 = reinterpret_cast<float4*>(a.theta);
    float4* m4 = reinterpret_cast<float4*>(a.ms);
#pragma unroll 2
    for (long long i = lo + tid; i < hi; i += RMS_THREADS) {
      const float4 gv = gsum4(a, i);
      float4 th = __ldcs(t4 + i), m = __ldcs(m4 + i);
      rms_update(th.x, m.x, gv.x, scale, a);
      rms_update(th.y, m.y, gv.y, scale, a);
      rms_update(th.z, m.z, gv.z, scale, a);
      rms_update(th.w, m.w, gv.w, scale, a);
      __stcs(t4 + i, th);
      __stcs(m4 + i, m);
    }
  } else {
    for (long long i = lo + tid; i < hi; i += RMS_THREADS) {
      float th = a.theta[i], m = a.ms[i];
      rms_update(th, m, gsum1(a, i), scale, a);
      a.theta[i] = th;
      a.ms[i] = m;
    }
  }
  if (has_tail) {
    for (long long i = tail0 + tid; i < a.n; i += RMS_THREADS) {
      float th = a.theta[i], m = a.ms[i];
      rms_update(th, m, gsum1(a, i), scale, a);
      a.theta[i] = th;
      a.ms[i] = m;
    }
  }
  peers_done(a, e);
}

static int rms_num_sms() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  return n;
}

static bool al(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

}  // namespace vtb200

using namespace vtb200;

extern "C" {

#ifdef RMS_TIMING
int vtrace_debug_rms_stamps(unsigned long long* host) {  // timing build only
  return (int)cudaMemcpyFromSymbol(host, rms_stamps, sizeof(unsigned long long) * 8 * 4096);
}
#endif

size_t vtrace_rmsprop_workspace_bytes(int64_t n) {
  if (n < 0) return 0;
  return RMS_RECS_OFF + (size_t)RMS_MAX_CTAS * sizeof(TagRec);
}

}  // extern "C"

static vt_status rmsprop_impl(int64_t n, float* params, float* mean_square,
                              const float* const* grads, int ng, uint32_t* const* flags,
                              int self, const vt_rmsprop_params* prm, double* global_norm_out,
                              void* workspace, size_t workspace_bytes, vt_stream_t stream,
                              float* const* peer_params = nullptr,
                              double* const* norm_mailboxes = nullptr) {
  if (!prm || !grads || ng < 1 || ng > RMS_MAX_GRADS) return VT_ERR_INVALID_ARG;
  const bool sharded = peer_params != nullptr;
  if (sharded) {
    if (!flags || !norm_mailboxes) return VT_ERR_INVALID_ARG;
    for (int j = 0; j < ng; ++j) {
      if (!peer_params[j] || !norm_mailboxes[j]) return VT_ERR_INVALID_ARG;
      if (!al(peer_params[j], 16) || !al(norm_mailboxes[j], 16)) return VT_ERR_ALIGNMENT;
    }
    if (self >= 0 && self < ng && peer_params[self] != params) return VT_ERR_INVALID_ARG;
  }
  if (flags) {
    if (self < 0 || self >= ng) return VT_ERR_INVALID_ARG;
    for (int j = 0; j < ng; ++j)
      if (!flags[j]) return VT_ERR_INVALID_ARG;
      else if (!al(flags[j], 8)) return VT_ERR_ALIGNMENT;
  }
  bool null_grad = false, g4 = true, g16 = true;
  for (int j = 0; j < ng; ++j) {
    null_grad = null_grad || !grads[j];
    g4 = g4 && al(grads[j], 4);
    g16 = g16 && al(grads[j], 16);
  }
  if (n > 0 && (!params || !mean_square || null_grad)) return VT_ERR_INVALID_ARG;
  if (n < 0) return VT_ERR_SHAPE;
  const float lr = prm->learning_rate, decay = prm->decay, eps = prm->epsilon,
              clip = prm->max_global_norm;
  if (!(lr > 0.f) || !isfinite(lr) || !(decay >= 0.f && decay < 1.f) || !(eps > 0.f) ||
      !isfinite(eps) || !(clip >= 0.f) || !isfinite(clip))
    return VT_ERR_PARAM;
  if (!al(params, 4) || !al(mean_square, 4) || !g4 ||
      (global_norm_out && !al(global_norm_out, 8)))
    return VT_ERR_ALIGNMENT;
  if (!workspace || !al(workspace, 256) || workspace_bytes < vtrace_rmsprop_workspace_bytes(n))
    return VT_ERR_WORKSPACE;
  int dev = 0, maj = 0, mnr = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&maj, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&mnr, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess)
    return VT_ERR_CUDA;
  if (!(maj == 10 && mnr == 0)) return VT_ERR_DEVICE;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (n == 0) {  // nothing to update; the norm of an empty gradient is 0
    if (global_norm_out && cudaMemsetAsync(global_norm_out, 0, sizeof(double), st) != cudaSuccess)
      return VT_ERR_CUDA;
    return VT_OK;
  }
  const bool vec = al(params, 16) && al(mean_square, 16) && g16;
  const int sms = rms_num_sms();
  if (sms <= 0) return VT_ERR_CUDA;
  RmsArgs a;
  a.n = n; a.theta = params; a.ms = mean_square;
  for (int j = 0; j < RMS_MAX_GRADS; ++j) {
    a.g[j] = grads[j < ng ? j : 0];
    a.flags[j] = flags ? reinterpret_cast<unsigned int*>(flags[j < ng ? j : 0]) : nullptr;
  }
  a.ng = ng;
  a.self = flags ? self : 0;
  a.sharded = sharded ? 1 : 0;
  a.u0 = 0;
  a.u1 = n / 4;
  a.tail_owner = 1;
  for (int j = 0; j < RMS_MAX_GRADS; ++j) {
    a.peer_theta[j] = sharded ? peer_params[j < ng ? j : 0] : nullptr;
    a.nmail[j] = sharded ? reinterpret_cast<NormSlot*>(norm_mailboxes[j < ng ? j : 0]) : nullptr;
  }
  if (sharded) {  // learner self's float4 units: an equal split in learner order
    const long long U = n / 4;
    a.u0 = U * self / ng;
    a.u1 = U * (self + 1) / ng;
    a.tail_owner = self == ng - 1;
  }
  a.lr = lr; a.decay = decay; a.eps = eps; a.clip = clip;
  a.norm_out = global_norm_out;
  a.ws = static_cast<unsigned char*>(workspace);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (norm exchange)
  attr[0].val.cooperative = 1;  // (measured: no cost over a plain launch)
#ifdef RMS_NO_COOP
  attr[0].val.cooperative = 0;  // A/B only
#endif
  auto launch = [&](auto kern, int grid) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(RMS_THREADS);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a) == cudaSuccess ? VT_OK : VT_ERR_CUDA;
  };
  if (sharded && !vec) return VT_ERR_ALIGNMENT;  // (the sharded form is vectorised)
  if (vec) {
    // register-resident (one CTA per SM, up to 128 registers a thread): the smallest
    // V (float4 per thread per array) that holds n on the CTAs n can occupy
    const long long units = std::max(a.u1 - a.u0, 1LL), cap = (long long)sms * RMS_THREADS;
    const int Vs[4] = {1, 2, 4, 6};
    for (int V : Vs) {
      if (units > cap * V) continue;
      // every SM that has a thread's worth of units (the grid's threads stride the
      // units, so some threads own V float4 and some V - 1)
      const long long need = (std::max(units, 1LL) + RMS_THREADS - 1) / RMS_THREADS;
      const int S = (int)std::min<long long>(need, std::min(sms, RMS_MAX_CTAS));
      if (units > (long long)S * RMS_THREADS * V) continue;
      switch (V) {
        case 1: return launch(rmsprop_reg_kernel<1>, S);
        case 2: return launch(rmsprop_reg_kernel<2>, S);
        case 4: return launch(rmsprop_reg_kernel<4>, S);
        default: return launch(rmsprop_reg_kernel<6>, S);
      }
    }
  }
  if (sharded) return VT_ERR_SHAPE;  // (a shard beyond the register-resident capacity)
  // streaming form: one CTA per SM, at least 4 units per thread before a CTA is added
  const long long units = vec ? n / 4 : n;
  long long want = (units + (long long)RMS_THREADS * 4 - 1) / ((long long)RMS_THREADS * 4);
  const int S = (int)std::max(1LL, std::min<long long>(want, std::min(sms, RMS_MAX_CTAS)));
  return vec ? launch(rmsprop_kernel<true>, S) : launch(rmsprop_kernel<false>, S);
}

extern "C" {

vt_status vtrace_rmsprop_step(int64_t n, float* params, float* mean_square, const float* grads,
                              const vt_rmsprop_params* prm, double* global_norm_out,
                              void* workspace, size_t workspace_bytes, vt_stream_t stream) {
  const float* g[1] = {grads};
  return rmsprop_impl(n, params, mean_square, g, 1, nullptr, 0, prm, global_norm_out, workspace,
                      workspace_bytes, stream);
}

vt_status vtrace_rmsprop_step_multi(int64_t n, float* params, float* mean_square,
                                    const float* const* grads, int32_t num_grads,
                                    const vt_rmsprop_params* prm, double* global_norm_out,
                                    void* workspace, size_t workspace_bytes,
                                    vt_stream_t stream) {
  return rmsprop_impl(n, params, mean_square, grads, num_grads, nullptr, 0, prm, global_norm_out,
                      workspace, workspace_bytes, stream);
}

vt_status vtrace_rmsprop_step_learners(int64_t n, float* params, float* mean_square,
                                       const float* const* grads, uint32_t* const* flags,
                                       int32_t num_learners, int32_t self,
                                       const vt_rmsprop_params* prm, double* global_norm_out,
                                       void* workspace, size_t workspace_bytes,
                                       vt_stream_t stream) {
  if (!flags) return VT_ERR_INVALID_ARG;
  return rmsprop_impl(n, params, mean_square, grads, num_learners, flags, self, prm,
                      global_norm_out, workspace, workspace_bytes, stream);
}

vt_status vtrace_grad_push(const float* grad, float* const* recv, int32_t num_learners,
                           int32_t self, int64_t n, vt_stream_t stream) {
  if (!grad || !recv) return VT_ERR_INVALID_ARG;
  if (num_learners < 1 || num_learners > RMS_MAX_GRADS || self < 0 || self >= num_learners)
    return VT_ERR_INVALID_ARG;
  if (n < 0 || n % 4) return VT_ERR_SHAPE;
  if (!al(grad, 16)) return VT_ERR_ALIGNMENT;
  PushArgs a = {};
  a.g = reinterpret_cast<const float4*>(grad);
  a.ng = num_learners;
  a.units = n / 4;
  for (int r = 0; r < RMS_MAX_GRADS; ++r) {
    float* base = recv[r < num_learners ? r : 0];
    if (!base) return VT_ERR_INVALID_ARG;
    if (!al(base, 16)) return VT_ERR_ALIGNMENT;
    a.dst[r] = reinterpret_cast<float4*>(base + (size_t)self * (size_t)n);
  }
  int dev = 0, maj = 0, mnr = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&maj, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&mnr, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess)
    return VT_ERR_CUDA;
  if (!(maj == 10 && mnr == 0)) return VT_ERR_DEVICE;
  if (n == 0) return VT_OK;
  const int sms = rms_num_sms();
  if (sms <= 0) return VT_ERR_CUDA;
  const long long want = (a.units + RMS_THREADS - 1) / RMS_THREADS;
  const int grid = (int)std::max(1LL, std::min<long long>(want, 4LL * sms));
  grad_push_kernel<<<grid, RMS_THREADS, 0, reinterpret_cast<cudaStream_t>(stream)>>>(a);
  return cudaGetLastError() == cudaSuccess ? VT_OK : VT_ERR_CUDA;
}

size_t vtrace_rmsprop_norm_mailbox_bytes(int32_t num_learners) {
  if (num_learners < 1 || num_learners > RMS_MAX_GRADS) return 0;
  return (size_t)2 * num_learners * sizeof(NormSlot);
}

vt_status vtrace_rmsprop_step_sharded(int64_t n, float* const* params, float* mean_square,
                                      const float* const* grads, uint32_t* const* flags,
                                      double* const* norm_mailboxes, int32_t num_learners,
                                      int32_t self, const vt_rmsprop_params* prm,
                                      double* global_norm_out, void* workspace,
                                      size_t workspace_bytes, vt_stream_t stream) {
  if (!params || !flags || !norm_mailboxes) return VT_ERR_INVALID_ARG;
  if (num_learners < 1 || num_learners > RMS_MAX_GRADS || self < 0 || self >= num_learners)
    return VT_ERR_INVALID_ARG;
  return rmsprop_impl(n, params[self], mean_square, grads, num_learners, flags, self, prm,
                      global_norm_out, workspace, workspace_bytes, stream, params,
                      norm_mailboxes);
}

}  // extern "C"
