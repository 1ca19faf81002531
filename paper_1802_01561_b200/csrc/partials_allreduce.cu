// SURVEY.md 8(a) row a13 over NVLink peer memory: the sum of the synchronous learners'
// partials (each learner computes the loss of its own trajectories, the
// losses add; summed loss) without a collective-library call.  One 32-thread
// kernel per step: learner `self` stores its 8 partials into its slot of every
// learner's mailbox (NVLink stores into peer memory, value then tag with release
// semantics), then waits until every learner's slot of this call has landed in its own
// mailbox and adds them in learner order (bitwise identical on every learner).
// See include/vtrace.h (vtrace_partials_allreduce) and DESIGN.md section 7.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "../../include/vtrace.h"

namespace vtpa {

constexpr int kMaxLearners = 16;

struct Slot {  // one partial: its value and the call tag that published it
  double v;
  unsigned long long tag;
};

struct Mailboxes {
  Slot* p[kMaxLearners];
};

__device__ __forceinline__ void st_relaxed_f64(double* p, double v) {
  asm volatile("st.relaxed.sys.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double ld_relaxed_f64(const double* p) {
  double v;
  asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}

constexpr unsigned long long kTimeoutNs = 20ull * 1000 * 1000 * 1000;

__device__ __forceinline__ unsigned long long now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Slots [parity][learner][k]: a learner can be at most one call ahead of another (call
// n + 1 cannot finish before every learner has published n + 1, i.e. finished n), so
// call n + 1 writes the other parity and never overwrites a slot still to be read.
__global__ void __launch_bounds__(32) partials_allreduce_kernel(const double* __restrict__ partials,
                                                                Mailboxes mb, int n, int self,
                                                                unsigned long long* counter,
                                                                double* out) {
  const int k = threadIdx.x;
  const unsigned long long tag = *reinterpret_cast<volatile unsigned long long*>(counter) + 1ull;
  const int par = (int)(tag & 1ull);
  double s = 0.0;
  if (k < VT_P_COUNT) {
    const double v = partials[k];
    for (int r = 0; r < n; ++r) {
      Slot* d = mb.p[r] + ((size_t)(par * n + self) * VT_P_COUNT + k);
      st_relaxed_f64(&d->v, v);
      st_release_u64(&d->tag, tag);  // orders the value before the tag
    }
    const Slot* own = mb.p[self] + (size_t)par * n * VT_P_COUNT + k;
    const unsigned long long t0 = now_ns();
    for (int r = 0; r < n; ++r) {
      const Slot* q = own + (size_t)r * VT_P_COUNT;
      bool late = false;
      while (ld_acquire_u64(&q->tag) != tag) {
        __nanosleep(20);
        if (now_ns() - t0 > kTimeoutNs) {  // a learner that never calls: NaN, not a hang
          late = true;
          break;
        }
      }
      s += late ? __longlong_as_double(0x7ff8000000000000ll) : ld_relaxed_f64(&q->v);
    }
  }
  __syncwarp();
  if (k < VT_P_COUNT) out[k] = s;
  if (k == 0) *reinterpret_cast<volatile unsigned long long*>(counter) = tag;
}

// The batched form: `batch` steps' partials in one call (thread t: step t / 8, partial t % 8);
// slots [parity][learner][step][k].  One call per `batch` steps keeps the side stream's
// per-step launches off the learners' kernel chain.
constexpr int kMaxBatch = 32;

struct PartialsPtrs {
  double* p[kMaxBatch];
};

__global__ void __launch_bounds__(256) partials_allreduce_batch_kernel(PartialsPtrs parts,
                                                                       int batch, int batch_max,
                                                                       Mailboxes mb, int n,
                                                                       int self,
                                                                       unsigned long long* counter) {
  const int t = threadIdx.x;
  const unsigned long long tag = *reinterpret_cast<volatile unsigned long long*>(counter) + 1ull;
  const int par = (int)(tag & 1ull);
  // (slots laid out for the mailbox's largest batch: a call's region of either parity is the
  // same whatever its own batch size, so calls of different sizes never overlap)
  const int per = batch_max * VT_P_COUNT;
  double s = 0.0;
  if (t < batch * VT_P_COUNT) {
    const double v = parts.p[t / VT_P_COUNT][t % VT_P_COUNT];
    for (int r = 0; r < n; ++r) {
      Slot* d = mb.p[r] + ((size_t)(par * n + self) * per + t);
      st_relaxed_f64(&d->v, v);
      st_release_u64(&d->tag, tag);
    }
    const Slot* own = mb.p[self] + (size_t)par * n * per + t;
    const unsigned long long t0 = now_ns();
    for (int r = 0; r < n; ++r) {
      const Slot* q = own + (size_t)r * per;
      bool late = false;
      while (ld_acquire_u64(&q->tag) != tag) {
        __nanosleep(20);
        if (now_ns() - t0 > kTimeoutNs) {
          late = true;
          break;
        }
      }
      s += late ? __longlong_as_double(0x7ff8000000000000ll) : ld_relaxed_f64(&q->v);
    }
  }
  __syncthreads();
  if (t < batch * VT_P_COUNT) parts.p[t / VT_P_COUNT][t % VT_P_COUNT] = s;
  if (t == 0) *reinterpret_cast<volatile unsigned long long*>(counter) = tag;
}

}  // namespace vtpa

extern "C" size_t vtrace_partials_mailbox_bytes_batched(int32_t num_learners, int32_t batch) {
  if (num_learners < 1 || num_learners > vtpa::kMaxLearners || batch < 1 || batch > vtpa::kMaxBatch)
    return 0;
  return (size_t)2 * (size_t)num_learners * (size_t)batch * VT_P_COUNT * sizeof(vtpa::Slot);
}

extern "C" vt_status vtrace_partials_allreduce_batched(double* const* partials, int32_t batch,
                                                       int32_t batch_max,
                                                       double* const* mailboxes,
                                                       int32_t num_learners, int32_t self,
                                                       uint64_t* counter, vt_stream_t stream) {
  using namespace vtpa;
  if (!partials || !mailboxes || !counter) return VT_ERR_INVALID_ARG;
  if (batch_max < 1 || batch_max > kMaxBatch || batch < 1 || batch > batch_max)
    return VT_ERR_INVALID_ARG;
  if (num_learners < 1 || num_learners > kMaxLearners || self < 0 || self >= num_learners)
    return VT_ERR_INVALID_ARG;
  if (reinterpret_cast<uintptr_t>(counter) & 7) return VT_ERR_ALIGNMENT;
  PartialsPtrs pp{};
  for (int m = 0; m < batch; ++m) {
    if (!partials[m]) return VT_ERR_INVALID_ARG;
    if (reinterpret_cast<uintptr_t>(partials[m]) & 7) return VT_ERR_ALIGNMENT;
    pp.p[m] = partials[m];
  }
  Mailboxes mb{};
  for (int r = 0; r < num_learners; ++r) {
    if (!mailboxes[r]) return VT_ERR_INVALID_ARG;
    if (reinterpret_cast<uintptr_t>(mailboxes[r]) & 15) return VT_ERR_ALIGNMENT;
    mb.p[r] = reinterpret_cast<Slot*>(mailboxes[r]);
  }
  const int threads = ((batch * VT_P_COUNT + 31) / 32) * 32;
  partials_allreduce_batch_kernel<<<1, threads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      pp, batch, batch_max, mb, num_learners, self,
      reinterpret_cast<unsigned long long*>(counter));
  return cudaGetLastError() == cudaSuccess ? VT_OK : VT_ERR_CUDA;
}

extern "C" size_t vtrace_partials_mailbox_bytes(int32_t num_learners) {
  if (num_learners < 1 || num_learners > vtpa::kMaxLearners) return 0;
  return (size_t)2 * (size_t)num_learners * VT_P_COUNT * sizeof(vtpa::Slot);
}

extern "C" vt_status vtrace_partials_allreduce(const double* partials, double* const* mailboxes,
                                               int32_t num_learners, int32_t self,
                                               uint64_t* counter, double* out,
                                               vt_stream_t stream) {
  using namespace vtpa;
  if (!partials || !mailboxes || !counter || !out) return VT_ERR_INVALID_ARG;
  if (num_learners < 1 || num_learners > kMaxLearners || self < 0 || self >= num_learners)
    return VT_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(partials) & 7) || (reinterpret_cast<uintptr_t>(out) & 7) ||
      (reinterpret_cast<uintptr_t>(counter) & 7))
    return VT_ERR_ALIGNMENT;
  Mailboxes mb{};
  for (int r = 0; r < num_learners; ++r) {
    if (!mailboxes[r]) return VT_ERR_INVALID_ARG;
    if (reinterpret_cast<uintptr_t>(mailboxes[r]) & 15) return VT_ERR_ALIGNMENT;
    mb.p[r] = reinterpret_cast<Slot*>(mailboxes[r]);
  }
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return VT_ERR_CUDA;
  if (dev < 0 || dev >= 64) return VT_ERR_DEVICE;
  static std::atomic<int> state[64];  // 0 unknown, 1 sm_100, 2 other
  if (state[dev].load(std::memory_order_relaxed) == 0) {
    int maj = 0, mnr = 0;
    if (cudaDeviceGetAttribute(&maj, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&mnr, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess)
      return VT_ERR_CUDA;
    state[dev].store((maj == 10 && mnr == 0) ? 1 : 2, std::memory_order_relaxed);
  }
  if (state[dev].load(std::memory_order_relaxed) != 1) return VT_ERR_DEVICE;
  partials_allreduce_kernel<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      partials, mb, num_learners, self, reinterpret_cast<unsigned long long*>(counter), out);
  return cudaGetLastError() == cudaSuccess ? VT_OK : VT_ERR_CUDA;
}
