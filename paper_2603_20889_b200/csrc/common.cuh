// Shared device helpers for the sm_100a kernels: mbarrier + bulk-copy (TMA engine) staging,
// warp-private panel stages, FP64 scalar helpers and the device status word.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "skinnyqr_b200.h"

namespace sqb {

constexpr int kWarp = 32;

// ---------------------------------------------------------------------------------------
// Device status word (one per context, lives in device memory, mirrored to the host on sync).
// word[0] = first error code raised (0 = none), word[1] = index attached to it,
// word[2] = non-finite-input flag (raised by the streaming kernels' fused validation).
// ---------------------------------------------------------------------------------------
struct StatusWord {
  int code;
  int index;
  int nonfinite;
  int reserved;
};

__device__ __forceinline__ void raise_status(StatusWord* st, int code, int index) {
  if (atomicCAS(&st->code, 0, code) == 0) st->index = index;
}

// ---------------------------------------------------------------------------------------
// mbarrier / bulk async copy (cp.async.bulk = the TMA engine's 1-D path; SASS: UBLKCP).
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_addr(bar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  }
}

// Generic-proxy reads of a stage must be ordered before the async proxy overwrites it.
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// One contiguous global -> shared bulk copy; completion is signalled on `bar` as transaction
// bytes.  dst, src and bytes must all be multiples of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// 16-byte asynchronous copy global -> shared issued per lane (LDGSTS, L2 only), tracked by per-thread commit
// groups.  A warp moves 512 bytes per instruction with per-lane addresses; cp.async.bulk takes uniform operands,
// so "one bulk copy per column" compiles to an election loop of ~9 instructions per column.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int PENDING>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(PENDING) : "memory");
}

// ---------------------------------------------------------------------------------------
// FP64 helpers
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ double shfl_xor_f64(double v, int mask) {
  return __shfl_xor_sync(0xffffffffu, v, mask);
}
__device__ __forceinline__ double shfl_idx_f64(double v, int src) {
  return __shfl_sync(0xffffffffu, v, src);
}

// Exponent-field test: true when x is Inf or NaN.  Integer pipe only (keeps the FP64 pipe free).
__device__ __forceinline__ uint32_t nonfinite_bits(double x) {
  return static_cast<uint32_t>(__double2hiint(x)) & 0x7fffffffu;
}
constexpr uint32_t kNonFiniteHi = 0x7ff00000u;

// Householder reflector scalars for the pencil [pivot; tail], sigma = |tail|^2, in the
// un-normalised form  H = I - gamma * u u^T,  u = [u0; tail],  u0 = pivot - beta,
// gamma = 1 / (norm * (norm + |pivot|)),  norm = sqrt(pivot^2 + sigma).  Same sign convention as the
// reference's make_reflector (tsqr.cpp:51-71): beta = -norm when pivot > 0 else +norm; sigma == 0
// gives the identity (gamma = u0 = 0, beta = pivot) so a zero column keeps an exact zero diagonal.
//
// The scalar chain is the serial bottleneck of every Householder kernel here, so it is short and
// BRANCH-FREE (one basic block per fold lets ptxas overlap it with the trailing updates): MUFU
// rsqrt seed (2^-22) -> one coupled Goldschmidt step (2^-43) -> residual correction (norm within
// 1 ulp); the reciprocal seed is taken from the first norm estimate, so that both MUFU results
// arrive while the Goldschmidt step runs, and finished with one cubic step on the exact
// d = a + norm*|pivot| (2^-63).  Inf/NaN propagate through it into R, which is how non-finite input
// is detected.  Guards: a = pivot^2 + sigma below ~1e-305 (the reciprocal would overflow; such a
// column is numerically zero) gives the identity; above ~1e290 (squares about to overflow - the
// reference's plain dot products are garbage there as well) beta is poisoned with NaN so that the
// call reports ArgumentError instead of a silently wrong R.  The exponent tests run on the integer
// pipe and, like the identity selects, sit off the path that leads to gamma.
struct Reflector {
  double beta, u0, gamma;
};
__device__ __forceinline__ Reflector make_reflector(double pivot, double sigma) {
  Reflector h;
  const double ap = fabs(pivot);
  const double a = fma(pivot, pivot, sigma);
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
  double g = a * y, hh = 0.5 * y;
  const double da = fma(g, ap, a);
  double z;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(z) : "d"(da));
  const double r = fma(-g, hh, 0.5);
  g = fma(g, r, g);
  hh = fma(hh, r, hh);
  const double norm = fma(fma(-g, g, a), hh, g);
  const double d = fma(norm, ap, a);
  const double e = fma(-d, z, 1.0);
  const double t = fma(e, e, e);
  const double inv = fma(z, t, z);
  const uint32_t ahi = static_cast<uint32_t>(__double2hiint(a));
  const bool live = (__double_as_longlong(sigma) << 1) != 0 && ahi >= 0x00b00000u;
  double beta = pivot > 0.0 ? -norm : norm;
  h.u0 = live ? pivot - beta : 0.0;
  h.gamma = live ? inv : 0.0;
  beta = ahi > 0x7c300000u ? __longlong_as_double(0x7ff8000000000000ll) : beta;
  h.beta = live ? beta : pivot;
  return h;
}

// Packed upper-triangular storage: column j holds rows 0..j at offset j(j+1)/2.
__host__ __device__ __forceinline__ int tri_index(int i, int j) { return j * (j + 1) / 2 + i; }
__host__ __device__ __forceinline__ int tri_size(int n) { return n * (n + 1) / 2; }

}  // namespace sqb
