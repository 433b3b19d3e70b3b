// Warp-private panel staging: every warp of a streaming CTA owns NS shared-memory stages that the
// TMA engine fills with bulk async copies (cp.async.bulk, one per column segment, completion on a
// warp-private mbarrier).  No __syncthreads anywhere in the streaming loops - warps run free.
//
// Reference analogue: TrapezoidalWorkspace::load_panel / the Gram workspace memcpy
// (reference src/tsqr.cpp:27-40, src/gram.cpp:57-68) - "bring a b-row panel of X on chip".
#pragma once

#include "common.cuh"

namespace sqb {

// Input matrix view: columns 0..n_main-1 come from base (leading dimension ld); an optional
// extra last column comes from `extra` (least squares: the [A rhs] pencil without assembling it,
// reference src/lstsq.cpp:24-26 copies instead).
struct MatView {
  const double* base;
  long long ld;
  const double* extra;
  int n_main;
  __device__ __forceinline__ const double* col(int j) const {
    return j < n_main ? base + static_cast<long long>(j) * ld : extra;
  }
};

// Stage pitch (doubles per column).  residue 8 (mod 16): the "two rows per lane" LDS.128 fragment
// pattern (address = col*PP + 8t + 2q) is bank-conflict free; residue 4: the transposed LDS.64
// fragment pattern (address = (4k+q)*PP + 8t + g) is.
constexpr int stage_pitch(int p, int residue) { return p + ((residue - (p % 16)) + 16) % 16; }

__device__ __forceinline__ bool view_bulk_aligned(const MatView& x, int n, long long begin) {
  bool ok = ((reinterpret_cast<uintptr_t>(x.base) & 15) == 0) && ((x.ld & 1) == 0) &&
            ((begin & 1) == 0);
  if (x.n_main < n) ok = ok && ((reinterpret_cast<uintptr_t>(x.extra) & 15) == 0);
  return ok;
}

// Fill one stage with rows [r0, min(r0+P, end)) of the n live columns.  Full, 16-byte aligned
// panels go through the async engine (returns true: wait on `bar`); ragged or unaligned panels
// are filled synchronously by the warp with zero padding (returns false).
// SWZ: column j starts 4 doubles later when bit 1 of j is set (stage_col_offset) - with a pitch == 8
// (mod 16) that makes BOTH fragment patterns above conflict-free in one stage.
template <int PP, bool SWZ>
__host__ __device__ __forceinline__ constexpr int stage_col_offset(int j) {
  return j * PP + (SWZ ? ((j & 2) << 1) : 0);
}

template <int P, int PP, bool SWZ = false>
__device__ __forceinline__ bool issue_panel(const MatView& x, int n, long long r0, long long end,
                                            bool aligned, double* stage, uint64_t* bar, int lane) {
  const long long left = end - r0;
  if (aligned && left >= P) {
    // lane 0 arms the barrier, then lane j issues the copy of column j: one UBLKCP per lane
    // instead of an n-iteration loop on a single lane.
    if (lane == 0) mbar_expect_tx(bar, static_cast<uint32_t>(n * P * sizeof(double)));
    __syncwarp();
    for (int j = lane; j < n; j += kWarp) {
      fence_async_smem();
      bulk_g2s(stage + stage_col_offset<PP, SWZ>(j), x.col(j) + r0, P * sizeof(double), bar);
    }
    return true;
  }
  const int live = static_cast<int>(left < P ? left : P);
  for (int j = 0; j < n; ++j) {
    const double* src = x.col(j) + r0;
    for (int r = lane; r < P; r += kWarp) stage[stage_col_offset<PP, SWZ>(j) + r] = r < live ? __ldg(src + r) : 0.0;
  }
  __syncwarp();
  return false;
}

// The same fill with per-lane 16-byte asynchronous copies (commit groups instead of an mbarrier): lane l takes
// the 16-byte chunks l, l + 32, ... of the panel, P / 2 chunks per column.  The caller commits one group per
// call (also when nothing was issued) and waits with cp_async_wait<NS - 1>() + __syncwarp().
template <int P, int PP, bool SWZ = false>
__device__ __forceinline__ void issue_panel_lanes(const MatView& x, int n, long long r0, long long end,
                                                  bool aligned, double* stage, int lane) {
  const long long left = end - r0;
  if (aligned && left >= P) {
    constexpr int CH = P / 2;
    const int total = n * CH;
    for (int c = lane; c < total; c += kWarp) {
      const int j = c / CH, r = c - j * CH;
      cp_async16(stage + stage_col_offset<PP, SWZ>(j) + 2 * r, x.col(j) + r0 + 2 * r);
    }
    return;
  }
  const int live = static_cast<int>(left < P ? left : P);
  for (int j = 0; j < n; ++j) {
    const double* src = x.col(j) + r0;
    for (int r = lane; r < P; r += kWarp) stage[stage_col_offset<PP, SWZ>(j) + r] = r < live ? __ldg(src + r) : 0.0;
  }
  __syncwarp();
}

// Running triangle of the TSQR kernels: packed ROW-major upper triangle of order npad; row c holds
// (c, c..npad-1).  row_base(c) + j addresses entry (c, j); consecutive rows differ by npad - c - 1,
// so a factorisation walks it with one running offset and no index multiplications.
__host__ __device__ __forceinline__ int row_base(int c, int npad) {
  return c * npad - (c * (c - 1)) / 2 - c;
}

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-DEVICE attribute: opt in once per device
// (a process may hold contexts on several GPUs), remembered in a per-kernel bit mask.
template <class Kernel>
inline cudaError_t opt_in_dynamic_smem(Kernel kernel, size_t bytes, unsigned long long* done_mask) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 64 && ((*done_mask >> dev) & 1ull)) return cudaSuccess;
  if (bytes > 48 * 1024) {
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
    if (e != cudaSuccess) return e;
  }
  if (dev < 64) *done_mask |= 1ull << dev;
  return cudaSuccess;
}

// Fused non-finite validation (replaces the reference's serial scans, src/types.cpp:40-48 and
// src/gram.cpp:96-102): an Inf/NaN anywhere in X makes the squared norm of its column - hence the
// diagonal of R or of the Gram matrix - non-finite, so testing the n x n result is enough.
__device__ __forceinline__ bool is_nonfinite(double x) { return nonfinite_bits(x) >= kNonFiniteHi; }

}  // namespace sqb
