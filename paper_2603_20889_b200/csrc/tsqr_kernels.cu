// Q-less TSQR streaming kernels (sm_100a).
//
//   tsqr_warp_kernel<NB>  - universal kernel, n <= 8*NB <= 64.  One CTA per plan block
//                           (PanelPlan::block_begin/end, reference include/skinnyqr/plan.hpp:24-37),
//                           every warp streams its own panels through a private TMA-fed stage
//                           and folds them into a private triangle (tsqr_warp.cuh); the CTA's
//                           warps are then combined and one triangle per CTA is written to Y
//                           exactly where tsqr_stage1 puts it (reference src/tsqr.cpp:168-184).
//                           The same kernel, launched on Y, is the inter-CTA combine
//                           (reference stage 2, tsqr.cpp:193-195) and applies sign_normalize
//                           (reference src/types.cpp:8-14) when `finalize` is set.
#include "kernels.h"

namespace sqb {

template <int NB>
__global__ void __launch_bounds__(WarpLayout<NB>::NW * kWarp, 1)
    tsqr_warp_kernel(const TsqrParams prm) {
  using L = WarpLayout<NB>;
  constexpr int RL = L::RL, P = L::P, PP = L::PP, NW = L::NW;
  extern __shared__ __align__(128) double smem[];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const int n = prm.n;

  double* my = smem + static_cast<size_t>(warp) * L::kWarpDoubles;
  double* stage = my;
  double* tri = my + L::kStageDoubles;
  double* vbuf = tri + L::kTriDoubles;
  uint64_t* bar = reinterpret_cast<uint64_t*>(vbuf + P);

  // zero the triangle and the stage (padded columns / pad rows must read as zero forever)
  for (int i = lane; i < L::kStageDoubles + L::kTriDoubles + P; i += kWarp) my[i] = 0.0;
  if (lane == 0) mbar_init(bar, 1);
  mbar_fence_init();
  __syncwarp();

  const long long blk = blockIdx.x;
  const long long begin = min(blk * prm.rows_per_block, prm.m);
  const long long end = min((blk + 1) * prm.rows_per_block, prm.m);
  const long long rows = end - begin;
  const long long npanels = (rows + P - 1) / P;

  const bool aligned = view_bulk_aligned(prm.x, n, begin);
  uint32_t phase = 0;
  uint32_t nf = 0;
  auto issue = [&](long long pnl) -> bool {
    return issue_panel<P, PP>(prm.x, n, begin + pnl * P, end, aligned, stage, bar, lane);
  };

  double w[NB][RL];
  long long pnl = warp;
  bool async = false;
  if (pnl < npanels) async = issue(pnl);
  for (; pnl < npanels; pnl += NW) {
    if (async) {
      mbar_wait(bar, phase);
      phase ^= 1;
    }
    nf = max(nf, load_panel_regs<NB, RL, PP>(w, stage, g, q));
    __syncwarp();
    if (pnl + NW < npanels) async = issue(pnl + NW);
    factor_panel<NB, RL>(w, tri, vbuf, n, lane);
  }

  if (prm.check_finite) flag_nonfinite(nf, prm.status, lane);

  // ---- intra-CTA combine: warp 0 folds the other warps' triangles (as dense row panels) ----
  __syncthreads();
  if (warp != 0) return;
  const long long stacked = static_cast<long long>(NW - 1) * n;
  for (long long r0 = 0; r0 < stacked; r0 += P) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int col = 8 * b + g;
#pragma unroll
      for (int i = 0; i < RL; ++i) {
        const long long vr = r0 + panel_row(q, i);
        double val = 0.0;
        if (vr < stacked && col < n) {
          const int src = 1 + static_cast<int>(vr / n);
          const int row = static_cast<int>(vr % n);
          if (row <= col)
            val = smem[static_cast<size_t>(src) * L::kWarpDoubles + L::kStageDoubles +
                       tri_index(row, col)];
        }
        w[b][i] = val;
      }
    }
    factor_panel<NB, RL>(w, tri, vbuf, n, lane);
  }

  // ---- write the CTA's triangle: rows [blk*n, blk*n+n) of Y, full square with zeros below ----
  double* dst = prm.y + blk * n;
  for (int idx = lane; idx < n * n; idx += kWarp) {
    const int i = idx % n, j = idx / n;
    double val = 0.0;
    if (i <= j) {
      val = tri[tri_index(i, j)];
      if (prm.finalize && tri[tri_index(i, i)] < 0.0) val = -val;
    }
    dst[i + j * prm.ldy] = val;
  }
}

// ---------------------------------------------------------------------------------------------
// host-side launcher
// ---------------------------------------------------------------------------------------------
template <int NB>
static cudaError_t launch_nb(const TsqrParams& prm, long long num_blocks, cudaStream_t stream) {
  using L = WarpLayout<NB>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(tsqr_warp_kernel<NB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(L::kSmemBytes));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  tsqr_warp_kernel<NB><<<static_cast<unsigned>(num_blocks), L::NW * kWarp, L::kSmemBytes, stream>>>(prm);
  return cudaGetLastError();
}

cudaError_t launch_tsqr_warp(const TsqrParams& prm, long long num_blocks, cudaStream_t stream) {
  const int nb = (prm.n + 7) / 8;
  switch (nb) {
    case 1: return launch_nb<1>(prm, num_blocks, stream);
    case 2: return launch_nb<2>(prm, num_blocks, stream);
    case 3: return launch_nb<3>(prm, num_blocks, stream);
    case 4: return launch_nb<4>(prm, num_blocks, stream);
    case 5: return launch_nb<5>(prm, num_blocks, stream);
    case 6: return launch_nb<6>(prm, num_blocks, stream);
    case 7: return launch_nb<7>(prm, num_blocks, stream);
    case 8: return launch_nb<8>(prm, num_blocks, stream);
    default: return cudaErrorInvalidValue;
  }
}

int tsqr_warp_warps(int n) {
  switch ((n + 7) / 8) {
    case 1: return WarpLayout<1>::NW;
    case 2: return WarpLayout<2>::NW;
    case 3: return WarpLayout<3>::NW;
    case 4: return WarpLayout<4>::NW;
    case 5: return WarpLayout<5>::NW;
    case 6: return WarpLayout<6>::NW;
    case 7: return WarpLayout<7>::NW;
    default: return WarpLayout<8>::NW;
  }
}

int tsqr_warp_panel_rows(int n) {
  switch ((n + 7) / 8) {
    case 1: return WarpLayout<1>::P;
    case 2: return WarpLayout<2>::P;
    case 3: return WarpLayout<3>::P;
    case 4: return WarpLayout<4>::P;
    case 5: return WarpLayout<5>::P;
    case 6: return WarpLayout<6>::P;
    case 7: return WarpLayout<7>::P;
    default: return WarpLayout<8>::P;
  }
}

}  // namespace sqb
