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
#include <cstdlib>

#include "kernels.h"

namespace sqb {

template <int NB, int VAR>
__global__ void __launch_bounds__(WarpLayout<NB, VAR>::NW * kWarp, 1)
    tsqr_warp_kernel(const TsqrParams prm) {
  using L = WarpLayout<NB, VAR>;
  constexpr int RL = L::RL, P = L::P, PP = L::PP, NW = L::NW, NPAD = L::NPAD;
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
    load_panel_regs<NB, RL, PP>(w, stage, g, q);
    __syncwarp();
    if (pnl + NW < npanels) async = issue(pnl + NW);
    factor_panel<NB, RL>(w, tri, vbuf, n, lane);
  }

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
                       row_base(row, NPAD) + col];
        }
        w[b][i] = val;
      }
    }
    factor_panel<NB, RL>(w, tri, vbuf, n, lane);
  }

  // ---- write the CTA's triangle: rows [blk*n, blk*n+n) of Y, full square with zeros below ----
  double* dst = prm.y + blk * n;
  bool bad = false;
  for (int idx = lane; idx < n * n; idx += kWarp) {
    const int i = idx % n, j = idx / n;
    double val = 0.0;
    if (i <= j) {
      val = tri[row_base(i, NPAD) + j];
      bad = bad || is_nonfinite(val);
      if (prm.finalize && tri[row_base(i, NPAD) + i] < 0.0) val = -val;
    }
    dst[i + j * prm.ldy] = val;
  }
  if (prm.check_finite && bad) atomicExch(&prm.status->nonfinite, 1);
}

// ---------------------------------------------------------------------------------------------
// host-side launcher
// ---------------------------------------------------------------------------------------------
template <int NB, int VAR>
static cudaError_t launch_nb(const TsqrParams& prm, long long num_blocks, cudaStream_t stream) {
  using L = WarpLayout<NB, VAR>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(tsqr_warp_kernel<NB, VAR>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(L::kSmemBytes));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  tsqr_warp_kernel<NB, VAR>
      <<<static_cast<unsigned>(num_blocks), L::NW * kWarp, L::kSmemBytes, stream>>>(prm);
  return cudaGetLastError();
}

// Which tuning variant runs for a given column-block count (see WarpCfg).  SQB_TSQR_VARIANT
// (0/1) overrides the table - used by the tuning sweeps in tools/.
static int tsqr_variant(int nb) {
  static int forced = [] {
    const char* e = getenv("SQB_TSQR_VARIANT");
    return e ? atoi(e) : -1;
  }();
  if (forced == 0 || forced == 1) return forced;
  static const int table[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  return table[nb];
}

#define SQB_NB_SWITCH(EXPR0, EXPR1)                    \
  switch (nb) {                                        \
    case 1: return var ? EXPR1(1) : EXPR0(1);          \
    case 2: return var ? EXPR1(2) : EXPR0(2);          \
    case 3: return var ? EXPR1(3) : EXPR0(3);          \
    case 4: return var ? EXPR1(4) : EXPR0(4);          \
    case 5: return var ? EXPR1(5) : EXPR0(5);          \
    case 6: return var ? EXPR1(6) : EXPR0(6);          \
    case 7: return var ? EXPR1(7) : EXPR0(7);          \
    default: return var ? EXPR1(8) : EXPR0(8);         \
  }

cudaError_t launch_tsqr_warp(const TsqrParams& prm, long long num_blocks, cudaStream_t stream) {
  const int nb = (prm.n + 7) / 8;
  if (nb < 1 || nb > 8) return cudaErrorInvalidValue;
  const int var = tsqr_variant(nb);
#define L0(NBV) launch_nb<NBV, 0>(prm, num_blocks, stream)
#define L1(NBV) launch_nb<NBV, 1>(prm, num_blocks, stream)
  SQB_NB_SWITCH(L0, L1)
#undef L0
#undef L1
}

int tsqr_forced_kind() {
  static int v = [] {
    const char* e = getenv("SQB_TSQR_KERNEL");
    return e ? atoi(e) : -1;
  }();
  return v;
}

int tsqr_warp_warps(int n) {
  const int nb = (n + 7) / 8;
  const int var = tsqr_variant(nb);
#define W0(NBV) WarpLayout<NBV, 0>::NW
#define W1(NBV) WarpLayout<NBV, 1>::NW
  SQB_NB_SWITCH(W0, W1)
#undef W0
#undef W1
}

int tsqr_warp_panel_rows(int n) {
  const int nb = (n + 7) / 8;
  const int var = tsqr_variant(nb);
#define P0(NBV) WarpLayout<NBV, 0>::P
#define P1(NBV) WarpLayout<NBV, 1>::P
  SQB_NB_SWITCH(P0, P1)
#undef P0
#undef P1
}

}  // namespace sqb
