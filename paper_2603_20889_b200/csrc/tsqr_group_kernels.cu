// Lane-group Q-less Householder TSQR for 8 < n <= 64.
//
// Reference semantics: block_qless_qr_core / factor_trapezoidal / make_reflector
// (reference src/tsqr.cpp:51-158).  Generalises the thread-private kernel (tsqr_thread_kernels.cu):
// a GROUP of G adjacent lanes is one leaf of the TSQR tree.  It owns P rows per step and a private
// running triangle in shared memory; lane g of the group keeps columns g, g+G, g+2G, ... of those
// rows in registers.  Per reflector the only communication is the broadcast of the P-entry
// reflector column from its owner lane (P 64-bit shuffles inside the group): every dot product is
// lane-local, and every lane derives the reflector scalars redundantly from its own copy, so there
// are no cross-lane reductions, no barriers and no shared-memory broadcast in the streaming loop.
// Global loads are 128-bit (two adjacent rows), 32/G row pairs contiguous per column.
#include <cstdlib>
#include <type_traits>

#include "kernels.h"

namespace sqb {

namespace {

template <int B, int E, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

template <int NS, int G, int P>
struct GroupCfg {
  static constexpr int NPAD = NS * G;                    // columns incl. padding
  static constexpr int GW = 32 / G;                      // groups per warp
  static constexpr int kTri = NPAD * (NPAD + 1) / 2;
  // triangle stride == G (mod 16) doubles: the G*GW lanes of a half warp hit distinct banks
  static constexpr int TS = kTri + ((G - kTri % 16) + 16) % 16;
  static constexpr int kMaxGroups = (220 * 1024) / (TS * 8);
  static constexpr int kGroupsRaw = kMaxGroups * G >= 256 ? 256 / G : kMaxGroups;
  static constexpr int T = (kGroupsRaw * G) / 32 * 32;   // threads per CTA
  static constexpr int NG = T / G;                       // groups per CTA
  static constexpr int kChunk = GW * P;                  // rows a warp consumes per step
  static constexpr size_t kSmemBytes = sizeof(double) * TS * NG;
  static_assert(T >= 64, "too few threads");
  static_assert(P % 2 == 0, "row pairs");
};

// Fold the group's P x n register panel (w[slot][row], column = slot*G + g) into its triangle
// (packed row-major, row_base() from tsqr_warp.cuh).  Lanes whose column is already finished run
// the same instructions on values nobody reads again; only the R store is predicated.
template <int NS, int G, int P>
__device__ __forceinline__ void fold_group(double (&w)[NS][P], double* tri, int n, int g, int lane) {
  constexpr int NPAD = NS * G;
  const int gbase = lane & ~(G - 1);
  int rowoff = 0;  // row_base(c, NPAD)
  __syncwarp();    // pivots written by other lanes in the previous fold are visible
  static_for<0, NS>([&](auto bb) {
    constexpr int bc = decltype(bb)::value;
    const int cols_here = min(G, n - G * bc);
#pragma unroll 1
    for (int gc = 0; gc < cols_here; ++gc) {
      const int c = G * bc + gc;
      double v[P];
#pragma unroll
      for (int i = 0; i < P; ++i) v[i] = __shfl_sync(0xffffffffu, w[bc][i], gbase | gc);
      double* rrow = tri + rowoff + g;  // entry (c, s*G+g) lives at rrow[s*G]
      const double pivot = tri[rowoff + c];
      double rc[NS];
#pragma unroll
      for (int s = bc; s < NS; ++s) rc[s] = rrow[s * G];
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int i = 0; i < P; i += 2) {
        s0 = fma(v[i], v[i], s0);
        s1 = fma(v[i + 1], v[i + 1], s1);
      }
      const Reflector h = make_reflector(pivot, s0 + s1);
#pragma unroll
      for (int s = bc; s < NS; ++s) {
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int i = 0; i < P; i += 2) {
          d0 = fma(v[i], w[s][i], d0);
          d1 = fma(v[i + 1], w[s][i + 1], d1);
        }
        const double sv = h.gamma * fma(h.u0, rc[s], d0 + d1);
        if (s * G + g > c) rrow[s * G] = fma(-h.u0, sv, rc[s]);
#pragma unroll
        for (int i = 0; i < P; ++i) w[s][i] = fma(-v[i], sv, w[s][i]);
      }
      if (g == gc) tri[rowoff + c] = h.beta;
      rowoff += NPAD - c - 1;
    }
  });
}

template <int NS, int G, int P>
__global__ void __launch_bounds__(GroupCfg<NS, G, P>::T, 1) tsqr_group_kernel(const TsqrParams prm) {
  using Cfg = GroupCfg<NS, G, P>;
  constexpr int T = Cfg::T, NW = T / 32, GW = Cfg::GW, CH = Cfg::kChunk, NPAD = Cfg::NPAD;
  constexpr int TS = Cfg::TS, NG = Cfg::NG;
  extern __shared__ __align__(16) double tris[];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane % G, grp = lane / G;  // lane inside group, group inside warp
  const int gid = tid / G;                 // group inside CTA
  const int n = prm.n;
  double* tri = tris + static_cast<size_t>(gid) * TS;
  for (int e = g; e < TS; e += G) tri[e] = 0.0;

  const long long blk = blockIdx.x;
  const long long begin = min(blk * prm.rows_per_block, prm.m);
  const long long end = min((blk + 1) * prm.rows_per_block, prm.m);
  const long long nchunks = (end - begin + CH - 1) / CH;
  const bool aligned = view_bulk_aligned(prm.x, n, begin);

  // this lane's column pointers (padding columns alias column 0 and are masked to zero)
  const double* colp[NS];
  bool colok[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const int col = s * G + g;
    colok[s] = col < n;
    colp[s] = prm.x.col(colok[s] ? col : 0);
  }

  double w[NS][P];
  for (long long ch = warp; ch < nchunks; ch += NW) {
    const long long r0 = begin + ch * CH;
    if (aligned && r0 + static_cast<long long>(NW + 1) * CH <= end) {
      for (int j = lane; j < n; j += 32) {
        const double* nxt = prm.x.col(j) + r0 + static_cast<long long>(NW) * CH;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nxt), "r"(CH * 8) : "memory");
      }
    }
    if (aligned && r0 + CH <= end) {
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const double* cp = colp[s] + r0 + 2 * grp;
#pragma unroll
        for (int k = 0; k < P / 2; ++k) {
          double2 v = make_double2(0.0, 0.0);
          if (colok[s]) v = __ldcs(reinterpret_cast<const double2*>(cp + 2 * GW * k));
          w[s][2 * k] = v.x;
          w[s][2 * k + 1] = v.y;
        }
      }
    } else {
#pragma unroll
      for (int s = 0; s < NS; ++s)
#pragma unroll
        for (int i = 0; i < P; ++i) {
          const long long row = r0 + 2 * GW * (i >> 1) + 2 * grp + (i & 1);
          w[s][i] = (colok[s] && row < end) ? __ldg(colp[s] + row) : 0.0;
        }
    }
    fold_group<NS, G, P>(w, tri, n, g, lane);
  }

  // ---- merge the CTA's group triangles: shared-memory tree, same folding routine ------------------
  int active = NG;
  while (active > 1) {
    const int half = (active + 1) / 2;
    __syncthreads();
    // a warp takes part when any of its groups has a partner; groups without one fold zero rows
    const bool has = gid < active - half;
    const bool warp_has = (warp * GW) < active - half;
    if (warp_has) {
      const double* other = tris + static_cast<size_t>(has ? gid + half : gid) * TS;
#pragma unroll 1
      for (int base = 0; base < n; base += P) {
#pragma unroll
        for (int s = 0; s < NS; ++s)
#pragma unroll
          for (int i = 0; i < P; ++i) {
            const int row = base + i, col = s * G + g;
            w[s][i] = (has && row <= col && row < n) ? other[row_base(row, NPAD) + col] : 0.0;
          }
        fold_group<NS, G, P>(w, tri, n, g, lane);
      }
    }
    active = half;
  }
  __syncthreads();

  // ---- CTA triangle -> rows [blk*n, blk*n+n) of Y (full square, zeros below the diagonal) ---------
  double* dst = prm.y + blk * n;
  bool bad = false;
  for (int idx = tid; idx < n * n; idx += T) {
    const int i = idx % n, j = idx / n;
    double val = 0.0;
    if (i <= j) {
      val = tris[row_base(i, NPAD) + j];
      bad = bad || is_nonfinite(val);
      if (prm.finalize && tris[row_base(i, NPAD) + i] < 0.0) val = -val;
    }
    dst[i + j * prm.ldy] = val;
  }
  if (prm.check_finite && bad) atomicExch(&prm.status->nonfinite, 1);
}

template <int NS, int G, int P>
cudaError_t launch_cfg(const TsqrParams& prm, long long num_blocks, cudaStream_t stream) {
  using Cfg = GroupCfg<NS, G, P>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(tsqr_group_kernel<NS, G, P>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(Cfg::kSmemBytes));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  tsqr_group_kernel<NS, G, P>
      <<<static_cast<unsigned>(num_blocks), Cfg::T, Cfg::kSmemBytes, stream>>>(prm);
  return cudaGetLastError();
}

}  // namespace

// column count -> (slots per lane, lanes per group, rows per step)
#define SQB_GROUP_SWITCH(EXPR)                                   \
  if (n <= 10) return EXPR(5, 2, 8);                             \
  if (n <= 12) return EXPR(6, 2, 8);                             \
  if (n <= 14) return EXPR(7, 2, 8);                             \
  if (n <= 16) return EXPR(8, 2, 8);                             \
  if (n <= 20) return EXPR(5, 4, 8);                             \
  if (n <= 24) return EXPR(6, 4, 8);                             \
  if (n <= 28) return EXPR(7, 4, 8);                             \
  if (n <= 32) return EXPR(8, 4, 8);                             \
  if (n <= 48) return EXPR(3, 16, 16);                           \
  return EXPR(4, 16, 16);

cudaError_t launch_tsqr_group(const TsqrParams& prm, long long num_blocks, cudaStream_t stream) {
  const int n = prm.n;
  if (n < 1 || n > 64) return cudaErrorInvalidValue;
#define LG(NSV, GV, PV) launch_cfg<NSV, GV, PV>(prm, num_blocks, stream)
  SQB_GROUP_SWITCH(LG)
#undef LG
}

int tsqr_group_chunk_rows(int n) {
#define CG(NSV, GV, PV) GroupCfg<NSV, GV, PV>::kChunk
  SQB_GROUP_SWITCH(CG)
#undef CG
}

int tsqr_group_warps(int n) {
#define WG(NSV, GV, PV) (GroupCfg<NSV, GV, PV>::T / 32)
  SQB_GROUP_SWITCH(WG)
#undef WG
}

}  // namespace sqb
