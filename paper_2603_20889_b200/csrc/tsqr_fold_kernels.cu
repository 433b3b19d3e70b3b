// Lookahead lane-group Q-less Householder TSQR, 3 <= n <= 64  ("fold" kernels).
//
// Reference semantics: block_qless_qr_core / factor_trapezoidal / make_reflector
// (reference src/tsqr.cpp:51-158): fold row panels into a running upper triangle with Householder
// reflectors and discard Q.  TSQR lets the rows be partitioned freely, so a GROUP of G adjacent
// lanes (G = 1, 2, 4, 16) is one leaf of the reduction tree: it owns P rows per step and a private
// packed triangle in shared memory; lane g of the group keeps columns g, g+G, g+2G, ... of those
// rows in registers (w[slot][row]).
//
// What is new against tsqr_thread_kernels.cu (FP64-latency bound beyond a handful of columns):
//   * LOOKAHEAD: step c first applies reflector c to the slot that holds column c+1, then derives
//     reflector c+1 (norm, sqrt, reciprocal - a ~15-instruction dependent chain) while the
//     remaining slots are still being updated with reflector c.  Both live in one basic block, so
//     ptxas interleaves the chain with independent FMAs instead of stalling on it.
//   * RETIRE LOADS: a slot whose G columns are finished is refilled at once with the rows of the
//     warp's NEXT chunk (predicated 128-bit streaming loads), so HBM latency hides behind the rest
//     of the fold without a second register panel or a shared-memory stage.
//   * G = 1 (thread-private leaves, no shuffles at all) up to n = 16 with 6-8 rows per step.
// Per reflector the only communication is the broadcast of the P-entry reflector column from its
// owner lane (P 64-bit shuffles inside the group, none for G = 1); every dot product is lane-local.
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

template <int NS, int G, int P, int TMAX>
struct FoldCfg {
  static constexpr int NPAD = NS * G;   // columns incl. padding
  static constexpr int GW = 32 / G;     // groups per warp
  static constexpr int kTri = NPAD * (NPAD + 1) / 2;
  // triangle stride == G (mod 16) doubles: the lanes of a half warp hit distinct banks
  static constexpr int TS = kTri + ((G - kTri % 16) + 16) % 16;
  static constexpr int kMaxGroups = (227 * 1024) / (TS * 8);
  // whole multiples of 4 warps: with 6 warps two SM sub-partitions carry two warps and two carry
  // one, and the FP64 pipe (16 lanes per sub-partition) tops out at 75 % (tools/probe_fp64.cu)
  static constexpr int kT0 = (kMaxGroups * G) / 128 * 128;
  static constexpr int T = kT0 < TMAX ? kT0 : TMAX;  // threads per CTA
  static constexpr int NG = T / G;                    // groups per CTA
  static constexpr int kChunk = GW * P;               // rows a warp consumes per step
  static constexpr size_t kSmemBytes = sizeof(double) * TS * NG;
  static_assert(T >= 64, "too few threads");
  static_assert(P % 2 == 0, "row pairs");
};

// two adjacent rows of one column, zero when the predicate is off
__device__ __forceinline__ void ld2_pred(double& a, double& b, const double* p, int pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %3, 0;\n\t"
      "mov.f64 %0, 0d0000000000000000;\n\tmov.f64 %1, 0d0000000000000000;\n\t"
      "@q ld.global.cs.v2.f64 {%0, %1}, [%2];\n\t}"
      : "=d"(a), "=d"(b)
      : "l"(p), "r"(pred));
}

// the same without predicate and zero fill: full chunks of a thread-private leaf (G == 1: every slot is a live
// column).  The two zero moves per load pair of the predicated form are ALU-pipe instructions, which share the
// FP64 dispatch slot - on the power cap the 8-column kernel is dispatch-bound
__device__ __forceinline__ void ld2_plain(double& a, double& b, const double* p) {
  asm volatile("ld.global.cs.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(b) : "l"(p));
}

// Where the group's next P rows come from when they can be fetched with aligned 128-bit loads.
struct NextChunk {
  const double* base;   // x.base + r_next + 2*grp (row pair of this group in the next chunk)
  const double* extra;  // same for the optional extra column
  long long ld;
  int n_main, n;
  int pred;             // 0: leave the panel zero (the caller fills it by the generic path)
};

template <int NS, int G, int P>
struct Fold {
  static constexpr int NPAD = NS * G;
  static constexpr int GW = 32 / G;

  // FULL: the caller knows that the next chunk is a full, aligned one
  template <int S, bool FULL = false>
  static __device__ __forceinline__ void refill(double (&w)[NS][P], const NextChunk& nx, int g) {
    const int col = S * G + g;
    const double* cp = col < nx.n_main ? nx.base + static_cast<long long>(col) * nx.ld : nx.extra;
    if constexpr (FULL && (G == 1 || S < NS - 1)) {  // every slot but the last holds live columns only (n > (NS-1) G)
#pragma unroll
      for (int k = 0; k < P / 2; ++k) ld2_plain(w[S][2 * k], w[S][2 * k + 1], cp + 2 * GW * k);
    } else {
      const int pred = nx.pred && col < nx.n;
#pragma unroll
      for (int k = 0; k < P / 2; ++k) ld2_pred(w[S][2 * k], w[S][2 * k + 1], cp + 2 * GW * k, pred);
    }
  }

  // column `S`-slot, lane `src` of the group -> v on every lane, plus its reflector
  template <int S>
  static __device__ __forceinline__ void head(const double (&w)[NS][P], double (&v)[P], Reflector& h,
                                              const double* tri, int rowoff, int c, int src) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int i = 0; i < P; ++i) {
      v[i] = G > 1 ? __shfl_sync(0xffffffffu, w[S][i], src, G) : w[S][i];
    }
#pragma unroll
    for (int i = 0; i < P; i += 2) {
      s0 = fma(v[i], v[i], s0);
      s1 = fma(v[i + 1], v[i + 1], s1);
    }
    h = make_reflector(tri[rowoff + c], s0 + s1);
  }

  // One reflector step.  BC = slot of column c; PEEL: c is the last column of its slot (gc == G-1).
  // Written in phases so that every phase offers (live slots) independent FP64 chains: all dot
  // products, all update scalars, then the slot of column c+1, the lookahead reflector, the rest.
  // GUARD: the triangle is only written when `store` (merge tree: a group without a partner folds zero rows
  // beside the others because the shuffles are warp-wide; its triangle is being read by its own partner's
  // owner at a lower slot, so it must not be written, not even with unchanged values).
  template <int BC, bool PEEL, bool GUARD, bool FULL = false>
  static __device__ __forceinline__ void step(double (&w)[NS][P], double (&v)[P], Reflector& h,
                                              double* tri, int& rowoff, int g, int gc,
                                              const NextChunk& nx, bool store) {
    constexpr int S1 = PEEL ? BC + 1 : BC;   // slot of column c+1
    constexpr int SLO = PEEL ? BC + 1 : BC;  // first slot that still has live columns
    constexpr bool HAS_NEXT = S1 < NS;
    const int c = BC * G + gc;
    const int gn = PEEL ? 0 : gc + 1;
    double* rrow = tri + rowoff + g;  // entry (c, s*G+g) at rrow[s*G]
    const int rowoff_next = rowoff + NPAD - c - 1;
    double acc[NS];
    static_for<SLO, NS>([&](auto ss) {
      constexpr int s = decltype(ss)::value;
      acc[s] = h.u0 * rrow[s * G];
    });
#pragma unroll
    for (int i = 0; i < P; ++i) {
      static_for<SLO, NS>([&](auto ss) {
        constexpr int s = decltype(ss)::value;
        acc[s] = fma(v[i], w[s][i], acc[s]);
      });
    }
    static_for<SLO, NS>([&](auto ss) {
      constexpr int s = decltype(ss)::value;
      acc[s] *= h.gamma;
      if ((!GUARD || store) && (s > BC || g > gc)) rrow[s * G] = fma(-h.u0, acc[s], rrow[s * G]);
    });
    Reflector hn;
    if constexpr (HAS_NEXT) {
#pragma unroll
      for (int i = 0; i < P; ++i) w[S1][i] = fma(-v[i], acc[S1], w[S1][i]);
      // lookahead: reflector c+1 from the freshly updated column, overlapped with the updates below
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int i = 0; i < P; i += 2) {
        s0 = fma(w[S1][i], w[S1][i], s0);
        s1 = fma(w[S1][i + 1], w[S1][i + 1], s1);
      }
      double sig = s0 + s1;
      if constexpr (G > 1) sig = __shfl_sync(0xffffffffu, sig, gn, G);
      hn = make_reflector(tri[rowoff_next + c + 1], sig);
    }
#pragma unroll
    for (int i = 0; i < P; ++i) {
      static_for<SLO, NS>([&](auto ss) {
        constexpr int s = decltype(ss)::value;
        if constexpr (!(HAS_NEXT && s == S1)) w[s][i] = fma(-v[i], acc[s], w[s][i]);
      });
    }
    if ((!GUARD || store) && g == gc) tri[rowoff + c] = h.beta;
    if constexpr (PEEL && BC < NS - 1) refill<BC, FULL>(w, nx, g);
    if constexpr (HAS_NEXT) {
      if constexpr (G > 1) {
#pragma unroll
        for (int i = 0; i < P; ++i) v[i] = __shfl_sync(0xffffffffu, w[S1][i], gn, G);
      } else {
#pragma unroll
        for (int i = 0; i < P; ++i) v[i] = w[S1][i];
      }
      h = hn;
    }
    rowoff = rowoff_next;
  }

  // Fold the group's P x n register panel into its triangle; on return the panel holds the rows
  // named by `nx` (or zeros).
  template <bool GUARD = false, bool FULL = false>
  static __device__ __forceinline__ void run(double (&w)[NS][P], double* tri, int n, int g,
                                             const NextChunk& nx, bool store = true) {
    double v[P];
    Reflector h;
    int rowoff = 0;
    if constexpr (G > 1) __syncwarp();  // pivots written by other lanes in the previous fold
    head<0>(w, v, h, tri, 0, 0, 0);
    static_for<0, NS>([&](auto bb) {
      constexpr int bc = decltype(bb)::value;
      if constexpr (bc < NS - 1) {
        if constexpr (G > 1) {
#pragma unroll 1
          for (int gc = 0; gc < G - 1; ++gc) step<bc, false, GUARD, FULL>(w, v, h, tri, rowoff, g, gc, nx, store);
        }
        step<bc, true, GUARD, FULL>(w, v, h, tri, rowoff, g, G - 1, nx, store);
      } else {
        const int cols_last = n - bc * G;  // 1..G live columns in the last slot
        if constexpr (G > 1) {
          const int lim = cols_last < G - 1 ? cols_last : G - 1;
#pragma unroll 1
          for (int gc = 0; gc < lim; ++gc) step<bc, false, GUARD, FULL>(w, v, h, tri, rowoff, g, gc, nx, store);
        }
        if (cols_last == G) step<bc, true, GUARD, FULL>(w, v, h, tri, rowoff, g, G - 1, nx, store);
        refill<bc, FULL>(w, nx, g);
      }
    });
  }
};

template <int NS, int G, int P, int TMAX>
__global__ void __launch_bounds__(FoldCfg<NS, G, P, TMAX>::T, 1) tsqr_fold_kernel(const TsqrParams prm) {
  using Cfg = FoldCfg<NS, G, P, TMAX>;
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

  NextChunk nx;
  nx.ld = prm.x.ld;
  nx.n_main = prm.x.n_main;
  nx.n = n;

  double w[NS][P];
  bool loaded = false;  // the panel already holds the rows of chunk `ch`

  // ---- stream the block's rows ------------------------------------------------------------------
  for (long long ch = warp; ch < nchunks; ch += NW) {
    const long long r0 = begin + ch * CH;
    if (!loaded) {
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const int col = s * G + g;
        const double* cp = prm.x.col(col < n ? col : 0);
#pragma unroll
        for (int i = 0; i < P; ++i) {
          const long long row = r0 + 2 * GW * (i >> 1) + 2 * grp + (i & 1);
          w[s][i] = (col < n && row < end) ? __ldg(cp + row) : 0.0;
        }
      }
    }
    const long long rn = r0 + static_cast<long long>(NW) * CH;  // the warp's next chunk
    const bool fast = aligned && rn + CH <= end;
    if (fast && rn + static_cast<long long>(NW + 1) * CH <= end) {
      // pull the chunk after the next one towards L2
      for (int j = lane; j < n; j += 32) {
        const double* nxt = prm.x.col(j) + rn + static_cast<long long>(NW) * CH;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nxt), "r"(CH * 8) : "memory");
      }
    }
    nx.base = prm.x.base + rn + 2 * grp;
    nx.extra = prm.x.extra + rn + 2 * grp;
    nx.pred = fast ? 1 : 0;
    // a full next chunk needs neither predicates nor zero fill (G > 1: except in the last, possibly padded slot).
    // Measured per group size (profiles/probes/r02_tsqr_experiments.txt, 8): +3-4 % for thread-private leaves from
    // 9 columns on and for lane quads, -3..-11 % for lane pairs (the second copy of the fold pushes ptxas into a
    // worse schedule there), so pairs keep the single predicated path
    if constexpr (G == 1 || G == 4) {
      if (fast) Fold<NS, G, P>::template run<false, true>(w, tri, n, g, nx);
      else Fold<NS, G, P>::run(w, tri, n, g, nx);
    } else {
      Fold<NS, G, P>::run(w, tri, n, g, nx);
    }
    loaded = fast;
  }

  // ---- merge the CTA's group triangles: shared-memory tree, same folding routine ------------------
  nx.pred = 0;
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
        Fold<NS, G, P>::template run<true>(w, tri, n, g, nx, has);
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

template <int NS, int G, int P, int TMAX>
cudaError_t launch_cfg(const TsqrParams& prm, long long num_blocks, cudaStream_t stream) {
  using Cfg = FoldCfg<NS, G, P, TMAX>;
  static unsigned long long smem_ready = 0;  // per-device opt-in mask
  {
    cudaError_t e = opt_in_dynamic_smem(tsqr_fold_kernel<NS, G, P, TMAX>, Cfg::kSmemBytes, &smem_ready);
    if (e != cudaSuccess) return e;
  }
  tsqr_fold_kernel<NS, G, P, TMAX>
      <<<static_cast<unsigned>(num_blocks), Cfg::T, Cfg::kSmemBytes, stream>>>(prm);
  return cudaGetLastError();
}

}  // namespace

// column count -> (slots per lane, lanes per group, rows per step, max threads per CTA); measured
// on B200 (gpurun_out/fold_select.txt, profiles/README.md): thread-private leaves up to 14 columns
// (5..8 columns: taller steps than the register-triangle kernel, 5-9 % faster under the power cap;
// 3 and 4 columns: 2-4 % slower than it on a settled board, 7-11 % faster on the power cap, which is what a
// long run sees - profiles/probes/r02_fold_n3_n4_sustained.txt),
// lane pairs up to 20, lane quads up to 28; above that the DMMA kernel (tsqr_mma_kernels.cu) wins
// and the last three rows only serve a forced kernel family (sqb_set_tsqr_kernel)
#define SQB_FOLD_SWITCH(EXPR)                 \
  switch (n) {                                \
    case 3: return EXPR(3, 1, 16, 256);       \
    case 4: return EXPR(4, 1, 20, 256);       \
    case 5: return EXPR(5, 1, 16, 256);       \
    case 6: return EXPR(6, 1, 16, 256);       \
    case 7: return EXPR(7, 1, 12, 256);       \
    case 8: return EXPR(8, 1, 12, 256);       \
    case 9: return EXPR(9, 1, 10, 256);       \
    case 10: return EXPR(10, 1, 10, 256);     \
    case 11: return EXPR(11, 1, 8, 256);      \
    case 12: return EXPR(12, 1, 8, 256);      \
    case 13: return EXPR(13, 1, 8, 256);      \
    case 14: return EXPR(14, 1, 6, 256);      \
    default: break;                           \
  }                                           \
  if (n <= 16) return EXPR(8, 2, 12, 256);    \
  if (n <= 18) return EXPR(9, 2, 10, 256);    \
  if (n <= 20) return EXPR(10, 2, 10, 256);   \
  if (n <= 24) return EXPR(6, 4, 14, 256);    \
  if (n <= 28) return EXPR(7, 4, 12, 256);    \
  if (n <= 32) return EXPR(8, 4, 12, 256);    \
  if (n <= 48) return EXPR(3, 16, 16, 256);   \
  return EXPR(4, 16, 16, 256);

cudaError_t launch_tsqr_fold(const TsqrParams& prm, long long num_blocks, cudaStream_t stream) {
  const int n = prm.n;
  if (n < kFoldTsqrMinN || n > 64) return cudaErrorInvalidValue;
#define LG(NSV, GV, PV, TV) launch_cfg<NSV, GV, PV, TV>(prm, num_blocks, stream)
  SQB_FOLD_SWITCH(LG)
#undef LG
}

int tsqr_fold_chunk_rows(int n) {
#define CG(NSV, GV, PV, TV) FoldCfg<NSV, GV, PV, TV>::kChunk
  SQB_FOLD_SWITCH(CG)
#undef CG
}

int tsqr_fold_warps(int n) {
#define WG(NSV, GV, PV, TV) (FoldCfg<NSV, GV, PV, TV>::T / 32)
  SQB_FOLD_SWITCH(WG)
#undef WG
}

}  // namespace sqb
