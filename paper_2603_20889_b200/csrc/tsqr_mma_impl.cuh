// Blocked Q-less Householder TSQR on the FP64 tensor cores (DMMA), 16 < n <= 64.
//
// Reference semantics: block_qless_qr_core / factor_trapezoidal / make_reflector
// (reference src/tsqr.cpp:51-158) - fold row panels into a running upper triangle with Householder
// reflectors and discard Q.  The reference pairs reflectors and updates 4 trailing columns at a
// time (tsqr.cpp:86-127); here reflectors are aggregated 8 at a time in compact-WY form
// (Q_b = I - U T U^T, LAPACK tpqrt structure: the top of U is diag(u0) because R is triangular) so
// that the trailing update becomes three small GEMMs on mma.sync.m8n8k4.f64.
//
// Why DMMA: a DFMA with three distinct register operands is register-file bound on sm_100
// (3 clk instead of 2, tools/probe_rf.cu) and the dot/axpy form of Householder has exactly that
// shape, so the FMA kernels top out near 40 % of FP64 peak; a DMMA moves 256 FMAs per 4 operand
// registers.
//
// A WARP owns a P x n register panel (P = 8*RG rows) and a private triangle in shared memory.
//   lane = (g, q), g = lane / 4, q = lane % 4
//   w[t][rr][e] = X[row 8rr + 2q + e, column 8t + g]            (e = 0, 1: one 128-bit load)
// This one layout is at once
//   * the A fragment of W_t^T (m = column g, k = row 2q+e) and the B fragment of V (k = row, n = g)
//     for S^T = W_t^T V (contraction over the panel rows, k-step = (rr, e)),
//   * the C/D fragment (m = column g, n = row 2q+e) of the update W_t^T += Z'^T V^T,
// so the panel never changes layout.  Only the 8 x 8 reflector block is transposed (through a
// shared-memory staging buffer that also serves as the broadcast channel of the in-block sweep).
//
// Per column block b:   in-block sweep (8 reflectors, FMA pipe, one dot pass per reflector: the
// dot with the own column is the norm, the dots with finished columns are the Gram entries that
// build T on the fly), then for every trailing tile t:
//   Y^T = S^T + R_bt^T diag(u0),  Z'^T = Y^T (-T),  R_bt += diag(u0) Z',  W_t^T += Z'^T V^T.
#pragma once

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

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void ld2_pred(double& a, double& b, const double* p, int pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %3, 0;\n\t"
      "mov.f64 %0, 0d0000000000000000;\n\tmov.f64 %1, 0d0000000000000000;\n\t"
      "@q ld.global.cs.v2.f64 {%0, %1}, [%2];\n\t}"
      : "=d"(a), "=d"(b)
      : "l"(p), "r"(pred));
}

template <int NB, int RG, int NW>
struct MmaCfg {
  static constexpr int NPAD = 8 * NB;
  static constexpr int P = 8 * RG;                       // panel rows per warp step
  static constexpr int kTiles = NB * (NB + 1) / 2;       // 8 x 8 tiles of the upper block triangle
  static constexpr int kTriDoubles = kTiles * 64;
  static constexpr int kStagePitch = 80;                 // doubles per 8-row group: 8 columns x pitch 10
  static constexpr int kStageDoubles = RG * kStagePitch;
  static constexpr int kWarpDoubles = kTriDoubles + kStageDoubles + 64;  // + the 8 x 8 T buffer
  static constexpr int T = NW * 32;
  static constexpr size_t kSmemBytes = sizeof(double) * static_cast<size_t>(kWarpDoubles) * NW;
  static_assert(kSmemBytes <= 227 * 1024, "shared memory budget");
};

// Tile (bi, tj), bi <= tj, of the block upper triangle; inside a tile element (r, c) lives at
// [c*8 + r] (column-major), so that lane (g, q) reads rows 2q, 2q+1 of column g with one LDS.128.
__host__ __device__ __forceinline__ constexpr int tile_index(int bi, int tj, int nb) {
  return bi * nb - (bi * (bi - 1)) / 2 + (tj - bi);
}

struct NextPanel {
  const double* base;   // x.base + r_next + 2q
  const double* extra;
  long long ld;
  int n_main, n;
  int pred;
};

template <int NB, int RG>
struct MmaFold {
  static constexpr int PITCH = 80;

  template <int TT>
  static __device__ __forceinline__ void refill(double (&w)[NB][RG][2], const NextPanel& nx, int g) {
    const int col = 8 * TT + g;
    const double* cp = col < nx.n_main ? nx.base + static_cast<long long>(col) * nx.ld : nx.extra;
    const int pred = nx.pred && col < nx.n;
#pragma unroll
    for (int rr = 0; rr < RG; ++rr) ld2_pred(w[TT][rr][0], w[TT][rr][1], cp + 8 * rr, pred);
  }

  // Fold the warp's P x n register panel into its triangle; on return the panel holds the rows
  // named by `nx` (or zeros).
  static __device__ __forceinline__ void run(double (&w)[NB][RG][2], double* tri, double* stage,
                                             double* tbuf, int g, int q, const NextPanel& nx) {
    static_for<0, NB>([&](auto bb) {
      constexpr int b = decltype(bb)::value;
      double* dt = tri + tile_index(b, b, NB) * 64;
      // column g of the diagonal tile: row j of R is only ever changed by reflector j itself, so it
      // can be read before the sweep starts (the pivots are re-read from shared memory, uniform)
      double dcol[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double2 t2 = *reinterpret_cast<const double2*>(dt + g * 8 + 2 * k);
        dcol[2 * k] = t2.x;
        dcol[2 * k + 1] = t2.y;
      }
      double u0p[2] = {0.0, 0.0};
      double gam[8];

      // ---- in-block sweep: 8 reflectors -------------------------------------------------------
      static_for<0, 8>([&](auto jj) {
        constexpr int j = decltype(jj)::value;
        // The last tile may hold fewer than 8 live columns (n = 8 (NB - 1) + r): its padding columns are
        // exact zeros, their reflectors the identity, so their steps are skipped - at n = 33 the padded
        // steps were a fifth of the kernel's reflector chains.  nx.n is the column count, warp-uniform.
        if constexpr (b == NB - 1 && j > 0) {
          if (8 * b + j >= nx.n) return;
        }
        // broadcast column j of the panel (the dense part of reflector j) through the staging buffer
        if (g == j) {
#pragma unroll
          for (int rr = 0; rr < RG; ++rr)
            *reinterpret_cast<double2*>(stage + rr * PITCH + j * 10 + 2 * q) =
                make_double2(w[b][rr][0], w[b][rr][1]);
        }
        __syncwarp();
        // the broadcast column is re-read from the staging buffer wherever it is used (dot pass, update
        // pass, trailing GEMMs) instead of being held: the registers go to a taller panel, and rows in
        // flight per SM is what the latency-bound sweep's throughput is proportional to
        const double* vsrc = stage + j * 10 + 2 * q;
        // one dot pass: v_j . (own column).  Own column == j: sigma.  Own column < j: Gram entry.
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
        for (int rp = 0; rp < RG / 2; ++rp) {
          const double2 t2 = *reinterpret_cast<const double2*>(vsrc + (2 * rp) * PITCH);
          const double2 u2 = *reinterpret_cast<const double2*>(vsrc + (2 * rp + 1) * PITCH);
          a0 = fma(t2.x, w[b][2 * rp][0], a0);
          a1 = fma(t2.y, w[b][2 * rp][1], a1);
          a2 = fma(u2.x, w[b][2 * rp + 1][0], a2);
          a3 = fma(u2.y, w[b][2 * rp + 1][1], a3);
        }
        const double dl = (a0 + a1) + (a2 + a3);
        // sigma straight from the four lanes of column j (independent shuffles: shorter than the
        // butterfly + broadcast); the butterfly for the own-column dot runs beside the scalar chain
        const double sg0 = __shfl_sync(0xffffffffu, dl, 4 * j), sg1 = __shfl_sync(0xffffffffu, dl, 4 * j + 1);
        const double sg2 = __shfl_sync(0xffffffffu, dl, 4 * j + 2), sg3 = __shfl_sync(0xffffffffu, dl, 4 * j + 3);
        const double sigma = (sg0 + sg1) + (sg2 + sg3);
        double d = dl + __shfl_xor_sync(0xffffffffu, dl, 1);
        d += __shfl_xor_sync(0xffffffffu, d, 2);
        const Reflector h = make_reflector(dt[j * 9], sigma);
        const double rc = dcol[j];
        double sv = h.gamma * fma(h.u0, rc, d);
        sv = g > j ? sv : 0.0;  // finished columns keep their reflector vectors
        dcol[j] = g == j ? h.beta : fma(-h.u0, sv, rc);
#pragma unroll
        for (int rr = 0; rr < RG; ++rr) {
          const double2 t2 = *reinterpret_cast<const double2*>(vsrc + rr * PITCH);
          w[b][rr][0] = fma(-t2.x, sv, w[b][rr][0]);
          w[b][rr][1] = fma(-t2.y, sv, w[b][rr][1]);
        }
        u0p[0] = (2 * q == j) ? h.u0 : u0p[0];
        u0p[1] = (2 * q + 1 == j) ? h.u0 : u0p[1];
        // Gram entries of V for the T factor: G(k, j) = v_k . v_j is the finished dot d on lane group k < j;
        // they go to the T buffer and -T is formed once per block after the sweep (in-order issue: a chain
        // of j shuffle-fed FMAs inside the sweep stalled the warp ~170 clk per reflector)
        gam[j] = h.gamma;
        if (q == 0 && g < j) tbuf[g * 8 + j] = d;
      });

      // diagonal tile back to the triangle (all q hold the same column; q == 0 writes) - once every lane has read
      // the last pivot of the sweep from it
      __syncwarp();
      if (q == 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          *reinterpret_cast<double2*>(dt + g * 8 + 2 * k) = make_double2(dcol[2 * k], dcol[2 * k + 1]);
      }

      if constexpr (b < NB - 1) {
        // row g of -T from the Gram entries: -T(g, j) = -gamma_j * sum_{k<j} (-T)(g, k) G(k, j), diagonal
        // -gamma_j (entries left of the diagonal come out as zero on their own); G read as broadcasts
        __syncwarp();
        double tn[8];
        static_for<0, 8>([&](auto jj) {
          constexpr int j = decltype(jj)::value;
          double acc0 = 0.0, acc1 = 0.0;
          static_for<0, j>([&](auto kk) {
            constexpr int k = decltype(kk)::value;
            if constexpr (k % 2 == 0) acc0 = fma(tn[k], tbuf[k * 8 + j], acc0);
            else acc1 = fma(tn[k], tbuf[k * 8 + j], acc1);
          });
          tn[j] = g == j ? -gam[j] : -gam[j] * (acc0 + acc1);
        });
        __syncwarp();
        if (q == 0) {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            *reinterpret_cast<double2*>(tbuf + g * 8 + 2 * k) = make_double2(tn[2 * k], tn[2 * k + 1]);
        }
        __syncwarp();
        double tb[2];
        tb[0] = tbuf[(2 * q) * 8 + g];
        tb[1] = tbuf[(2 * q + 1) * 8 + g];
        const double* vt0 = stage + (2 * q) * 10 + g;  // V^T fragments: row 8rr + g of reflector columns 2q, 2q+1
        // ---- trailing tiles: three small GEMMs on the tensor cores ------------------------------
        static_for<b + 1, NB>([&](auto tt) {
          constexpr int t = decltype(tt)::value;
          double s0 = 0.0, s1 = 0.0;
#pragma unroll
          for (int rr = 0; rr < RG; ++rr) {
            dmma(s0, s1, w[t][rr][0], w[b][rr][0]);
            dmma(s0, s1, w[t][rr][1], w[b][rr][1]);
          }
          double* rt = tri + tile_index(b, t, NB) * 64 + g * 8 + 2 * q;
          double2 r2 = *reinterpret_cast<const double2*>(rt);
          const double y0 = fma(u0p[0], r2.x, s0), y1 = fma(u0p[1], r2.y, s1);
          double z0 = 0.0, z1 = 0.0;
          dmma(z0, z1, y0, tb[0]);
          dmma(z0, z1, y1, tb[1]);
          r2.x = fma(u0p[0], z0, r2.x);
          r2.y = fma(u0p[1], z1, r2.y);
          *reinterpret_cast<double2*>(rt) = r2;
#pragma unroll
          for (int rr = 0; rr < RG; ++rr) {
            dmma(w[t][rr][0], w[t][rr][1], z0, vt0[rr * PITCH]);
            dmma(w[t][rr][0], w[t][rr][1], z1, vt0[rr * PITCH + 10]);
          }
        });
      }
      refill<b>(w, nx, g);
      __syncwarp();  // staging / T buffer reads of this block precede the next block's writes
    });
  }
};

template <int NB, int RG, int NW>
__global__ void __launch_bounds__(NW * 32, 1) tsqr_mma_kernel(const TsqrParams prm) {
  using Cfg = MmaCfg<NB, RG, NW>;
  constexpr int P = Cfg::P, NPAD = Cfg::NPAD, T = Cfg::T;
  extern __shared__ __align__(16) double smem[];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q = lane & 3;
  const int n = prm.n;
  double* my = smem + static_cast<size_t>(warp) * Cfg::kWarpDoubles;
  double* tri = my;
  double* stage = my + Cfg::kTriDoubles;
  double* tbuf = stage + Cfg::kStageDoubles;
  for (int e = lane; e < Cfg::kWarpDoubles; e += 32) my[e] = 0.0;
  __syncwarp();

  const long long blk = blockIdx.x;
  const long long begin = min(blk * prm.rows_per_block, prm.m);
  const long long end = min((blk + 1) * prm.rows_per_block, prm.m);
  const long long npanels = (end - begin + P - 1) / P;
  const bool aligned = view_bulk_aligned(prm.x, n, begin);

  NextPanel nx;
  nx.ld = prm.x.ld;
  nx.n_main = prm.x.n_main;
  nx.n = n;

  double w[NB][RG][2];
  bool loaded = false;

  // ---- stream the block's rows ------------------------------------------------------------------
  for (long long pn = warp; pn < npanels; pn += NW) {
    const long long r0 = begin + pn * P;
    if (!loaded) {
#pragma unroll
      for (int t = 0; t < NB; ++t) {
        const int col = 8 * t + g;
        const double* cp = prm.x.col(col < n ? col : 0);
#pragma unroll
        for (int rr = 0; rr < RG; ++rr)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const long long row = r0 + 8 * rr + 2 * q + e;
            w[t][rr][e] = (col < n && row < end) ? __ldg(cp + row) : 0.0;
          }
      }
    }
    const long long rn = r0 + static_cast<long long>(NW) * P;  // the warp's next panel
    const bool fast = aligned && rn + P <= end;
    nx.base = prm.x.base + rn + 2 * q;
    nx.extra = prm.x.extra + rn + 2 * q;
    nx.pred = fast ? 1 : 0;
    MmaFold<NB, RG>::run(w, tri, stage, tbuf, g, q, nx);
    loaded = fast;
  }

  // ---- merge the CTA's warp triangles: shared-memory tree, same folding routine -------------------
  nx.pred = 0;
  int active = NW;
  while (active > 1) {
    const int half = (active + 1) / 2;
    __syncthreads();
    if (warp < active - half) {
      const double* other = smem + static_cast<size_t>(warp + half) * Cfg::kWarpDoubles;
#pragma unroll 1
      for (int base = 0; base < n; base += P) {
#pragma unroll
        for (int t = 0; t < NB; ++t)
#pragma unroll
          for (int rr = 0; rr < RG; ++rr)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int row = base + 8 * rr + 2 * q + e;
              const int bi = row >> 3;
              w[t][rr][e] = (bi <= t && row < n) ? other[tile_index(bi, t, NB) * 64 + g * 8 + (row & 7)] : 0.0;
            }
        MmaFold<NB, RG>::run(w, tri, stage, tbuf, g, q, nx);
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
      val = smem[tile_index(i >> 3, j >> 3, NB) * 64 + (j & 7) * 8 + (i & 7)];
      bad = bad || is_nonfinite(val);
      const double dg = smem[tile_index(i >> 3, i >> 3, NB) * 64 + (i & 7) * 9];
      if (prm.finalize && dg < 0.0) val = -val;
    }
    dst[i + j * prm.ldy] = val;
  }
  if (prm.check_finite && bad) atomicExch(&prm.status->nonfinite, 1);
  (void)NPAD;
}

template <int NB, int RG, int NW>
cudaError_t launch_cfg(const TsqrParams& prm, long long num_blocks, cudaStream_t stream) {
  using Cfg = MmaCfg<NB, RG, NW>;
  static unsigned long long smem_ready = 0;  // per-device opt-in mask
  {
    cudaError_t e = opt_in_dynamic_smem(tsqr_mma_kernel<NB, RG, NW>, Cfg::kSmemBytes, &smem_ready);
    if (e != cudaSuccess) return e;
  }
  tsqr_mma_kernel<NB, RG, NW><<<static_cast<unsigned>(num_blocks), Cfg::T, Cfg::kSmemBytes, stream>>>(prm);
  return cudaGetLastError();
}

}  // namespace

}  // namespace sqb
