// Warp-cooperative Q-less Householder kernel pieces ("warp panel").
//
// Reference semantics restated here: block_qless_qr_core / factor_trapezoidal / make_reflector
// (reference src/tsqr.cpp:51-158): stream a row block panel by panel, fold every panel into a
// running n x n upper triangle with Householder reflectors, never keep Q.
//
// B200 design (not the reference's pencil): a WARP owns a P x n panel entirely in registers and
// a private running triangle in shared memory.
//   * lane = (g, q), g = lane / 4 (column inside an 8-column block), q = lane % 4 (row group);
//     register w[b][i] = X[row(q,i), 8b + g] with row(q, 2t+s) = 8t + 2q + s, so one LDS.128 of
//     the warp's stage fills two rows and is bank-conflict free (stage pitch == 8 mod 16);
//   * reflector c pivots on R(c,c) and spans the P panel rows ("triangle on top" form, LAPACK
//     tpqrt structure) - the dot products touch only the dense panel, R(c, c:n) is a row update;
//   * ONE dot pass per reflector: the panel column c is broadcast through a P-double buffer and
//     every lane dots it with its own columns - the owning column group's dot IS the reflector's
//     sigma, the trailing groups' dots drive the update;
//   * dots reduce over the 4 row groups with two xor-shuffles;
//   * no __syncthreads anywhere in the streaming loop - warps are fully independent.
#pragma once

#include "warp_pipe.cuh"

namespace sqb {

template <int NB>
struct WarpCfg;
// RL = panel rows held per lane per 8-column block; P = 4*RL panel rows; NW = warps per CTA.
template <> struct WarpCfg<1> { static constexpr int RL = 32, NW = 8; };
template <> struct WarpCfg<2> { static constexpr int RL = 24, NW = 8; };
template <> struct WarpCfg<3> { static constexpr int RL = 16, NW = 8; };
template <> struct WarpCfg<4> { static constexpr int RL = 16, NW = 8; };
template <> struct WarpCfg<5> { static constexpr int RL = 12, NW = 8; };
template <> struct WarpCfg<6> { static constexpr int RL = 10, NW = 8; };
template <> struct WarpCfg<7> { static constexpr int RL = 8, NW = 7; };
template <> struct WarpCfg<8> { static constexpr int RL = 8, NW = 6; };

template <int NB>
struct WarpLayout {
  static constexpr int RL = WarpCfg<NB>::RL;
  static constexpr int NW = WarpCfg<NB>::NW;
  static constexpr int P = 4 * RL;
  static constexpr int PP = stage_pitch(P, 8);
  static constexpr int NPAD = 8 * NB;
  static constexpr int kStageDoubles = NPAD * PP;
  static constexpr int kTriDoubles = NPAD * (NPAD + 1) / 2;
  static constexpr int kWarpDoubles = kStageDoubles + kTriDoubles + P + 2;  // +2: mbarrier slot
  static constexpr size_t kSmemBytes = sizeof(double) * static_cast<size_t>(kWarpDoubles) * NW;
};

__device__ __forceinline__ int panel_row(int q, int i) { return 8 * (i >> 1) + 2 * q + (i & 1); }

// Registers <- stage.  Returns the running max of the exponent fields (fused finite check).
template <int NB, int RL, int PP>
__device__ __forceinline__ uint32_t load_panel_regs(double (&w)[NB][RL], const double* stage,
                                                    int g, int q) {
  uint32_t mx = 0;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const double* colp = stage + (8 * b + g) * PP + 2 * q;
#pragma unroll
    for (int t = 0; t < RL / 2; ++t) {
      const double2 v = *reinterpret_cast<const double2*>(colp + 8 * t);
      w[b][2 * t] = v.x;
      w[b][2 * t + 1] = v.y;
      mx = max(mx, max(nonfinite_bits(v.x), nonfinite_bits(v.y)));
    }
  }
  return mx;
}

// Fold the register panel into the warp's packed triangle `tri` (n live columns).
template <int NB, int RL>
__device__ __forceinline__ void factor_panel(double (&w)[NB][RL], double* tri, double* vbuf,
                                             int n, int lane) {
  const int g = lane >> 2, q = lane & 3;
#pragma unroll
  for (int bc = 0; bc < NB; ++bc) {
    const int cols_here = min(8, n - 8 * bc);
    for (int gc = 0; gc < cols_here; ++gc) {
      const int c = 8 * bc + gc;
      // Broadcast panel column c (= the reflector's dense part) to all column groups.
      if (g == gc) {
#pragma unroll
        for (int t = 0; t < RL / 2; ++t)
          *reinterpret_cast<double2*>(vbuf + 8 * t + 2 * q) =
              make_double2(w[bc][2 * t], w[bc][2 * t + 1]);
      }
      __syncwarp();
      double v[RL];
#pragma unroll
      for (int t = 0; t < RL / 2; ++t) {
        const double2 p = *reinterpret_cast<const double2*>(vbuf + 8 * t + 2 * q);
        v[2 * t] = p.x;
        v[2 * t + 1] = p.y;
      }

      // dot pass: v . (own column of every block from bc on)
      double dot[NB];
#pragma unroll
      for (int b = bc; b < NB; ++b) {
        double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
#pragma unroll
        for (int i = 0; i < RL; i += 4) {
          d0 = fma(v[i], w[b][i], d0);
          d1 = fma(v[i + 1], w[b][i + 1], d1);
          if (i + 2 < RL) {
            d2 = fma(v[i + 2], w[b][i + 2], d2);
            d3 = fma(v[i + 3], w[b][i + 3], d3);
          }
        }
        double d = (d0 + d1) + (d2 + d3);
        d += shfl_xor_f64(d, 1);
        d += shfl_xor_f64(d, 2);
        dot[b] = d;
      }
      const double sigma = shfl_idx_f64(dot[bc], 4 * gc);  // |panel column c|^2
      if (sigma != 0.0) {  // sigma == 0: zero reflector, R(c,c) keeps its value (tsqr.cpp:57-60)
        const double pivot = tri[tri_index(c, c)];
        const Reflector h = make_reflector(pivot, sigma);
#pragma unroll
        for (int b = bc; b < NB; ++b) {
          const int j = 8 * b + g;
          const bool live = (j > c) && (j < n);
          const int rix = tri_index(c, live ? j : c);
          const double rcj = live ? tri[rix] : 0.0;
          const double s = live ? h.gamma * fma(h.u0, rcj, dot[b]) : 0.0;
          if (live && q == 0) tri[rix] = fma(-h.u0, s, rcj);
#pragma unroll
          for (int i = 0; i < RL; ++i) w[b][i] = fma(-v[i], s, w[b][i]);
        }
        __syncwarp();
        if (lane == 0) tri[tri_index(c, c)] = h.beta;
      }
      __syncwarp();
    }
  }
}

}  // namespace sqb
