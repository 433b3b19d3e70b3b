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

// Tuning table.  RL = panel rows held per lane per 8-column block (P = 4*RL panel rows per warp),
// NW = warps per CTA.  Variant 0 favours long panels (fewer reflector generations per row),
// variant 1 favours more resident warps (latency hiding for the per-reflector scalar chain).
template <int NB, int VAR>
struct WarpCfg;
template <> struct WarpCfg<1, 0> { static constexpr int RL = 32, NW = 8; };
template <> struct WarpCfg<2, 0> { static constexpr int RL = 24, NW = 8; };
template <> struct WarpCfg<3, 0> { static constexpr int RL = 16, NW = 8; };
template <> struct WarpCfg<4, 0> { static constexpr int RL = 16, NW = 8; };
template <> struct WarpCfg<5, 0> { static constexpr int RL = 12, NW = 8; };
template <> struct WarpCfg<6, 0> { static constexpr int RL = 10, NW = 8; };
template <> struct WarpCfg<7, 0> { static constexpr int RL = 8, NW = 7; };
template <> struct WarpCfg<8, 0> { static constexpr int RL = 8, NW = 6; };
template <> struct WarpCfg<1, 1> { static constexpr int RL = 16, NW = 16; };
template <> struct WarpCfg<2, 1> { static constexpr int RL = 12, NW = 16; };
template <> struct WarpCfg<3, 1> { static constexpr int RL = 8, NW = 16; };
template <> struct WarpCfg<4, 1> { static constexpr int RL = 8, NW = 14; };
template <> struct WarpCfg<5, 1> { static constexpr int RL = 6, NW = 12; };
template <> struct WarpCfg<6, 1> { static constexpr int RL = 6, NW = 10; };
template <> struct WarpCfg<7, 1> { static constexpr int RL = 4, NW = 9; };
template <> struct WarpCfg<8, 1> { static constexpr int RL = 4, NW = 7; };

template <int NB, int VAR = 0>
struct WarpLayout {
  static constexpr int RL = WarpCfg<NB, VAR>::RL;
  static constexpr int NW = WarpCfg<NB, VAR>::NW;
  static constexpr int P = 4 * RL;
  static constexpr int PP = stage_pitch(P, 8);
  static constexpr int NPAD = 8 * NB;
  static constexpr int kStageDoubles = NPAD * PP;
  static constexpr int kTriDoubles = NPAD * (NPAD + 1) / 2;
  static constexpr int kWarpDoubles = kStageDoubles + kTriDoubles + P + 2;  // +2: mbarrier slot
  static constexpr size_t kSmemBytes = sizeof(double) * static_cast<size_t>(kWarpDoubles) * NW;
  static_assert(kSmemBytes <= 227 * 1024, "shared memory budget");
};

// Running triangle: packed ROW-major upper triangle of order NPAD; row c holds (c, c..NPAD-1).
// row_base(c) + j addresses entry (c, j); consecutive rows differ by NPAD - c - 1, so the
// factorisation walks it with one running offset and no index multiplications.
__host__ __device__ __forceinline__ int row_base(int c, int npad) {
  return c * npad - (c * (c - 1)) / 2 - c;
}

__device__ __forceinline__ int panel_row(int q, int i) { return 8 * (i >> 1) + 2 * q + (i & 1); }

// Registers <- stage.
template <int NB, int RL, int PP>
__device__ __forceinline__ void load_panel_regs(double (&w)[NB][RL], const double* stage, int g,
                                                int q) {
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const double* colp = stage + (8 * b + g) * PP + 2 * q;
#pragma unroll
    for (int t = 0; t < RL / 2; ++t) {
      const double2 v = *reinterpret_cast<const double2*>(colp + 8 * t);
      w[b][2 * t] = v.x;
      w[b][2 * t + 1] = v.y;
    }
  }
}

// Fold the register panel into the warp's packed triangle `tri` (n live columns).
// Lanes whose column is not live for a reflector (finished columns, the reflector column itself)
// run the same instructions on values nobody reads again; only the R-row store is predicated.
template <int NB, int RL>
__device__ __forceinline__ void factor_panel(double (&w)[NB][RL], double* tri, double* vbuf,
                                             int n, int lane) {
  constexpr int NPAD = 8 * NB;
  constexpr int ACC = RL >= 16 ? 8 : (RL >= 8 ? 4 : 2);
  const int g = lane >> 2, q = lane & 3;
  double* vq = vbuf + 2 * q;
  int rowoff = 0;  // row_base(c, NPAD)
#pragma unroll
  for (int bc = 0; bc < NB; ++bc) {
    const int cols_here = min(8, n - 8 * bc);
#pragma unroll 1
    for (int gc = 0; gc < cols_here; ++gc) {
      const int c = 8 * bc + gc;
      // Broadcast panel column c (= the reflector's dense part) to all column groups.
      if (g == gc) {
#pragma unroll
        for (int t = 0; t < RL / 2; ++t)
          *reinterpret_cast<double2*>(vq + 8 * t) = make_double2(w[bc][2 * t], w[bc][2 * t + 1]);
      }
      __syncwarp();
      double* rrow = tri + rowoff + g;  // entry (c, 8b+g) lives at rrow[8b]
      const double pivot = tri[rowoff + c];
      double rc[NB];
#pragma unroll
      for (int b = bc; b < NB; ++b) rc[b] = rrow[8 * b];
      double v[RL];
#pragma unroll
      for (int t = 0; t < RL / 2; ++t) {
        const double2 p = *reinterpret_cast<const double2*>(vq + 8 * t);
        v[2 * t] = p.x;
        v[2 * t + 1] = p.y;
      }

      // dot pass: v . (own column of every block from bc on); the owning group's dot is sigma
      double dot[NB];
#pragma unroll
      for (int b = bc; b < NB; ++b) {
        double d[ACC];
#pragma unroll
        for (int a = 0; a < ACC; ++a) d[a] = v[a] * w[b][a];
#pragma unroll
        for (int i = ACC; i < RL; ++i) d[i % ACC] = fma(v[i], w[b][i], d[i % ACC]);
#pragma unroll
        for (int st = ACC / 2; st > 0; st >>= 1)
#pragma unroll
          for (int a = 0; a < st; ++a) d[a] += d[a + st];
        double s = d[0];
        s += shfl_xor_f64(s, 1);
        s += shfl_xor_f64(s, 2);
        dot[b] = s;
      }
      const double sigma = shfl_idx_f64(dot[bc], 4 * gc);  // |panel column c|^2
      // sigma == 0 gives the identity (gamma = u0 = 0, beta = pivot): R(c,c) keeps its value
      // (reference tsqr.cpp:57-60) and every update below is a no-op.
      const Reflector h = make_reflector(pivot, sigma);
#pragma unroll
      for (int b = bc; b < NB; ++b) {
        const double s = h.gamma * fma(h.u0, rc[b], dot[b]);
        if (q == 0 && 8 * b + g > c) rrow[8 * b] = fma(-h.u0, s, rc[b]);
#pragma unroll
        for (int i = 0; i < RL; ++i) w[b][i] = fma(-v[i], s, w[b][i]);
      }
      if (lane == 0) tri[rowoff + c] = h.beta;
      __syncwarp();
      rowoff += NPAD - c - 1;
    }
  }
}

}  // namespace sqb
