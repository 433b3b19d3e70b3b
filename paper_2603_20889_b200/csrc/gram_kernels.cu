// Fused Gram streaming kernels (sm_100a): one pass over X, no m x n intermediate ever leaves the SM.
//
//   OP_PLAIN     C = X^T X                      reference tsmttsm    (src/gram.cpp:113-121)
//   OP_SOLVE     C = (X R^-1)^T (X R^-1)        reference tsmRttsmR  (src/gram.cpp:123-140)
//   OP_MULTIPLY  C = (X B)^T (X B)              reference tsmmttsmm  (src/gram.cpp:142-151)
//
// Structure (reference blocked_gram, src/gram.cpp:23-94): one CTA per plan block, private
// upper-triangle partial per block, partials summed in ascending block order by
// gram_reduce_kernel (deterministic mode, gram.cpp:81-92), then mirrored.
//
// B200 design: every warp streams its own panels through TMA-fed private stages.  The rank-P
// update runs on the FP64 tensor pipe: lane (g,q) of a warp holds X[row(q), 8b+g], which is at
// the same time the A fragment (8 columns x 4 rows, transposed) and the B fragment (4 rows x 8
// columns) of mma.m8n8k4.f64 - so  C[8b.., 8b'..] += mma(w[b], w[b'])  needs no data movement.
//   * OP_SOLVE substitutes by 8-column blocks on the tensor cores: Y_b^T = Rbb^-T (X_b^T - sum_{a<b} R_ab^T
//     Y_a^T) with explicit inverses of the 8 x 8 diagonal blocks; finished blocks go back to the stage,
//     where later blocks read them as B fragments - X R^-1 never leaves the SM.  (Up to 12 columns the
//     register-resident kernel of gram_thread_kernels.cu substitutes column by column in the reference's
//     order, src/kernels_scalar.cpp:19-32, and is faster.)
//   * OP_MULTIPLY forms (X B) for 8 rows at a time with DMMAs whose accumulator layout is exactly
//     the Gram fragment layout, then feeds those accumulators straight into the Gram MMAs.
#include "kernels.h"

namespace sqb {

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// NB full 8-column tiles go through the tensor pipe; R in 1..4 REMAINDER columns (n = 8 NB + R) are
// handled on the FMA pipe instead of paying for a whole padded tile column of DMMAs (at n = 33 that
// padded tile column was half of the kernel's time): every lane dots its own fragments with the
// remainder columns, which it reads from the stage as warp-wide broadcasts.
template <int NB, int OP, int R = 0>
struct GramCfg {
  static constexpr int NT = NB + (R > 0 ? 1 : 0);  // tile slots of the n x n side (factor, CTA sum)
  static constexpr int NCOL = 8 * NB + R;          // staged columns
  static constexpr int NPAD = 8 * NT;
  static constexpr int NW = 8;  // whole multiples of 4 warps: 6 would leave two SM sub-partitions half idle
  static constexpr int NS = 2;
  // OP_SOLVE: blocked substitution on the tensor cores (8 x 8 diagonal blocks by their explicit
  // inverses, everything off the diagonal as DMMA updates) instead of lane = row
  static_assert(NB >= 2, "up to 8 columns every operation runs the register-resident kernel");
  static constexpr bool kBlockedSolve = OP == OP_SOLVE;
  // streaming panel heights: P == 8 (mod 16) keeps the plain fragment pattern unpadded, P == 0
  // (mod 16) costs the transposed pattern only 4 pad rows
#ifndef SQB_GRAM_2CTA
#define SQB_GRAM_2CTA 1
#endif
  // plain Gram at 17..32 columns: two CTAs per SM (shorter panels, half the shared memory, 16 warps)
#ifndef SQB_GRAM_2CTA_ALL
#define SQB_GRAM_2CTA_ALL 1
#endif
#ifndef SQB_GRAM_2CTA_NB2
#define SQB_GRAM_2CTA_NB2 1
#endif
  // measured: the plain pass wants two CTAs per SM at 3 and 4 tiles, the fused passes at 2 and 4 tiles (at 3
  // tiles one CTA with taller panels and, for the solve, the swizzled stage is 3-5 % faster)
  static constexpr int kCtas = ((SQB_GRAM_2CTA && ((OP == OP_PLAIN && (NB == 3 || NB == 4)) ||
                                                   (OP != OP_PLAIN && SQB_GRAM_2CTA_ALL && NB == 4))) ||
                                (SQB_GRAM_2CTA_NB2 && OP != OP_PLAIN && NB == 2)) ? 2 : 1;
  static constexpr int kPlainP[8] = {120, 72, kCtas == 2 ? 24 : 40, kCtas == 2 ? 24 : 40, 40, 24, 24, 24};
  static constexpr int kMultP[8] = {112, kCtas == 2 ? 32 : 64, kCtas == 2 ? 16 : 48, kCtas == 2 ? 16 : 32, 32, 16, 16, 16};
  static constexpr int kBlockedP[8] = {64, kCtas == 2 ? 32 : 64, kCtas == 2 ? 16 : 48, kCtas == 2 ? 16 : 32, 32, 16, 16, 16};  // == 0 (mod 16): pitch P + 4
  // row groups unrolled in the plain pass - measured per tile count (the DMMA issue order that ptxas derives
  // from it is worth -29 % .. +34 %): 6 and 8 tiles want pairs, everything else the whole panel
  // (two to four remainder columns: pairs again, except at 18 columns - measured)
  static constexpr int kPlainUnroll = (NB == 6 || NB == 8 || R >= 3 || (R == 2 && NB >= 3)) ? 2 : 15;
  static constexpr int kMultUnroll = NB == 2 ? 4 : (NB == 3 ? (kCtas == 2 ? 2 : 3) : 2);  // row groups multiplied together (measured per tile count)
  static constexpr int kSolveUnroll = NB <= 2 ? 4 : (kCtas == 2 ? 2 : (NB == 3 ? 3 : (NB == 4 ? 4 : (NB == 5 ? 4 : 2))));  // row groups solved together
  static constexpr int P =
      kBlockedSolve ? kBlockedP[NB - 1] : (OP == OP_PLAIN ? kPlainP[NB - 1] : kMultP[NB - 1]);
  // Blocked solve: the stage is read with the transposed LDS.64 pattern (DMMA B operands) AND read / written
  // with the own-row 128-bit pattern.  A single pitch serves only one of them (pitch P + 4: 2-way conflicts on
  // every 128-bit access, 3.2-3.8e8 per launch in ncu); pitch == 8 (mod 16) plus a 4-double offset of every
  // second column pair serves both (kSwz), where the slightly larger stage still fits.
  // At 64 columns the swizzled stage only fits when the factor is stored packed: the blocked solve reads
  // nothing but the strictly upper 8 x 8 blocks (column 8b+g: rows 0..8b-1 at pitch 8b+4, which is
  // 4 or 12 (mod 16): conflict-free A-fragment reads), the diagonal blocks live on as their inverses.
  static constexpr bool kPackFac = kBlockedSolve && R == 0 && NB == 8;
  static constexpr int kFacMain = kPackFac ? 32 * (NB * NB - 1) : NPAD * (NPAD + 4);
  static constexpr int kFacDoublesPre = OP == OP_PLAIN ? 0 : kFacMain + NPAD + (kBlockedSolve ? NT * 8 * 12 : 0);
  // measured: the swizzle pays where one CTA owns the SM (5..8 tiles: +8 % at 48 columns); the two-CTA
  // configurations (16..32 columns) already run the tensor pipe at 83-87 % and gain nothing
  static constexpr bool kSwz =
      kBlockedSolve && kCtas == 1 &&
      (sizeof(double) * (static_cast<size_t>(NS) * (NCOL * stage_pitch(P, 8) + 4) * NW + kFacDoublesPre) + 1024) <= 227 * 1024;
  static constexpr int PP = kSwz ? stage_pitch(P, 8) : stage_pitch(P, (OP == OP_MULTIPLY || kBlockedSolve) ? 4 : 8);
  static constexpr int kStageDoubles = NCOL * PP + (kSwz ? 4 : 0);
  static constexpr int kVbuf = 0;
  static constexpr int kWarpDoubles = NS * kStageDoubles + kVbuf;
  static constexpr int FP = NPAD + 4;  // factor pitch: conflict-free A-fragment reads
  static constexpr int kDinvPitch = 12;  // (4k+q) + 12 g: conflict-free A-fragment reads of an 8 x 8 block
  static constexpr int kFacDoubles = kFacDoublesPre;
  static_assert(FP == NPAD + 4 && kDinvPitch == 12, "kFacDoublesPre assumes these pitches");
  static constexpr int kSumDoubles = NPAD * NPAD;  // aliases the warp stages after the streaming loop
  static_assert(kSumDoubles <= kWarpDoubles * NW, "the CTA sum must fit into the stage area");
  static constexpr size_t kSmemBytes =
      sizeof(double) * (static_cast<size_t>(kWarpDoubles) * NW + kFacDoubles);
  static constexpr int NPAIR = NB * (NB + 1) / 2;
  // How a warp fills its stages.  cp.async.bulk takes uniform operands, so "one bulk copy per column" compiles
  // to an election loop of ~9 instructions per column and panel (40-64 columns: as many issue slots as the
  // panel's DMMAs, and with two warps per scheduler the tensor pipe idles whenever both are in it: 62 / 73 /
  // 80 % DMMA pipe at 40 / 48 / 56 columns against 88 % at 64).  Per-lane 16-byte cp.async copies (LDGSTS,
  // commit groups) move a panel in P * NCOL / 64 instructions: plain pass +14 / +17 / +28 % at 40 / 48 / 56
  // columns, solve pass +9 % from 48 columns and +14 / +19 % at 17 / 33, multiply pass +8 % from 48.  The bulk
  // form stays where it measured faster (profiles/probes/r02_lane_copies_ab.txt).
#ifndef SQB_GRAM_LANE_COPIES
#define SQB_GRAM_LANE_COPIES 1
#endif
  static constexpr bool kLaneCopies =
      SQB_GRAM_LANE_COPIES != 0 &&
      (OP == OP_PLAIN ? R == 0 : (NB >= 4 || R > 0));
  static_assert(P >= 8 && P % 8 == 0, "panel rows");
  static_assert(kSmemBytes * kCtas + 1024 * kCtas <= 227 * 1024, "shared memory budget");
  static_assert(R == 0 || OP == OP_PLAIN || OP == OP_MULTIPLY || kBlockedSolve, "remainder variants");
};

template <int NB, int OP, int R>
__global__ void __launch_bounds__(GramCfg<NB, OP, R>::NW * kWarp, GramCfg<NB, OP, R>::kCtas)
    gram_mma_kernel(const GramParams prm) {
  using Cfg = GramCfg<NB, OP, R>;
  constexpr int P = Cfg::P, PP = Cfg::PP, NW = Cfg::NW, NS = Cfg::NS, NPAD = Cfg::NPAD;
  constexpr int FP = Cfg::FP, NPAIR = Cfg::NPAIR, NT = Cfg::NT;
  constexpr bool SWZ = Cfg::kSwz;
  auto coff = [](int c) { return stage_col_offset<PP, SWZ>(c); };  // stage offset of column c
  constexpr int RR = R > 0 ? R : 1;  // array extent of the remainder accumulators
  extern __shared__ __align__(128) double smem[];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, q = lane & 3;
  const int n = prm.n;

  double* my = smem + static_cast<size_t>(warp) * Cfg::kWarpDoubles;
  double* vbuf = my + NS * Cfg::kStageDoubles;
  // the mbarriers live OUTSIDE the dynamic stage area: that area is repurposed as the CTA sum at the
  // end, and the memory of a live mbarrier object must not be overwritten (PTX: mbarrier.inval first);
  // racecheck runs of the aliased layout produced intermittent NaNs from 40 columns on
  __shared__ uint64_t bars_all[NW * NS];
  uint64_t* bars = bars_all + warp * NS;
  (void)vbuf;
  double* fac = smem + static_cast<size_t>(NW) * Cfg::kWarpDoubles;  // NPAD x FP (or packed), then inv diag
  double* inv = fac + Cfg::kFacMain;
  constexpr bool PACK = Cfg::kPackFac;
  // element (row, column 8b+g) of the factor as the blocked solve reads it (row < 8b when packed)
  auto fidx = [](int row, int b, int g) { return PACK ? 32 * (b * b - 1) + g * (8 * b + 4) + row : row + (8 * b + g) * FP; };
  double* csum = smem;  // reused once every warp has left the streaming loop

  for (int i = lane; i < NS * Cfg::kStageDoubles + Cfg::kVbuf; i += kWarp) my[i] = 0.0;
  if (lane < NS) mbar_init(bars + lane, 1);
  mbar_fence_init();
  if (OP != OP_PLAIN) {
    for (int i = threadIdx.x; i < Cfg::kFacDoubles; i += NW * kWarp) fac[i] = 0.0;
    __syncthreads();
    // packed factor: the full copy only exists during this prologue, in the (still idle) stage area
    double* ff = PACK ? smem : fac;
    for (int i = threadIdx.x; i < n * n; i += NW * kWarp) {
      const int r = i % n, c = i / n;
      if (OP == OP_MULTIPLY || r <= c) ff[r + c * FP] = prm.factor[i];
    }
    __syncthreads();
    if constexpr (Cfg::kBlockedSolve) {
      // explicit inverses of the 8 x 8 diagonal blocks (thread = one column of one block, back
      // substitution; padded columns act as identity), then the strictly upper blocks are negated
      // so that the DMMA updates subtract
      double* dinv = inv + NPAD;
      if (threadIdx.x < NPAD) {
        const int b = threadIdx.x >> 3, j = threadIdx.x & 7;
        double xcol[8];
#pragma unroll
        for (int i = 7; i >= 0; --i) {
          double v = i == j ? 1.0 : 0.0;
#pragma unroll
          for (int k2 = i + 1; k2 < 8; ++k2)
            if (k2 <= j) v = fma(-ff[(8 * b + i) + (8 * b + k2) * FP], xcol[k2], v);
          const double dgn = (8 * b + i) < n ? ff[(8 * b + i) + (8 * b + i) * FP] : 1.0;
          xcol[i] = i <= j ? v / dgn : 0.0;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) dinv[b * 8 * Cfg::kDinvPitch + i + Cfg::kDinvPitch * j] = xcol[i];
      }
    }
    if (OP == OP_SOLVE) {
      // reference tsmRttsmR pre-check (gram.cpp:126-134): |r_jj| > n*eps*max|r_jj|, else
      // SingularFactorError(j) for the first offending j; inv_diag precomputed.
      if (threadIdx.x == 0) {
        double mx = 0.0;
        for (int j = 0; j < n; ++j) mx = fmax(mx, fabs(ff[j + j * FP]));
        const double dtol = static_cast<double>(n) * 2.220446049250313e-16 * mx;
        int bad = -1;
        for (int j = 0; j < n; ++j) {
          const double d = ff[j + j * FP];
          if (bad < 0 && !(fabs(d) > dtol)) bad = j;
          inv[j] = 1.0 / d;
        }
        if (bad >= 0 && blockIdx.x == 0) raise_status(prm.status, SQB_E_SINGULAR, bad);
      }
    }
    if constexpr (Cfg::kBlockedSolve) {
      __syncthreads();
      for (int i = threadIdx.x; i < NPAD * NPAD; i += NW * kWarp) {
        const int r = i % NPAD, c = i / NPAD;
        if ((r >> 3) < (c >> 3)) fac[fidx(r, c >> 3, c & 7)] = -ff[r + c * FP];
      }
      if constexpr (PACK) {  // give the stage area back as zeros
        __syncthreads();
        for (int i = threadIdx.x; i < NPAD * FP; i += NW * kWarp) smem[i] = 0.0;
      }
    }
  }
  __syncthreads();

  const long long blk = blockIdx.x;
  const long long begin = min(blk * prm.rows_per_block, prm.m);
  const long long end = min((blk + 1) * prm.rows_per_block, prm.m);
  const long long npanels = (end - begin + P - 1) / P;
  const bool aligned = view_bulk_aligned(prm.x, n, begin);

  double acc[NPAIR][2];
#pragma unroll
  for (int p = 0; p < NPAIR; ++p) acc[p][0] = acc[p][1] = 0.0;
  // racc[b][k]: this lane's rows of (own column of tile b) . (remainder column k); b == NB is the
  // remainder block against itself (lanes g < R)
  double racc[NT][RR];
#pragma unroll
  for (int b = 0; b < NT; ++b)
#pragma unroll
    for (int k = 0; k < RR; ++k) racc[b][k] = 0.0;
  uint32_t phase_bits = 0;   // bit s = parity to wait for on stage s
  uint32_t async_bits = 0;   // bit s = stage s was filled by the async engine

  constexpr bool kLaneCopies = Cfg::kLaneCopies;
  auto issue = [&](long long pnl, int s) {
    if constexpr (kLaneCopies) {
      if (pnl < npanels)
        issue_panel_lanes<P, PP, SWZ>(prm.x, n, begin + pnl * P, end, aligned, my + s * Cfg::kStageDoubles, lane);
      cp_async_commit();  // one group per slot, empty past the last panel: the wait below counts groups
    } else {
      if (pnl >= npanels) return;
      const bool a = issue_panel<P, PP, SWZ>(prm.x, n, begin + pnl * P, end, aligned,
                                        my + s * Cfg::kStageDoubles, bars + s, lane);
      async_bits = a ? (async_bits | (1u << s)) : (async_bits & ~(1u << s));
    }
  };

  // prologue: fill all stages
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    issue(warp + static_cast<long long>(s) * NW, s);
  }

  long long it = 0;
  for (long long pnl = warp; pnl < npanels; pnl += NW, ++it) {
    const int s = static_cast<int>(it % NS);
    const double* stage = my + s * Cfg::kStageDoubles;
    if constexpr (kLaneCopies) {
      cp_async_wait<NS - 1>();
      __syncwarp();
    } else if (async_bits & (1u << s)) {
      mbar_wait(bars + s, (phase_bits >> s) & 1u);
      phase_bits ^= 1u << s;
    }

    if (OP == OP_PLAIN) {
#pragma unroll(Cfg::kPlainUnroll)
      for (int t = 0; t < P / 8; ++t) {
        double2 a[NB];
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          a[b] = *reinterpret_cast<const double2*>(stage + (8 * b + g) * PP + 8 * t + 2 * q);
        }
        // all pairs with the even rows, then all pairs with the odd rows: NPAIR independent MMAs
        // between two updates of the same accumulator
        int p = 0;
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
          for (int b2 = b; b2 < NB; ++b2, ++p) dmma884(acc[p][0], acc[p][1], a[b].x, a[b2].x);
        p = 0;
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
          for (int b2 = b; b2 < NB; ++b2, ++p) dmma884(acc[p][0], acc[p][1], a[b].y, a[b2].y);
        if constexpr (R > 0) {
          double2 ar = make_double2(0.0, 0.0);
          if (g < R) ar = *reinterpret_cast<const double2*>(stage + (8 * NB + g) * PP + 8 * t + 2 * q);
#pragma unroll
          for (int k = 0; k < R; ++k) {
            const double2 c = *reinterpret_cast<const double2*>(stage + (8 * NB + k) * PP + 8 * t + 2 * q);
#pragma unroll
            for (int b = 0; b < NB; ++b) racc[b][k] = fma(a[b].y, c.y, fma(a[b].x, c.x, racc[b][k]));
            racc[NB][k] = fma(ar.y, c.y, fma(ar.x, c.x, racc[NB][k]));
          }
        }
      }
      __syncwarp();
      issue(pnl + static_cast<long long>(NS) * NW, s);
    } else if (Cfg::kBlockedSolve) {
      // Y = X R^-1 by 8-column blocks, 8 rows at a time, transposed so that the result lands in the
      // Gram fragment layout: Y_b^T = Rbb^-T (X_b^T - sum_{a<b} R_ab^T Y_a^T).  Finished blocks are
      // written back to the stage, where later blocks read them as B fragments (row g, column 4k+q).
      double* wstage = my + s * Cfg::kStageDoubles;
      const double* dinv = inv + NPAD;
      // TU row groups advance together: their chains are independent (ILP for the latency-bound narrow
      // cases) and they share the three warp barriers of a block
      constexpr int TU = Cfg::kSolveUnroll;
      static_assert(!Cfg::kBlockedSolve || (P / 8) % TU == 0, "row groups per panel");
#pragma unroll 1
      // One remainder column is cheapest substituted on the FMA pipe (kRemFma); two to four go through the
      // padded-tile DMMA substitution like a full block (the shuffle reductions of the FMA form cost more
      // than the padded DMMAs from two columns on: measured, profiles/README.md) - their Gram products
      // are formed on the FMA pipe either way.
      constexpr bool kRemFma = R == 1;
      constexpr int NSV = kRemFma ? NB : NT;  // tile slots the DMMA substitution walks
      for (int t0 = 0; t0 < P / 8; t0 += TU) {
        double2 y[TU][NT];
#pragma unroll
        for (int b = 0; b < NSV; ++b) {
          // the remainder block (b == NB, R live columns) keeps a tight stage: its dead lanes hold zeros
          const bool live = b < NB || g < R;
          double* own = wstage + coff(8 * b + g) + 8 * t0 + 2 * q;
          double z[TU][2];
#pragma unroll
          for (int u = 0; u < TU; ++u) {
            double2 x2 = make_double2(0.0, 0.0);
            if (live) x2 = *reinterpret_cast<const double2*>(own + 8 * u);
            z[u][0] = x2.x;
            z[u][1] = x2.y;
          }
#pragma unroll
          for (int a = 0; a < b; ++a) {
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
              const double af = fac[fidx(8 * a + 4 * kk + q, b, g)];  // -R_ab
#pragma unroll
              for (int u = 0; u < TU; ++u)
                dmma884(z[u][0], z[u][1], af, wstage[coff(8 * a + 4 * kk + q) + 8 * (t0 + u) + g]);
            }
          }
          if (live) {
#pragma unroll
            for (int u = 0; u < TU; ++u) *reinterpret_cast<double2*>(own + 8 * u) = make_double2(z[u][0], z[u][1]);
          }
          __syncwarp();
          double w[TU][2];
#pragma unroll
          for (int u = 0; u < TU; ++u) w[u][0] = w[u][1] = 0.0;
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            const double af = dinv[b * 8 * Cfg::kDinvPitch + (4 * kk + q) + Cfg::kDinvPitch * g];
            const bool zlive = b < NB || 4 * kk + q < R;
#pragma unroll
            for (int u = 0; u < TU; ++u)
              dmma884(w[u][0], w[u][1], af, zlive ? wstage[coff(8 * b + 4 * kk + q) + 8 * (t0 + u) + g] : 0.0);
          }
          __syncwarp();  // every lane has read Z_b before Y_b replaces it
#pragma unroll
          for (int u = 0; u < TU; ++u) {
            if (live) *reinterpret_cast<double2*>(own + 8 * u) = make_double2(w[u][0], w[u][1]);
            y[u][b] = make_double2(w[u][0], w[u][1]);
          }
          __syncwarp();
        }
        // yr[u][k]: remainder column k of Y for this lane's two rows (the broadcast operand of the remainder
        // Gram products)
        double2 yr[TU][RR];
        if constexpr (kRemFma) {
          // y_c = (x_c - sum_{i < c} y_i R(i, c)) / R(c, c): a lane sums over its own columns of the full tiles
          // (the strictly upper blocks of the factor are stored negated), three xor-shuffles over the column
          // index g complete the sum; the result never goes back to the stage
          constexpr int c = 8 * NB;
          double fcol[NB];
#pragma unroll
          for (int b = 0; b < NB; ++b) fcol[b] = fac[(8 * b + g) + c * FP];
          const double dinv_c = inv[c];
#pragma unroll
          for (int u = 0; u < TU; ++u) {
            const double2 xr = *reinterpret_cast<const double2*>(wstage + coff(c) + 8 * (t0 + u) + 2 * q);
            double px = 0.0, py = 0.0;
#pragma unroll
            for (int b = 0; b < NB; ++b) {
              px = fma(fcol[b], y[u][b].x, px);
              py = fma(fcol[b], y[u][b].y, py);
            }
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) {
              px += __shfl_xor_sync(0xffffffffu, px, o);
              py += __shfl_xor_sync(0xffffffffu, py, o);
            }
            yr[u][0] = make_double2((px + xr.x) * dinv_c, (py + xr.y) * dinv_c);
            y[u][NB] = g == 0 ? yr[u][0] : make_double2(0.0, 0.0);
          }
        } else if constexpr (R > 0) {
#pragma unroll
          for (int u = 0; u < TU; ++u)
#pragma unroll
            for (int k = 0; k < R; ++k)
              yr[u][k] = *reinterpret_cast<const double2*>(wstage + coff(8 * NB + k) + 8 * (t0 + u) + 2 * q);
        }
#pragma unroll
        for (int u = 0; u < TU; ++u) {
          int p = 0;
#pragma unroll
          for (int b = 0; b < NB; ++b)
#pragma unroll
            for (int b2 = b; b2 < NB; ++b2, ++p) dmma884(acc[p][0], acc[p][1], y[u][b].x, y[u][b2].x);
          p = 0;
#pragma unroll
          for (int b = 0; b < NB; ++b)
#pragma unroll
            for (int b2 = b; b2 < NB; ++b2, ++p) dmma884(acc[p][0], acc[p][1], y[u][b].y, y[u][b2].y);
          if constexpr (R > 0) {
#pragma unroll
            for (int k = 0; k < R; ++k) {
              const double2 c = yr[u][k];
#pragma unroll
              for (int b = 0; b < NT; ++b) racc[b][k] = fma(y[u][b].y, c.y, fma(y[u][b].x, c.x, racc[b][k]));
            }
          }
        }
      }
      __syncwarp();
      issue(pnl + static_cast<long long>(NS) * NW, s);
    } else {  // OP_MULTIPLY
      const int kchunks = (n + 3) / 4;
      // MU row groups advance together: NT * MU independent DMMA chains of length kchunks, and every
      // factor fragment is loaded once per MU groups
      constexpr int MU = Cfg::kMultUnroll;
      static_assert(OP != OP_MULTIPLY || (P / 8) % MU == 0, "row groups per panel");
#pragma unroll 1
      for (int t0 = 0; t0 < P / 8; t0 += MU) {
        double y[MU][NT][2];
#pragma unroll
        for (int u = 0; u < MU; ++u)
#pragma unroll
          for (int b = 0; b < NT; ++b) y[u][b][0] = y[u][b][1] = 0.0;
#pragma unroll 1
        for (int kc = 0; kc < kchunks; ++kc) {
          double bf[MU];
          // the stage holds exactly the n live columns when there is a remainder tile
          const bool klive = R == 0 || 4 * kc + q < Cfg::NCOL;
#pragma unroll
          for (int u = 0; u < MU; ++u) bf[u] = klive ? stage[(4 * kc + q) * PP + 8 * (t0 + u) + g] : 0.0;
#pragma unroll
          for (int b = 0; b < NT; ++b) {
            const double af = fac[(4 * kc + q) + (8 * b + g) * FP];
#pragma unroll
            for (int u = 0; u < MU; ++u) dmma884(y[u][b][0], y[u][b][1], af, bf[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < MU; ++u) {
          int p = 0;
#pragma unroll
          for (int b = 0; b < NB; ++b)
#pragma unroll
            for (int b2 = b; b2 < NB; ++b2, ++p) dmma884(acc[p][0], acc[p][1], y[u][b][0], y[u][b2][0]);
          p = 0;
#pragma unroll
          for (int b = 0; b < NB; ++b)
#pragma unroll
            for (int b2 = b; b2 < NB; ++b2, ++p) dmma884(acc[p][0], acc[p][1], y[u][b][1], y[u][b2][1]);
          if constexpr (R > 0) {
            // remainder columns of X B sit in the accumulators of lane group k: one shuffle per row
            // hands them to every column group, the products go to the FMA pipe
#pragma unroll
            for (int k = 0; k < R; ++k) {
              const double c0 = __shfl_sync(0xffffffffu, y[u][NB][0], 4 * k + q);
              const double c1 = __shfl_sync(0xffffffffu, y[u][NB][1], 4 * k + q);
#pragma unroll
              for (int b = 0; b < NT; ++b) racc[b][k] = fma(y[u][b][1], c1, fma(y[u][b][0], c0, racc[b][k]));
            }
          }
        }
      }
      __syncwarp();
      issue(pnl + static_cast<long long>(NS) * NW, s);
    }
  }

  // ---- CTA reduction in fixed warp order, then the block's upper-triangle partial -------------
  if constexpr (kLaneCopies) cp_async_wait<0>();
  __syncthreads();  // all stages drained: the stage area becomes the CTA sum
  for (int i = threadIdx.x; i < Cfg::kSumDoubles; i += NW * kWarp) csum[i] = 0.0;
  for (int wi = 0; wi < NW; ++wi) {
    __syncthreads();
    if (warp == wi) {
      int p = 0;
#pragma unroll
      for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int b2 = b; b2 < NB; ++b2, ++p) {
          const int row = 8 * b + g, col = 8 * b2 + 2 * q;
          csum[row + col * NPAD] += acc[p][0];
          csum[row + (col + 1) * NPAD] += acc[p][1];
        }
      if constexpr (R > 0) {
#pragma unroll
        for (int b = 0; b < NT; ++b)
#pragma unroll
          for (int k = 0; k < R; ++k) {
            double sr = racc[b][k];
            sr += __shfl_xor_sync(0xffffffffu, sr, 1);
            sr += __shfl_xor_sync(0xffffffffu, sr, 2);
            if (q == 0) csum[(8 * b + g) + (8 * NB + k) * NPAD] += sr;
          }
      }
    }
  }
  __syncthreads();
  double* dst = prm.partial + blk * static_cast<long long>(n) * n;
  for (int idx = threadIdx.x; idx < n * n; idx += NW * kWarp) {
    const int i = idx % n, j = idx / n;
    dst[idx] = i <= j ? csum[i + j * NPAD] : 0.0;
  }
}

// Sum the per-block partials in ascending block order over the upper triangle and mirror
// (reference gram.cpp:81-92).
__global__ void gram_reduce_kernel(const double* partial, long long num_blocks, int n, double* c,
                                   int check_finite, StatusWord* status) {
  for (int idx = threadIdx.x + blockIdx.x * blockDim.x; idx < n * n; idx += blockDim.x * gridDim.x) {
    const int i = idx % n, j = idx / n;
    if (i > j) continue;
    double s = 0.0;
    for (long long b = 0; b < num_blocks; ++b) s += partial[b * static_cast<long long>(n) * n + idx];
    c[i + j * n] = s;
    c[j + i * n] = s;
    if (check_finite && is_nonfinite(s)) atomicExch(&status->nonfinite, 1);
  }
}

template <int NB, int OP, int R = 0>
static cudaError_t launch_gram_nb(const GramParams& prm, long long num_blocks, cudaStream_t stream) {
  using Cfg = GramCfg<NB, OP, R>;
  static unsigned long long smem_ready = 0;  // per-device opt-in mask
  {
    cudaError_t e = opt_in_dynamic_smem(gram_mma_kernel<NB, OP, R>, Cfg::kSmemBytes, &smem_ready);
    if (e != cudaSuccess) return e;
  }
  gram_mma_kernel<NB, OP, R>
      <<<static_cast<unsigned>(num_blocks), Cfg::NW * kWarp, Cfg::kSmemBytes, stream>>>(prm);
  return cudaGetLastError();
}

// 8 NB + R columns, 2 <= NB <= 4: the R remainder columns on the FMA pipe instead of a padded tile column,
// wherever that measured faster than the padded (NB + 1)-tile kernel (profiles/probes/r02_remainder_ab.txt):
// largest R per (operation, NB).  The multiply pass hands its remainder entries to the other column groups
// through shuffles, the solve pass substitutes them with a padded DMMA from R = 2 on - both stop paying early.
constexpr bool gram_remainder_variant(int n, int op) {
  const int nb = n / 8, r = n % 8;
  if (r == 0 || nb < 2 || nb > 4) return false;
  const int max_r = op == OP_PLAIN ? (nb == 3 ? 3 : 4) : (op == OP_SOLVE ? (nb == 2 ? 4 : (nb == 3 ? 2 : 1)) : (nb == 4 ? 0 : 2));
  return r <= max_r;
}

template <int NB, int OP>
static cudaError_t launch_gram_rem(const GramParams& prm, long long num_blocks, cudaStream_t stream) {
  switch (prm.n % 8) {
    case 1: return launch_gram_nb<NB, OP, 1>(prm, num_blocks, stream);
    case 2: return launch_gram_nb<NB, OP, 2>(prm, num_blocks, stream);
    case 3: return launch_gram_nb<NB, OP, 3>(prm, num_blocks, stream);
    default: return launch_gram_nb<NB, OP, 4>(prm, num_blocks, stream);
  }
}

template <int OP>
static cudaError_t launch_gram_op(const GramParams& prm, long long num_blocks, cudaStream_t stream) {
  if (gram_remainder_variant(prm.n, OP)) {
    switch (prm.n / 8) {
      case 2: return launch_gram_rem<2, OP>(prm, num_blocks, stream);
      case 3: return launch_gram_rem<3, OP>(prm, num_blocks, stream);
      default: return launch_gram_rem<4, OP>(prm, num_blocks, stream);
    }
  }
  switch ((prm.n + 7) / 8) {
    case 2: return launch_gram_nb<2, OP>(prm, num_blocks, stream);
    case 3: return launch_gram_nb<3, OP>(prm, num_blocks, stream);
    case 4: return launch_gram_nb<4, OP>(prm, num_blocks, stream);
    case 5: return launch_gram_nb<5, OP>(prm, num_blocks, stream);
    case 6: return launch_gram_nb<6, OP>(prm, num_blocks, stream);
    case 7: return launch_gram_nb<7, OP>(prm, num_blocks, stream);
    case 8: return launch_gram_nb<8, OP>(prm, num_blocks, stream);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_gram(const GramParams& prm, int op, long long num_blocks, cudaStream_t stream) {
  if (gram_use_thread(prm.n, op)) return launch_gram_thread(prm, op, num_blocks, stream);
  switch (op) {
    case OP_PLAIN: return launch_gram_op<OP_PLAIN>(prm, num_blocks, stream);
    case OP_SOLVE: return launch_gram_op<OP_SOLVE>(prm, num_blocks, stream);
    case OP_MULTIPLY: return launch_gram_op<OP_MULTIPLY>(prm, num_blocks, stream);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_gram_reduce(const double* partial, long long num_blocks, int n, double* c,
                               int check_finite, StatusWord* status, cudaStream_t stream) {
  gram_reduce_kernel<<<(n * n + 255) / 256, 256, 0, stream>>>(partial, num_blocks, n, c, check_finite,
                                                              status);
  return cudaGetLastError();
}

int gram_panel_rows(int n, int op) {
  if (gram_use_thread(n, op)) return gram_thread_chunk_rows(n, op);
  const int nb = gram_remainder_variant(n, op) ? n / 8 : (n + 7) / 8;  // same tables, indexed by the full tiles
#define SQB_CASE(NBV)                                                                   \
  case NBV:                                                                              \
    return op == OP_PLAIN ? GramCfg<NBV, OP_PLAIN>::P                                    \
                          : (op == OP_SOLVE ? GramCfg<NBV, OP_SOLVE>::P : GramCfg<NBV, OP_MULTIPLY>::P);
  switch (nb) {
    SQB_CASE(2) SQB_CASE(3) SQB_CASE(4) SQB_CASE(5) SQB_CASE(6) SQB_CASE(7)
    default: return op == OP_PLAIN ? GramCfg<8, OP_PLAIN>::P
                                   : (op == OP_SOLVE ? GramCfg<8, OP_SOLVE>::P : GramCfg<8, OP_MULTIPLY>::P);
  }
#undef SQB_CASE
}

int gram_warps(int n) {
  return 8;
}

int gram_ctas_per_sm(int n, int op) {
  if (gram_use_thread(n, op)) return gram_thread_ctas_per_sm(n, op);
  const int nb = gram_remainder_variant(n, op) ? n / 8 : (n + 7) / 8;
  if (SQB_GRAM_2CTA_NB2 && op != OP_PLAIN && nb == 2) return 2;
  if (op != OP_PLAIN) return (SQB_GRAM_2CTA && SQB_GRAM_2CTA_ALL && nb == 4) ? 2 : 1;
  return (SQB_GRAM_2CTA && (nb == 3 || nb == 4)) ? 2 : 1;
}

}  // namespace sqb
