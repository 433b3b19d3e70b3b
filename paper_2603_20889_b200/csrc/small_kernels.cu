// n x n factorisations and products, one CTA each, so that the Gram-based drivers never leave the
// device between their two streaming passes.
//
//   cholesky_kernel     reference cholesky            (src/gram_qr.cpp:36-58)
//   eigh_kernel         reference eigh_small          (src/gram_qr.cpp:60-121)
//   svqb_pass_kernel    reference svqb_pass           (src/gram_qr.cpp:133-176)
//   tri_multiply        reference triangular_multiply (src/small.cpp:9-20)
//   small_multiply      reference small_multiply      (src/small.cpp:22-32)
//   backsolve_kernel    reference solve_lstsq tail    (src/lstsq.cpp:44-59)
//   apply_rinv_kernel   reference reconstruct_q       (src/gram_qr.cpp:193-221)
#include <algorithm>
#include <cfloat>

#include "kernels.h"

namespace sqb {

namespace {

constexpr int kSmallThreads = 256;
constexpr int kJacobiMaxThreads = 512;
// a thread per pair of index groups (<= 496 at 128 columns) and a warp per group (<= 32), at 128 registers
inline int jacobi_threads(int n) { return n <= 32 ? 256 : 512; }
constexpr double kEps = 2.220446049250313e-16;  // std::numeric_limits<double>::epsilon()
constexpr int kJacobiMaxSweeps = 30;               // gram_qr.cpp:69

// ------------------------------------------------------------------------------------------------
// Cholesky: right-looking, upper factor R^T R = C.  Arithmetic per entry is the reference's
// (subtract r_ki r_kj for ascending k, divide by r_ii, sqrt of the reduced pivot); breakdown when
// the reduced pivot is <= n*eps*max_j|c_jj| (gram_qr.cpp:39-54), reported with its column index.
// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kSmallThreads)
    cholesky_kernel(const double* __restrict__ c, int n, double* __restrict__ r, StatusWord* status) {
  extern __shared__ __align__(16) double sm[];
  const int ld = n | 1;  // odd pitch: the row walk a[k + i * ld] of the rank-1 update is conflict-free (an even
                         // pitch made odd n twice as slow: 0.27 ms at n = 127 against 0.14 ms at n = 128)
  double* a = sm;
  __shared__ double tol_s;
  __shared__ int fail_s;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < n * n; idx += kSmallThreads) {
    const int i = idx % n, j = idx / n;
    a[i + j * ld] = c[idx];
  }
  __syncthreads();
  if (tid < 32) {  // max |c_jj| from the shared copy (a serial walk over global memory costs ~0.5 us per entry)
    double mx = 0.0;
    for (int j = tid; j < n; j += 32) mx = fmax(mx, fabs(a[j + j * ld]));
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (tid == 0) {
      tol_s = static_cast<double>(n) * kEps * mx;
      fail_s = -1;
    }
  }
  __syncthreads();
  const double tol = tol_s;
  const int tx = tid & 15, ty = tid >> 4;
  for (int k = 0; k < n; ++k) {
    const double d = a[k + k * ld];
    if (d <= tol) {
      if (tid == 0) {
        fail_s = k;
        raise_status(status, SQB_E_BREAKDOWN, k);
      }
      break;
    }
    const double rkk = sqrt(d);
    __syncthreads();
    if (tid == 0) a[k + k * ld] = rkk;
    for (int j = k + 1 + tid; j < n; j += kSmallThreads) a[k + j * ld] = a[k + j * ld] / rkk;
    __syncthreads();
    for (int j = k + 1 + ty; j < n; j += 16) {
      const double rkj = a[k + j * ld];
      for (int i = k + 1 + tx; i <= j; i += 16) a[i + j * ld] = fma(-a[k + i * ld], rkj, a[i + j * ld]);
    }
    __syncthreads();
  }
  __syncthreads();
  const bool failed = fail_s >= 0;
  for (int idx = tid; idx < n * n; idx += kSmallThreads) {
    const int i = idx % n, j = idx / n;
    r[idx] = (i <= j && !failed) ? a[i + j * ld] : 0.0;
  }
}

// Cholesky beyond 128 columns (the reference's cholesky has no column limit, gram_qr.cpp:36-58; BASELINE
// config 5 names n = 256): the matrix no longer fits one CTA's shared memory, so it is factored in place
// in the output buffer (L2-resident, n = 256 is 512 KB) by one 1024-thread CTA, right-looking, row k staged
// in shared memory for the rank-1 update.  Same per-entry operation order and breakdown rule as above.
constexpr int kCholGlobalThreads = 1024;
__global__ void __launch_bounds__(kCholGlobalThreads)
    cholesky_global_kernel(const double* __restrict__ c, int n, double* __restrict__ r, StatusWord* status) {
  extern __shared__ __align__(16) double rowk[];  // n doubles
  __shared__ double tol_s, red_s[32];
  __shared__ int fail_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double mx = 0.0;
  for (int idx = tid; idx < n * n; idx += kCholGlobalThreads) {
    const int i = idx % n, j = idx / n;
    const double v = c[idx];
    r[idx] = i <= j ? v : 0.0;
    if (i == j) mx = fmax(mx, fabs(v));
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) red_s[warp] = mx;
  __syncthreads();
  if (tid == 0) {
    double m2 = 0.0;
    for (int w = 0; w < kCholGlobalThreads / 32; ++w) m2 = fmax(m2, red_s[w]);
    tol_s = static_cast<double>(n) * kEps * m2;
    fail_s = -1;
  }
  __syncthreads();
  const double tol = tol_s;
  const int tx = tid & 31, ty = tid >> 5;
  for (int k = 0; k < n; ++k) {
    const double d = r[k + static_cast<long long>(k) * n];
    if (d <= tol) {
      if (tid == 0) {
        fail_s = k;
        raise_status(status, SQB_E_BREAKDOWN, k);
      }
      break;
    }
    const double rkk = sqrt(d);
    __syncthreads();  // everyone has read the pivot
    for (int j = k + tid; j < n; j += kCholGlobalThreads) {
      const double v = j == k ? rkk : r[k + static_cast<long long>(j) * n] / rkk;
      r[k + static_cast<long long>(j) * n] = v;
      rowk[j] = v;
    }
    __syncthreads();
    for (int j = k + 1 + ty; j < n; j += 32) {
      const double rkj = rowk[j];
      double* col = r + static_cast<long long>(j) * n;
      for (int i = k + 1 + tx; i <= j; i += 32) col[i] = fma(-rowk[i], rkj, col[i]);
    }
    __syncthreads();
  }
  __syncthreads();
  if (fail_s >= 0)
    for (int idx = tid; idx < n * n; idx += kCholGlobalThreads) r[idx] = 0.0;
}

// U = R^-1 for an upper triangular R of any order (the explicit inverse the wide fused sweeps multiply
// with, see gram_wide_kernels.cu), one CTA, thread j owns column j: back substitution up the column.
// `urm` is n x n scratch holding U row-major (the threads of a warp then touch consecutive addresses);
// the result is written column-major to `u`.  Also the reference's pre-check
// |R(j,j)| > n eps max|diag| (gram.cpp:126-134).
__global__ void __launch_bounds__(256)
    rinv_global_kernel(const double* __restrict__ r, int n, double* __restrict__ urm, double* __restrict__ u,
                       StatusWord* status) {
  __shared__ double red_s[8];
  __shared__ double mx_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double mx = 0.0;
  for (int j = tid; j < n; j += 256) mx = fmax(mx, fabs(r[j + static_cast<long long>(j) * n]));
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) red_s[warp] = mx;
  __syncthreads();
  if (tid == 0) {
    double m2 = 0.0;
    for (int w = 0; w < 8; ++w) m2 = fmax(m2, red_s[w]);
    mx_s = m2;
    const double dtol = static_cast<double>(n) * kEps * m2;
    for (int j = 0; j < n; ++j)
      if (fabs(r[j + static_cast<long long>(j) * n]) <= dtol) {
        raise_status(status, SQB_E_SINGULAR, j);
        break;
      }
  }
  for (int j = tid; j < n; j += 256) {
    for (int i = n - 1; i > j; --i) urm[static_cast<long long>(i) * n + j] = 0.0;
    urm[static_cast<long long>(j) * n + j] = 1.0 / r[j + static_cast<long long>(j) * n];
    for (int i = j - 1; i >= 0; --i) {
      double s0 = 0.0, s1 = 0.0;
      int k = i + 1;
      for (; k + 1 <= j; k += 2) {
        s0 = fma(r[i + static_cast<long long>(k) * n], urm[static_cast<long long>(k) * n + j], s0);
        s1 = fma(r[i + static_cast<long long>(k + 1) * n], urm[static_cast<long long>(k + 1) * n + j], s1);
      }
      if (k <= j) s0 = fma(r[i + static_cast<long long>(k) * n], urm[static_cast<long long>(k) * n + j], s0);
      urm[static_cast<long long>(i) * n + j] = -(s0 + s1) / r[i + static_cast<long long>(i) * n];
    }
  }
  __syncthreads();
  for (int idx = tid; idx < n * n; idx += 256) {
    const int i = idx % n, j = idx / n;
    u[idx] = urm[static_cast<long long>(i) * n + j];
  }
}

// ------------------------------------------------------------------------------------------------
// Symmetric eigensolver: Jacobi with the reference's rotation formulas, skip rule (a_pq == 0),
// stopping test off(A) <= 10*n*eps*|C|_F checked once per sweep, 30-sweep cap and stable
// descending sort (gram_qr.cpp:60-121).  The reference sweeps cyclic-by-row, one rotation at a
// time; here a sweep is a TWO-LEVEL round-robin: the indices form blocks of two, the blocks are paired
// round-robin, and a block pair (I, J) = indices (a, b | c, d) is a GROUP that performs, back to back,
//     set 0 (first block round of a sweep only):  (a, b), (c, d)      - the pairs inside the blocks
//     set 1:  (a, c), (b, d)            set 2:  (a, d), (b, c)
// so that every index pair is rotated once per sweep (np - 1 sets of np/2 disjoint rotations, the same count
// as a plain round-robin), but A and U are read and written once per BLOCK round instead of once per set.
//
// One CTA, everything in shared memory:
//   * A is kept as its packed upper triangle (a(i, j), i <= j, at j (j + 1) / 2 + i): 66 KB at 128 columns,
//     which leaves room for the full U (132 KB) beside it.
//   * A block round = (1) one THREAD per group loads its 4 x 4 diagonal block, derives the two or three sets of
//     rotations from it (the two rotations of a set are independent chains the compiler interleaves) and
//     writes the block back; (2) after a barrier one thread per unordered PAIR OF GROUPS (G, H) updates the
//     4 x 4 block A[G, H] <- J_G^T A[G, H] J_H (16 loads, 128-192 flops, 16 stores; every entry of the triangle
//     touched once) while a warp per group rotates four columns of U; (3) barrier.
//   History (ncu, n = 128): column phase / row phase over a full square A with U in global memory: 23.6 M
//   warp instructions, 7.9 ms, issue bound; one thread per 2 x 2 block pair, one set per round: 10.6 M, 3.1 ms,
//   shared-memory pipe 84 % busy (U alone 40 % of the wavefronts) - hence the grouping.
// Returns false when the sweep cap is hit.  On return lam[j] = eigenvalue at index j, perm[j] = source
// index of output j, and column perm[j] of U the eigenvector.
// ------------------------------------------------------------------------------------------------
// The rotation scalars are a serial chain of two divisions, a square root and a reciprocal square root;
// the IEEE software sequences for those cost ~3000 clk.  MUFU seed + two Newton steps each (<= 1-2 ulp)
// take a tenth of that; the eigen-decomposition is compared through its invariants, never bitwise
// (DESIGN.md, section 2).
__device__ __forceinline__ double fast_rcp(double x) {
  double z;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(z) : "d"(x));
  double e = fma(-x, z, 1.0);
  z = fma(z, e, z);
  e = fma(-x, z, 1.0);
  return fma(z, e, z);
}
__device__ __forceinline__ double fast_rsqrt(double x) {  // x in [1, 1e200]
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y;
}

// Rotation annihilating a_pq (gram_qr.cpp:74-83), branch-free: a_pq == 0 gives the identity (t = 0).
__device__ __forceinline__ void jacobi_params(double app, double aqq, double apq, double& cs, double& sn, double& tt) {
  const bool rot = apq != 0.0;
  const double theta = (aqq - app) * fast_rcp(2.0 * (rot ? apq : 1.0));
  const double ath = fabs(theta);
  const double r2 = fma(theta, theta, 1.0);
  const double y2 = fast_rsqrt(r2);
  double sq = r2 * y2;
  sq = fma(fma(-sq, sq, r2), 0.5 * y2, sq);  // sqrt(1 + theta^2), residual-corrected
  const double t_small = (theta >= 0.0 ? 1.0 : -1.0) * fast_rcp(ath + sq);
  // sqrt(1 + theta^2) == |theta| in working precision: t = 1 / (2 theta) (0 once that underflows)
  const double t_big = ath < 1e300 ? fast_rcp(2.0 * (ath < 1e300 ? theta : 1.0)) : 0.0;
  const double t = ath < 1e100 ? t_small : t_big;
  const double c = fast_rsqrt(fma(t, t, 1.0));
  tt = rot ? t : 0.0;
  cs = rot ? c : 1.0;
  sn = rot ? t * c : 0.0;
}

__device__ __forceinline__ void jrot(double& x, double& y, double c, double s) {
  const double nx = c * x - s * y;
  y = s * x + c * y;
  x = nx;
}

// The rotation sets of a group on a 4-vector over its indices (a row of A[., G] / U[., G] or a column of A[G, .])
__device__ __forceinline__ void apply_sets(double& v0, double& v1, double& v2, double& v3, const double* __restrict__ c,
                                           const double* __restrict__ s, bool intra) {
  if (intra) {
    jrot(v0, v1, c[0], s[0]);
    jrot(v2, v3, c[1], s[1]);
  }
  jrot(v0, v2, c[2], s[2]);
  jrot(v1, v3, c[3], s[3]);
  jrot(v0, v3, c[4], s[4]);
  jrot(v1, v2, c[5], s[5]);
}

// Two disjoint rotations (X0, Y0), (X1, Y1) of the symmetric 4 x 4 diagonal block, two-sided, with the exact
// 2 x 2 results (gram_qr.cpp:84-87)
template <int X0, int Y0, int X1, int Y1>
__device__ __forceinline__ void diag_set(double (&m)[4][4], double* c, double* s) {
  double t0, t1;
  jacobi_params(m[X0][X0], m[Y0][Y0], m[X0][Y0], c[0], s[0], t0);
  jacobi_params(m[X1][X1], m[Y1][Y1], m[X1][Y1], c[1], s[1], t1);
  const double p0 = m[X0][X0] - t0 * m[X0][Y0], q0 = m[Y0][Y0] + t0 * m[X0][Y0];
  const double p1 = m[X1][X1] - t1 * m[X1][Y1], q1 = m[Y1][Y1] + t1 * m[X1][Y1];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    jrot(m[r][X0], m[r][Y0], c[0], s[0]);
    jrot(m[r][X1], m[r][Y1], c[1], s[1]);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    jrot(m[X0][k], m[Y0][k], c[0], s[0]);
    jrot(m[X1][k], m[Y1][k], c[1], s[1]);
  }
  m[X0][X0] = p0;
  m[Y0][Y0] = q0;
  m[X1][X1] = p1;
  m[Y1][Y1] = q1;
  if (t0 != 0.0) m[X0][Y0] = m[Y0][X0] = 0.0;
  if (t1 != 0.0) m[X1][Y1] = m[Y1][X1] = 0.0;
}

struct JacobiScratch {
  double* rc;      // G x 6: cosines of the group's rotations, set-major
  double* rs;      // G x 6: sines
  int2* gb;        // G: the block pair (I < J) of group slot t in this block round
  double* red;     // 32
  int* perm;       // n
  double* lam;     // n: the eigenvalues by index (diagonal of the converged A)
  unsigned* blk;   // G (G - 1) / 2: the unordered pairs (tG < tH) of group slots, (tG << 16) | tH
};

__device__ __forceinline__ int tri_at(int i, int j) {  // packed upper triangle, either order
  const int hi = max(i, j), lo = min(i, j);
  return ((hi * (hi + 1)) >> 1) + lo;
}

__device__ double block_sum(double v, double* red) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double out = 0.0;
  for (int w = 0; w < nw; ++w) out += red[w];  // every thread, same order: a CTA-uniform result
  __syncthreads();
  return out;
}

// want_vectors = false skips U altogether (the sigma eigensolve of an SVQB pass only needs the eigenvalues).
// `a`: packed upper triangle of order np = n rounded up to a multiple of 4, entries (i <= j < n) filled by the
// caller; `u`: n rows x np columns, pitch ldu.
__device__ bool jacobi_eigh(double* a, double* u, int ldu, int n, const JacobiScratch& js, bool want_vectors = true) {
  const int tid = threadIdx.x, nt_ = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31, nwarps = nt_ >> 5;
  const int np = (n + 3) & ~3;
  const int nb2 = np / 2;      // index blocks of two
  const int ng = nb2 / 2;      // groups (block pairs) per block round
  const int nblk = ng * (ng - 1) / 2;

  // the list of group pairs: the strict upper triangle of the ng x ng slot grid, folded into ng/2 rows of
  // ng - 1 entries (row r of the triangle together with row ng - 1 - r)
  for (int k = tid; k < nblk; k += nt_) {
    const int r = k / (ng - 1), c = k % (ng - 1);
    int tg, th;
    if (c < ng - 1 - r) {
      tg = r;
      th = r + 1 + c;
    } else {
      tg = ng - 1 - r;
      th = tg + 1 + (c - (ng - 1 - r));
    }
    js.blk[k] = (static_cast<unsigned>(tg) << 16) | static_cast<unsigned>(th);
  }
  // padding indices n .. np - 1: zero rows / columns, never rotated (a_pq == 0 rule)
  for (int idx = ((n * (n + 1)) >> 1) + tid; idx < ((np * (np + 1)) >> 1); idx += nt_) a[idx] = 0.0;
  // |C|_F and identity U
  double fro = 0.0;
  for (int idx = tid; idx < n * n; idx += nt_) {
    const int i = idx % n, j = idx / n;
    if (i <= j) {
      const double v = a[tri_at(i, j)];
      fro = fma(i == j ? v : 2.0 * v, v, fro);
    }
  }
  if (want_vectors)
    for (int idx = tid; idx < n * np; idx += nt_) {
      const int i = idx % n, j = idx / n;
      u[i + j * ldu] = i == j ? 1.0 : 0.0;
    }
  const double thr = 10.0 * static_cast<double>(n) * kEps * sqrt(block_sum(fro, js.red));

  auto offdiag = [&]() {
    double s = 0.0;
    for (int j = 1 + warp; j < n; j += nwarps) {
      const double* col = a + ((j * (j + 1)) >> 1);
      for (int i = lane; i < j; i += 32) s = fma(col[i], col[i], s);
    }
    return sqrt(2.0 * block_sum(s, js.red));
  };

  bool converged = offdiag() <= thr;
  for (int sweep = 0; sweep < kJacobiMaxSweeps && !converged; ++sweep) {
    for (int step = 0; step < nb2 - 1; ++step) {
      const bool intra = step == 0;
      // (1) the group's rotations from its 4 x 4 diagonal block (round-robin over blocks: slot 0 keeps the last)
      if (tid < ng) {
        const int t = tid;
        int x, y;
        if (t == 0) {
          x = nb2 - 1;
          y = step;
        } else {
          x = (step + t) % (nb2 - 1);
          y = (step - t + (nb2 - 1)) % (nb2 - 1);
        }
        const int bi = min(x, y), bj = max(x, y);
        const int g[4] = {2 * bi, 2 * bi + 1, 2 * bj, 2 * bj + 1};  // ascending
        double m[4][4];
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int r = 0; r <= c; ++r) m[r][c] = m[c][r] = a[((g[c] * (g[c] + 1)) >> 1) + g[r]];
        double c6[6], s6[6];
        c6[0] = c6[1] = 1.0;
        s6[0] = s6[1] = 0.0;
        if (intra) diag_set<0, 1, 2, 3>(m, c6, s6);
        diag_set<0, 2, 1, 3>(m, c6 + 2, s6 + 2);
        diag_set<0, 3, 1, 2>(m, c6 + 4, s6 + 4);
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int r = 0; r <= c; ++r) a[((g[c] * (g[c] + 1)) >> 1) + g[r]] = m[r][c];
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          js.rc[t * 6 + k] = c6[k];
          js.rs[t * 6 + k] = s6[k];
        }
        js.gb[t] = make_int2(bi, bj);
      }
      __syncthreads();
      // (2a) off-diagonal blocks: A[G, H] <- J_G^T (A[G, H] J_H), sets in order on either side
      for (int k = tid; k < nblk; k += nt_) {
        const unsigned e = js.blk[k];
        const int tg = e >> 16, th = e & 0xffffu;
        const int2 gbk = js.gb[tg], hbk = js.gb[th];
        const int gblk[2] = {gbk.x, gbk.y}, hblk[2] = {hbk.x, hbk.y};
        int ix[4][4];
        double m[4][4];
#pragma unroll
        for (int rb = 0; rb < 2; ++rb)
#pragma unroll
          for (int cb = 0; cb < 2; ++cb) {
            // the four entries between index blocks gblk[rb] and hblk[cb] (distinct blocks: one is wholly above)
            const int lo = 2 * min(gblk[rb], hblk[cb]), hi = 2 * max(gblk[rb], hblk[cb]);
            const bool row_low = gblk[rb] < hblk[cb];
            const int base0 = ((hi * (hi + 1)) >> 1) + lo, base1 = (((hi + 1) * (hi + 2)) >> 1) + lo;
            // packed (lo + x, hi + y) = base_y + x; (row, col) = (lo + x, hi + y) when the row block is the lower
            ix[2 * rb][2 * cb] = base0;
            ix[2 * rb + 1][2 * cb + 1] = base1 + 1;
            ix[2 * rb][2 * cb + 1] = row_low ? base1 : base0 + 1;
            ix[2 * rb + 1][2 * cb] = row_low ? base0 + 1 : base1;
          }
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) m[r][c] = a[ix[r][c]];
        {
          const double* hc = js.rc + th * 6;
          const double* hs = js.rs + th * 6;
#pragma unroll
          for (int r = 0; r < 4; ++r) apply_sets(m[r][0], m[r][1], m[r][2], m[r][3], hc, hs, intra);
          const double* gc = js.rc + tg * 6;
          const double* gs = js.rs + tg * 6;
#pragma unroll
          for (int c = 0; c < 4; ++c) apply_sets(m[0][c], m[1][c], m[2][c], m[3][c], gc, gs, intra);
        }
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) a[ix[r][c]] = m[r][c];
      }
      // (2b) U <- U J: a warp per group, lanes over the rows
      if (want_vectors) {
        for (int t = warp; t < ng; t += nwarps) {
          const int2 gbk = js.gb[t];
          double* u0 = u + (2 * gbk.x) * ldu;
          double* u2 = u + (2 * gbk.y) * ldu;
          const double* gc = js.rc + t * 6;
          const double* gs = js.rs + t * 6;
          for (int i = lane; i < n; i += 32) {
            double v0 = u0[i], v1 = u0[i + ldu], v2 = u2[i], v3 = u2[i + ldu];
            apply_sets(v0, v1, v2, v3, gc, gs, intra);
            u0[i] = v0;
            u0[i + ldu] = v1;
            u2[i] = v2;
            u2[i + ldu] = v3;
          }
        }
      }
      __syncthreads();
    }
    converged = offdiag() <= thr;
  }
  // eigenvalues by index, then the stable descending rank (gram_qr.cpp:107-110)
  for (int j = tid; j < n; j += nt_) {
    js.lam[j] = a[((j * (j + 1)) >> 1) + j];
    js.perm[j] = j;
  }
  __syncthreads();
  for (int j = tid; j < n; j += nt_) {
    const double lj = js.lam[j];
    int rank = 0;
    for (int i = 0; i < n; ++i) {
      const double li = js.lam[i];
      rank += (li > lj) || (li == lj && i < j);
    }
    js.perm[rank] = j;
  }
  __syncthreads();
  return converged;
}

struct SmallLayout {
  int ldu;
  size_t a_off, u_off, misc_off, total_doubles;
};

__host__ __device__ inline SmallLayout small_layout(int n) {
  SmallLayout L;
  const int np = (n + 3) & ~3;
  const int ng = np / 4;
  L.ldu = n + 1;
  L.a_off = 0;
  size_t off = static_cast<size_t>(np) * (np + 1) / 2;  // even: np is a multiple of 4
  L.u_off = off;
  off += (static_cast<size_t>(np) * L.ldu + 1) & ~static_cast<size_t>(1);
  L.misc_off = off;
  // rc, rs (6 ng each), gb (ng), red (32), perm (n ints), lam (n), blk (ng (ng - 1) / 2 unsigned)
  off += 13 * ng + 32 + (n + 1) / 2 + 2 + np + (static_cast<size_t>(ng) * (ng - 1) / 2 + 1) / 2 + 2;
  L.total_doubles = off;
  return L;
}

__device__ JacobiScratch carve_scratch(double* sm, const SmallLayout& L, int n) {
  const int np = (n + 3) & ~3;
  const int ng = np / 4;
  JacobiScratch js;
  double* p = sm + L.misc_off;
  js.rc = p; p += 6 * ng;
  js.rs = p; p += 6 * ng;
  js.gb = reinterpret_cast<int2*>(p); p += ng;
  js.red = p; p += 32;
  js.perm = reinterpret_cast<int*>(p); p += (n + 1) / 2 + 2;
  js.lam = p; p += np;
  js.blk = reinterpret_cast<unsigned*>(p);
  return js;
}

__global__ void __launch_bounds__(kJacobiMaxThreads)
    eigh_kernel(const double* __restrict__ c, int n, double* values, double* vectors, StatusWord* status) {
  extern __shared__ __align__(16) double sm[];
  const SmallLayout L = small_layout(n);
  double* a = sm + L.a_off;
  double* u = sm + L.u_off;
  const JacobiScratch js = carve_scratch(sm, L, n);
  const int tid = threadIdx.x, nt_ = blockDim.x;
  for (int idx = tid; idx < n * n; idx += nt_) {
    const int i = idx % n, j = idx / n;
    if (i <= j) a[tri_at(i, j)] = c[idx];
  }
  __syncthreads();
  const bool ok = jacobi_eigh(a, u, L.ldu, n, js);
  if (!ok && tid == 0) raise_status(status, SQB_E_NO_CONVERGENCE, -1);
  for (int j = tid; j < n; j += nt_) values[j] = js.lam[js.perm[j]];
  for (int idx = tid; idx < n * n; idx += nt_) {
    const int i = idx % n, j = idx / n;
    vectors[idx] = u[i + js.perm[j] * L.ldu];
  }
}

// One SVQB pass on a Gram matrix (gram_qr.cpp:133-176): D = diag(C)^-1/2 (1 for zero columns),
// eigen-decomposition of D C D, rank = #{lambda >= 10 n eps lambda_max}, B = D U L^-1/2,
// Z = L^1/2 U^T D^-1 with truncated columns/rows exactly zero; sigma = sqrt(max(eig(C), 0)) from a
// second eigen-decomposition of the unscaled Gram matrix - independent of the first, so it runs beside it
// as the launch's second CTA (eigenvalues only).
__global__ void __launch_bounds__(kJacobiMaxThreads)
    svqb_pass_kernel(const double* __restrict__ c, int n, double* bmat, double* z, double* sigma,
                     long long* rank_out, double* gscratch, StatusWord* status) {
  extern __shared__ __align__(16) double sm[];
  const SmallLayout L = small_layout(n);
  double* a = sm + L.a_off;
  double* u = sm + L.u_off;
  double* ds = gscratch;      // n
  double* dsi = ds + n;       // n
  const JacobiScratch js = carve_scratch(sm, L, n);
  __shared__ int rank_s;
  __shared__ int fail_s;
  const int tid = threadIdx.x, nt_ = blockDim.x;

  if (blockIdx.x == 1) {
    for (int idx = tid; idx < n * n; idx += nt_) {
      const int i = idx % n, j = idx / n;
      if (i <= j) a[tri_at(i, j)] = c[idx];
    }
    __syncthreads();
    const bool sok = jacobi_eigh(a, u, L.ldu, n, js, false);
    if (!sok && tid == 0) raise_status(status, SQB_E_NO_CONVERGENCE, -1);
    for (int j = tid; j < n; j += nt_) sigma[j] = sqrt(fmax(js.lam[js.perm[j]], 0.0));
    return;
  }

  for (int j = tid; j < n; j += nt_) {
    const double d = c[j + j * n];
    ds[j] = d > 0.0 ? 1.0 / sqrt(d) : 1.0;
    dsi[j] = d > 0.0 ? sqrt(d) : 1.0;
  }
  if (tid == 0) fail_s = 0;
  __syncthreads();
  for (int idx = tid; idx < n * n; idx += nt_) {
    const int i = idx % n, j = idx / n;
    if (i <= j) a[tri_at(i, j)] = c[idx] * ds[i] * ds[j];
  }
  __syncthreads();
  const bool ok = jacobi_eigh(a, u, L.ldu, n, js);
  if (tid == 0) {
    int rank = 0;
    if (!ok) {
      raise_status(status, SQB_E_NO_CONVERGENCE, -1);
      fail_s = 1;
    } else {
      const double lmax = js.lam[js.perm[0]];
      if (!(lmax > 0.0)) {
        raise_status(status, SQB_E_ZERO_MATRIX, -1);
        fail_s = 1;
      } else {
        const double tol = 10.0 * static_cast<double>(n) * kEps;
        while (rank < n && js.lam[js.perm[rank]] >= tol * lmax) ++rank;
        if (rank == 0) {
          raise_status(status, SQB_E_ZERO_MATRIX, -1);
          fail_s = 1;
        }
      }
    }
    rank_s = rank;
    *rank_out = rank;
  }
  __syncthreads();
  const int rank = rank_s;
  for (int idx = tid; idx < n * n; idx += nt_) {
    const int i = idx % n, j = idx / n;
    double bv = 0.0, zv = 0.0;
    if (j < rank && !fail_s) {
      const int src = js.perm[j];
      const double lam = js.lam[src];
      const double uij = u[i + src * L.ldu];
      bv = ds[i] * uij * (1.0 / sqrt(lam));
      zv = sqrt(lam) * uij * dsi[i];
    }
    bmat[i + j * n] = bv;   // B(i,j)
    z[j + i * n] = zv;      // Z(j,i)
  }
}

// out = A B for upper-triangular A, B (small.cpp:9-20): sum over t in [i, j], ascending.
__global__ void tri_multiply_kernel(const double* __restrict__ a, const double* __restrict__ b, int n,
                                    double* __restrict__ out) {
  for (int idx = threadIdx.x + blockIdx.x * blockDim.x; idx < n * n; idx += blockDim.x * gridDim.x) {
    const int i = idx % n, j = idx / n;
    double s = 0.0;
    if (i <= j)
      for (int t = i; t <= j; ++t) s = fma(a[i + t * n], b[t + j * n], s);
    out[idx] = s;
  }
}

// out = A B, dense n x n (small.cpp:22-32)
__global__ void small_multiply_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                      int n, double* __restrict__ out) {
  for (int idx = threadIdx.x + blockIdx.x * blockDim.x; idx < n * n; idx += blockDim.x * gridDim.x) {
    const int i = idx % n, j = idx / n;
    double s = 0.0;
    for (int t = 0; t < n; ++t) s = fma(a[i + t * n], b[t + j * n], s);
    out[idx] = s;
  }
}

// ------------------------------------------------------------------------------------------------
// Householder QR of a small n x n matrix (reference hhqr_small as used by solve_lstsq's SVQB2 route,
// lstsq.cpp:37-39), n <= 128, one CTA: the 65..128-column complement of the streaming TSQR kernels
// (which stop at 64 columns like tsqr.cpp:188).  Same reflector convention (make_reflector), R is
// sign-normalised (types.cpp:8-14) and its strict lower triangle is exact zero.
// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kSmallThreads)
    hhqr_small_kernel(const double* __restrict__ z, int n, double* __restrict__ r) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[kSmallThreads];
  __shared__ Reflector hs;
  const int ld = n + 1;
  double* a = sm;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int idx = tid; idx < n * n; idx += kSmallThreads) a[idx % n + (idx / n) * ld] = z[idx];
  __syncthreads();
  for (int c = 0; c < n; ++c) {
    double sg = 0.0;
    for (int i = c + 1 + tid; i < n; i += kSmallThreads) sg = fma(a[i + c * ld], a[i + c * ld], sg);
    const double sigma = block_sum(sg, red);
    if (tid == 0) hs = make_reflector(a[c + c * ld], sigma);
    __syncthreads();
    const Reflector h = hs;
    for (int j = c + 1 + warp; j < n; j += kSmallThreads / 32) {  // a warp per trailing column
      double d = 0.0;
      for (int i = c + 1 + lane; i < n; i += 32) d = fma(a[i + c * ld], a[i + j * ld], d);
      for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
      d = h.gamma * fma(h.u0, a[c + j * ld], d);
      for (int i = c + 1 + lane; i < n; i += 32) a[i + j * ld] = fma(-d, a[i + c * ld], a[i + j * ld]);
      __syncwarp();
      if (lane == 0) a[c + j * ld] = fma(-d, h.u0, a[c + j * ld]);
    }
    __syncthreads();
    if (tid == 0) a[c + c * ld] = h.beta;
  }
  __syncthreads();
  for (int idx = tid; idx < n * n; idx += kSmallThreads) {
    const int i = idx % n, j = idx / n;
    double v = 0.0;
    if (i <= j) {
      v = a[i + j * ld];
      if (a[i + i * ld] < 0.0) v = -v;
    }
    r[idx] = v;
  }
}

// Least-squares tail (lstsq.cpp:44-59): back-substitution on the leading n x n block of the
// (n+1) x (n+1) triangle of [A rhs]; residual = |R(n,n)|; RankDeficiencyError(i) when
// |R(i,i)| <= n*eps*max|diag R[0:n]|.
__global__ void backsolve_kernel(const double* __restrict__ r, int ne, double* xsol, double* residual,
                                 StatusWord* status) {
  if (threadIdx.x != 0) return;
  const int n = ne - 1;
  double mx = 0.0;
  for (int j = 0; j < n; ++j) mx = fmax(mx, fabs(r[j + j * ne]));
  const double dtol = static_cast<double>(n) * kEps * mx;
  for (int i = n - 1; i >= 0; --i) {
    const double d = r[i + i * ne];
    if (fabs(d) <= dtol) {
      raise_status(status, SQB_E_RANK_DEFICIENT, i);
      return;
    }
    double s = r[i + n * ne];
    for (int j = i + 1; j < n; ++j) s -= r[i + j * ne] * xsol[j];
    xsol[i] = s / d;
  }
  *residual = fabs(r[n + n * ne]);
}

__global__ void check_finite_kernel(const double* __restrict__ a, long long count, StatusWord* status) {
  uint32_t nf = 0;
  for (long long i = threadIdx.x + static_cast<long long>(blockIdx.x) * blockDim.x; i < count;
       i += static_cast<long long>(blockDim.x) * gridDim.x)
    nf = max(nf, nonfinite_bits(a[i]));
  if (nf >= kNonFiniteHi) atomicExch(&status->nonfinite, 1);
}

// Q = X R^-1, one row per thread, column-oriented substitution with the reciprocal diagonal and
// exact-zero r_ij skipped, i.e. the reference's order (gram_qr.cpp:203-215).
template <int NMAX>
__global__ void __launch_bounds__(128)
    apply_rinv_kernel(const double* __restrict__ x, long long m, int n, long long ld,
                      const double* __restrict__ r, double* __restrict__ qout, long long ldq) {
  __shared__ double rs[NMAX * NMAX];
  __shared__ double inv[NMAX];
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) rs[idx % n + (idx / n) * NMAX] = r[idx];
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += blockDim.x) inv[j] = 1.0 / rs[j + j * NMAX];
  __syncthreads();
  for (long long row = threadIdx.x + static_cast<long long>(blockIdx.x) * blockDim.x; row < m;
       row += static_cast<long long>(blockDim.x) * gridDim.x) {
    double y[NMAX];
#pragma unroll
    for (int j = 0; j < NMAX; ++j) y[j] = j < n ? x[row + j * ld] : 0.0;
#pragma unroll
    for (int j = 0; j < NMAX; ++j) {
      if (j < n) {
        double acc = y[j];
#pragma unroll
        for (int i = 0; i < j; ++i) {
          const double rij = rs[i + j * NMAX];
          if (rij != 0.0) acc = fma(-rij, y[i], acc);
        }
        y[j] = acc * inv[j];
      }
    }
#pragma unroll
    for (int j = 0; j < NMAX; ++j)
      if (j < n) qout[row + j * ldq] = y[j];
  }
}

__global__ void rinv_precheck_kernel(const double* __restrict__ r, int n, StatusWord* status) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double mx = 0.0;
  for (int j = 0; j < n; ++j) mx = fmax(mx, fabs(r[j + j * n]));
  const double dtol = static_cast<double>(n) * kEps * mx;   // trsm_diag_tolerance, gram.cpp:106-111
  for (int j = 0; j < n; ++j)
    if (fabs(r[j + j * n]) <= dtol) {
      raise_status(status, SQB_E_SINGULAR, j);
      return;
    }
}

size_t small_smem_bytes(int n) { return small_layout(n).total_doubles * sizeof(double); }

template <typename K>
cudaError_t opt_in_smem(K kernel, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(bytes));
}

}  // namespace

cudaError_t launch_cholesky(const double* c, int n, double* r, StatusWord* status,
                            cudaStream_t stream) {
  if (n > kSmallMaxN) {
    cholesky_global_kernel<<<1, kCholGlobalThreads, sizeof(double) * n, stream>>>(c, n, r, status);
    return cudaGetLastError();
  }
  const size_t bytes = sizeof(double) * static_cast<size_t>(n) * (n + 1);
  cudaError_t e = opt_in_smem(cholesky_kernel, bytes);
  if (e != cudaSuccess) return e;
  cholesky_kernel<<<1, kSmallThreads, bytes, stream>>>(c, n, r, status);
  return cudaGetLastError();
}

cudaError_t launch_rinv_global(const double* r, int n, double* scratch_rowmajor, double* u, StatusWord* status,
                               cudaStream_t stream) {
  rinv_global_kernel<<<1, 256, 0, stream>>>(r, n, scratch_rowmajor, u, status);
  return cudaGetLastError();
}

size_t small_scratch_doubles(int n) {
  const size_t nn = static_cast<size_t>(n) * n;
  return nn + 3 * static_cast<size_t>(n) + 16;
}

cudaError_t launch_eigh(const double* c, int n, double* values, double* vectors, double* scratch,
                        StatusWord* status, cudaStream_t stream) {
  const size_t bytes = small_smem_bytes(n);
  cudaError_t e = opt_in_smem(eigh_kernel, bytes);
  if (e != cudaSuccess) return e;
  (void)scratch;
  eigh_kernel<<<1, jacobi_threads(n), bytes, stream>>>(c, n, values, vectors, status);
  return cudaGetLastError();
}

cudaError_t launch_svqb_pass(const double* c, int n, double* b, double* z, double* sigma,
                             long long* rank, int want_sigma, double* scratch, StatusWord* status,
                             cudaStream_t stream) {
  const size_t bytes = small_smem_bytes(n);
  cudaError_t e = opt_in_smem(svqb_pass_kernel, bytes);
  if (e != cudaSuccess) return e;
  svqb_pass_kernel<<<want_sigma ? 2 : 1, jacobi_threads(n), bytes, stream>>>(c, n, b, z, sigma, rank, scratch,
                                                                          status);
  return cudaGetLastError();
}

cudaError_t launch_tri_multiply(const double* a, const double* b, int n, double* out,
                                cudaStream_t stream) {
  tri_multiply_kernel<<<n > 64 ? (n * n + 4095) / 4096 : 1, 256, 0, stream>>>(a, b, n, out);
  return cudaGetLastError();
}

cudaError_t launch_small_multiply(const double* a, const double* b, int n, double* out,
                                  cudaStream_t stream) {
  small_multiply_kernel<<<n > 64 ? (n * n + 4095) / 4096 : 1, 256, 0, stream>>>(a, b, n, out);
  return cudaGetLastError();
}

cudaError_t launch_hhqr_small(const double* z, int n, double* r, cudaStream_t stream) {
  if (n < 1 || n > kSmallMaxN) return cudaErrorInvalidValue;
  const size_t bytes = sizeof(double) * static_cast<size_t>(n) * (n + 1);
  cudaError_t e = opt_in_smem(hhqr_small_kernel, bytes);
  if (e != cudaSuccess) return e;
  hhqr_small_kernel<<<1, kSmallThreads, bytes, stream>>>(z, n, r);
  return cudaGetLastError();
}

cudaError_t launch_backsolve(const double* r, int ne, double* xsol, double* residual,
                             StatusWord* status, cudaStream_t stream) {
  backsolve_kernel<<<1, 32, 0, stream>>>(r, ne, xsol, residual, status);
  return cudaGetLastError();
}

cudaError_t launch_check_finite(const double* a, long long count, StatusWord* status,
                                cudaStream_t stream) {
  const int blocks = static_cast<int>(count < 65536 ? 1 : 296);
  check_finite_kernel<<<blocks, 256, 0, stream>>>(a, count, status);
  return cudaGetLastError();
}

cudaError_t launch_apply_rinv(const double* x, long long m, int n, long long ld, const double* r,
                              double* q, long long ldq, StatusWord* status, cudaStream_t stream) {
  rinv_precheck_kernel<<<1, 32, 0, stream>>>(r, n, status);
  const long long want = (m + 127) / 128;
  const int blocks = static_cast<int>(want < 148 * 8 ? (want < 1 ? 1 : want) : 148 * 8);
  if (n <= 8) apply_rinv_kernel<8><<<blocks, 128, 0, stream>>>(x, m, n, ld, r, q, ldq);
  else if (n <= 16) apply_rinv_kernel<16><<<blocks, 128, 0, stream>>>(x, m, n, ld, r, q, ldq);
  else if (n <= 32) apply_rinv_kernel<32><<<blocks, 128, 0, stream>>>(x, m, n, ld, r, q, ldq);
  else if (n <= 64) apply_rinv_kernel<64><<<blocks, 128, 0, stream>>>(x, m, n, ld, r, q, ldq);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

}  // namespace sqb
