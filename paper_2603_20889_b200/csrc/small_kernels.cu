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
// The Jacobi kernels scale their thread count with n: a round of the 64 x 64 problem rotates 2 x 2048
// column / row entries of A and U, which 256 threads walk in 8 trips between CTA barriers.
constexpr int kJacobiMaxThreads = 1024;
// one warp per rotation pair of a round (n/2 pairs), at most 32 warps
inline int jacobi_threads(int n) {
  const int warps = (n + 1) / 2;
  return warps <= 8 ? 256 : (warps <= 16 ? 512 : (warps <= 24 ? 768 : 1024));
}
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
  const int ld = n + 1;
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
// time; here the n/2 disjoint rotations J = J_1 ... J_{n/2} of a round-robin round are applied together
// as one two-sided update A <- J^T A J.
//
// One CTA, everything in shared memory:
//   * A is kept as its packed upper triangle (a(i, j), i <= j, at j (j + 1) / 2 + i): 66 KB at 128 columns,
//     which leaves room for the full U (132 KB) beside it - no global-memory U, no second pass.
//   * A round = (1) one THREAD per pair derives (c, s) and writes the exact 2 x 2 result of its own diagonal
//     block (gram_qr.cpp:84-87); (2) after a barrier one thread per unordered PAIR OF PAIRS (P, Q) updates the
//     2 x 2 block A[P, Q] <- J_P^T (A[P, Q] J_Q) - four loads, 16 flops, four stores, each entry of the
//     triangle touched once - while the warps rotate the columns of U; (3) barrier.
//   The former column-phase / row-phase formulation over a full square A touched every entry twice with
//   ~8 integer instructions per FMA and was ISSUE bound: 23.6 M warp instructions, 10 300 clk per round at
//   n = 128 (ncu, round 2); this one issues about a quarter of that.
// Returns false when the sweep cap is hit.  On return lam[j] = eigenvalue at index j, perm[j] = source
// index of output j, and column perm[j] of U the eigenvector.
// ------------------------------------------------------------------------------------------------
// The rotation scalars are a serial chain of two divisions, a square root and a reciprocal square root
// per round; the IEEE software sequences for those cost ~3000 clk per round.  MUFU seed + two Newton steps
// each (<= 1-2 ulp) take a tenth of that; the eigen-decomposition is compared through its invariants,
// never bitwise.
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

struct JacobiScratch {
  double* cs;      // np/2
  double* sn;      // np/2
  int2* pq;        // np/2: the (p, q), p < q, of pair t in this round
  double* red;     // 32
  int* perm;       // n
  double* lam;     // n: the eigenvalues by index (diagonal of the converged A)
  unsigned* blk;   // (np/2)(np/2 - 1)/2: the unordered pairs (tP < tQ) of pair slots, (tP << 16) | tQ
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
// `a`: packed upper triangle of order np = n rounded up to even, entries (i <= j < n) filled by the caller.
__device__ bool jacobi_eigh(double* a, double* u, int ldu, int n, const JacobiScratch& js, bool want_vectors = true) {
  const int tid = threadIdx.x, nt_ = blockDim.x;
  const int warp = tid >> 5, lane = tid & 31, nwarps = nt_ >> 5;
  const int np = (n + 1) & ~1;
  const int half = np / 2;
  const int nblk = half * (half - 1) / 2;

  // the block list: the strict upper triangle of the half x half slot grid, folded into half/2 rows of
  // half - 1 entries (row r of the triangle together with row half - 1 - r)
  for (int k = tid; k < nblk; k += nt_) {
    const int r = k / (half - 1), c = k % (half - 1);
    int tp, tq;
    if (c < half - 1 - r) {
      tp = r;
      tq = r + 1 + c;
    } else {
      tp = half - 1 - r;
      tq = tp + 1 + (c - (half - 1 - r));
    }
    js.blk[k] = (static_cast<unsigned>(tp) << 16) | static_cast<unsigned>(tq);
  }
  if (np > n) {  // padding index n: zero row/column, never rotated (a_pq == 0 rule)
    for (int i = tid; i < np; i += nt_) a[tri_at(i, n)] = 0.0;
  }
  // |C|_F and identity U
  double fro = 0.0;
  for (int idx = tid; idx < n * n; idx += nt_) {
    const int i = idx % n, j = idx / n;
    if (i <= j) {
      const double v = a[tri_at(i, j)];
      fro = fma(i == j ? v : 2.0 * v, v, fro);
    }
    if (want_vectors) u[i + j * ldu] = i == j ? 1.0 : 0.0;
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
    for (int step = 0; step < np - 1; ++step) {
      // (1) rotation of pair slot t (round-robin: slot 0 keeps index np - 1)
      if (tid < half) {
        const int t = tid;
        int x, y;
        if (t == 0) {
          x = np - 1;
          y = step;
        } else {
          x = (step + t) % (np - 1);
          y = (step - t + (np - 1)) % (np - 1);
        }
        const int p = min(x, y), q = max(x, y);
        const int ipp = ((p * (p + 1)) >> 1) + p, iqq = ((q * (q + 1)) >> 1) + q, ipq = ((q * (q + 1)) >> 1) + p;
        const double apq = a[ipq];
        double cs = 1.0, sn = 0.0;
        if (apq != 0.0) {
          const double app = a[ipp], aqq = a[iqq];
          const double theta = (aqq - app) * fast_rcp(2.0 * apq);
          const double ath = fabs(theta);
          double tt;
          if (ath < 1e100) {
            const double r2 = fma(theta, theta, 1.0);
            const double y2 = fast_rsqrt(r2);
            double sq = r2 * y2;
            sq = fma(fma(-sq, sq, r2), 0.5 * y2, sq);  // sqrt(1 + theta^2), residual-corrected
            tt = (theta >= 0.0 ? 1.0 : -1.0) * fast_rcp(ath + sq);
          } else {
            tt = 0.5 / theta;  // sqrt(1 + theta^2) == |theta| in working precision (also theta = +-inf)
          }
          cs = fast_rsqrt(fma(tt, tt, 1.0));
          sn = tt * cs;
          a[ipp] = app - tt * apq;  // the exact 2 x 2 results (gram_qr.cpp:84-87)
          a[iqq] = aqq + tt * apq;
          a[ipq] = 0.0;
        }
        js.cs[t] = cs;
        js.sn[t] = sn;
        js.pq[t] = make_int2(p, q);
      }
      __syncthreads();
      // (2a) off-diagonal blocks: A[P, Q] <- J_P^T (A[P, Q] J_Q).  An unrotated pair has (c, s) = (1, 0): exact.
      for (int k = tid; k < nblk; k += nt_) {
        const unsigned e = js.blk[k];
        const int tp = e >> 16, tq = e & 0xffffu;
        const int2 P = js.pq[tp], Q = js.pq[tq];
        const double cp = js.cs[tp], sp = js.sn[tp], cq = js.cs[tq], sq = js.sn[tq];
        const int i00 = tri_at(P.x, Q.x), i01 = tri_at(P.x, Q.y), i10 = tri_at(P.y, Q.x), i11 = tri_at(P.y, Q.y);
        const double a00 = a[i00], a01 = a[i01], a10 = a[i10], a11 = a[i11];
        const double b00 = cq * a00 - sq * a01, b01 = sq * a00 + cq * a01;  // columns: . J_Q
        const double b10 = cq * a10 - sq * a11, b11 = sq * a10 + cq * a11;
        a[i00] = cp * b00 - sp * b10;                                       // rows: J_P^T .
        a[i10] = sp * b00 + cp * b10;
        a[i01] = cp * b01 - sp * b11;
        a[i11] = sp * b01 + cp * b11;
      }
      // (2b) U <- U J: a warp per pair, lanes over the rows
      if (want_vectors) {
        for (int t = warp; t < half; t += nwarps) {
          const double cs = js.cs[t], sn = js.sn[t];
          if (sn == 0.0) continue;  // identity (this also keeps the padding index out of U)
          const int2 P = js.pq[t];
          double* up = u + P.x * ldu;
          double* uq = u + P.y * ldu;
          for (int i = lane; i < n; i += 32) {
            const double uip = up[i], uiq = uq[i];
            up[i] = cs * uip - sn * uiq;
            uq[i] = sn * uip + cs * uiq;
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
  const int np = (n + 1) & ~1;
  const int half = np / 2;
  L.ldu = n + 1;
  L.a_off = 0;
  size_t off = (static_cast<size_t>(np) * (np + 1) / 2 + 1) & ~static_cast<size_t>(1);
  L.u_off = off;
  off += (static_cast<size_t>(n) * L.ldu + 1) & ~static_cast<size_t>(1);
  L.misc_off = off;
  // cs, sn, pq (half each), red (32), perm (n ints), lam (n), blk (half (half - 1) / 2 unsigned)
  off += 3 * half + 32 + (n + 1) / 2 + 2 + np + (static_cast<size_t>(half) * (half - 1) / 2 + 1) / 2 + 2;
  L.total_doubles = off;
  return L;
}

__device__ JacobiScratch carve_scratch(double* sm, const SmallLayout& L, int n) {
  const int np = (n + 1) & ~1;
  const int half = np / 2;
  JacobiScratch js;
  double* p = sm + L.misc_off;
  js.cs = p; p += half;
  js.sn = p; p += half;
  js.pq = reinterpret_cast<int2*>(p); p += half;
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
