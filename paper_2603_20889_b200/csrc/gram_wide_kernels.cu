// Wide Gram kernel, 64 < n <= 256 (BASELINE config 5: the transitional regime n = 128 / 256 where
// C = X^T X is a genuine FP64 tensor-core SYRK: 32 / 64 flop per byte against a machine balance of 5).
//
// Reference semantics: tsmttsm -> blocked_gram(plain) (reference src/gram.cpp:23-94, 113-121):
// per-block upper-triangle partials, summed in ascending block order, mirrored.  The reference has
// no column limit for tsmttsm; its cache-resident panel times n(n+1)/2 dot products becomes here:
//
//   * the n x n output is cut into 128-column chunks (16 x 16 tiles of 8 x 8).  A CTA owns one chunk
//     pair (ci <= cj) and one row block; n = 128 is a single triangular chunk, n = 256 is two
//     triangular chunks plus one full off-diagonal chunk - 32.9 K accumulators do not fit one SM's
//     register file, so the off-diagonal chunk gets its own CTAs (and re-reads its 256 columns).
//   * the CTA streams P-row panels of the chunk's columns through a 3-stage shared-memory
//     stage (cp.async.bulk per column segment, one mbarrier per stage, every thread issues one copy);
//   * every warp owns fixed tile pairs in registers for the whole row block - triangular chunk: tile
//     rows w and 15-w (17 pairs per warp, perfectly balanced); full chunk: tile rows 2w, 2w+1 against
//     all 16 tile columns (32 pairs) - so a fragment is loaded once per 8 rows and reused across the
//     tile row, and no cross-warp reduction is needed;
//   * lane (g,q) holds X[row 2q+e, 8T+g]: at once the A fragment (transposed) and the B fragment of
//     mma.sync.m8n8k4.f64, as in gram_kernels.cu.
#include "kernels.h"

namespace sqb {

namespace {

constexpr int kWT = 16;          // tiles per chunk side
constexpr int kWC = 8 * kWT;     // columns per chunk (128)
// panel rows == stage pitch == 8 (mod 16): conflict-free LDS.128 fragment reads without padding.  The
// triangular chunk stages 128 columns, the full one 256, so the former affords taller panels (fewer
// CTA barriers per row) in the same shared memory.
constexpr int kTriP = 56;
constexpr int kFullP = 24;
constexpr int kWThreads = 256;   // 8 warps
constexpr int kWStages = 3;      // panels in flight (a panel is several us of DMMAs: far more than the HBM latency)

__device__ __forceinline__ void dmma_w(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

struct WideParams {
  MatView x;  // columns [0, n_main) from base (leading dimension ld), the optional last one from `extra`
  long long m;
  int n;
  int kb_tri, kb_full;  // row blocks per triangular / full chunk
  int nchunk;           // 128-column chunks (1 or 2)
  double* partial;      // one 128 x 128 column-major slab per CTA
};

template <int PP>
__device__ __forceinline__ double2 frag(const double* stage, int tile, int t, int g, int q) {
  return *reinterpret_cast<const double2*>(stage + (8 * tile + g) * PP + 8 * t + 2 * q);
}

// Triangular chunk, warp W: tile rows W and 15-W of the 16 x 16 upper block triangle.
template <int W, int PP = kTriP, int ROWS = PP>
__device__ __forceinline__ void tri_panel(const double* stage, double (&acc)[32][2], int g, int q) {
  constexpr int R1 = W, R2 = kWT - 1 - W;
  // the body is replicated once per warp (register-indexed accumulators): keep it to ONE row group per
  // copy so that the eight variants stay resident in the instruction cache (ncu: no_instruction stalls)
#pragma unroll 1
  for (int t = 0; t < ROWS / 8; ++t) {
    double2 b[kWT - R1];
#pragma unroll
    for (int j = R1; j < kWT; ++j) b[j - R1] = frag<PP>(stage, j, t, g, q);
    const double2 a1 = b[0], a2 = b[R2 - R1];
#pragma unroll
    for (int j = R1; j < kWT; ++j) dmma_w(acc[j - R1][0], acc[j - R1][1], a1.x, b[j - R1].x);
#pragma unroll
    for (int j = R2; j < kWT; ++j) dmma_w(acc[kWT - R1 + j - R2][0], acc[kWT - R1 + j - R2][1], a2.x, b[j - R1].x);
#pragma unroll
    for (int j = R1; j < kWT; ++j) dmma_w(acc[j - R1][0], acc[j - R1][1], a1.y, b[j - R1].y);
#pragma unroll
    for (int j = R2; j < kWT; ++j) dmma_w(acc[kWT - R1 + j - R2][0], acc[kWT - R1 + j - R2][1], a2.y, b[j - R1].y);
  }
}

// Full chunk: tile rows 2w, 2w+1 of the I chunk (stage slots 0..127) against the 16 tile columns of
// the J chunk (stage slots 128..255).
__device__ __forceinline__ void full_panel(const double* stage, double (&acc)[32][2], int w, int g, int q) {
#pragma unroll
  for (int t = 0; t < kFullP / 8; ++t) {
    const double2 a1 = frag<kFullP>(stage, 2 * w, t, g, q), a2 = frag<kFullP>(stage, 2 * w + 1, t, g, q);
    double2 b[kWT];
#pragma unroll
    for (int j = 0; j < kWT; ++j) b[j] = frag<kFullP>(stage, kWT + j, t, g, q);
#pragma unroll
    for (int j = 0; j < kWT; ++j) dmma_w(acc[j][0], acc[j][1], a1.x, b[j].x);
#pragma unroll
    for (int j = 0; j < kWT; ++j) dmma_w(acc[kWT + j][0], acc[kWT + j][1], a2.x, b[j].x);
#pragma unroll
    for (int j = 0; j < kWT; ++j) dmma_w(acc[j][0], acc[j][1], a1.y, b[j].y);
#pragma unroll
    for (int j = 0; j < kWT; ++j) dmma_w(acc[kWT + j][0], acc[kWT + j][1], a2.y, b[j].y);
  }
}

template <int W>
__device__ __forceinline__ void tri_store(double* dst, const double (&acc)[32][2], int g, int q) {
  constexpr int R1 = W, R2 = kWT - 1 - W;
#pragma unroll
  for (int j = R1; j < kWT; ++j) {
    double* p = dst + (8 * R1 + g) + static_cast<long long>(8 * j + 2 * q) * kWC;
    p[0] = acc[j - R1][0];
    p[kWC] = acc[j - R1][1];
  }
#pragma unroll
  for (int j = R2; j < kWT; ++j) {
    double* p = dst + (8 * R2 + g) + static_cast<long long>(8 * j + 2 * q) * kWC;
    p[0] = acc[kWT - R1 + j - R2][0];
    p[kWC] = acc[kWT - R1 + j - R2][1];
  }
}

#define SQB_WARP_SWITCH(CALL)  \
  switch (warp) {              \
    case 0: CALL(0); break;    \
    case 1: CALL(1); break;    \
    case 2: CALL(2); break;    \
    case 3: CALL(3); break;    \
    case 4: CALL(4); break;    \
    case 5: CALL(5); break;    \
    case 6: CALL(6); break;    \
    default: CALL(7); break;   \
  }

__global__ void __launch_bounds__(kWThreads, 1) gram_wide_kernel(const WideParams prm) {
  extern __shared__ __align__(128) double smem[];
  __shared__ uint64_t bars[kWStages];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q = lane & 3;

  // which chunk pair and row block
  int ci, cj, kb, rb;
  {
    int b = blockIdx.x;
    if (b < prm.kb_tri) { ci = cj = 0; kb = prm.kb_tri; rb = b; }
    else if (prm.nchunk == 1) return;
    else if (b < 2 * prm.kb_tri) { ci = cj = 1; kb = prm.kb_tri; rb = b - prm.kb_tri; }
    else { ci = 0; cj = 1; kb = prm.kb_full; rb = b - 2 * prm.kb_tri; }
  }
  const bool tri = ci == cj;
  const int nslots = tri ? kWC : 2 * kWC;
  const int kWP = tri ? kTriP : kFullP, kWPP = kWP;  // panel rows and stage pitch of this chunk type
  const int stage_doubles = nslots * kWPP;

  // column of this thread's stage slot (every thread copies one column segment per panel)
  const int slot = tid;
  const int col = slot < kWC ? kWC * ci + slot : kWC * cj + (slot - kWC);
  const bool slot_ok = slot < nslots && col < prm.n;
  int valid_slots = 0;
  for (int s = 0; s < nslots; ++s) valid_slots += ((s < kWC ? kWC * ci + s : kWC * cj + (s - kWC)) < prm.n) ? 1 : 0;

  for (int i = tid; i < kWStages * stage_doubles; i += kWThreads) smem[i] = 0.0;
  if (tid < kWStages) mbar_init(&bars[tid], 1);
  mbar_fence_init();
  __syncthreads();

  // rows of this block: ceil(m / kb) rounded up to whole panels
  long long rpb = (prm.m + kb - 1) / kb;
  rpb = (rpb + kWP - 1) / kWP * kWP;
  const long long begin = min(static_cast<long long>(rb) * rpb, prm.m);
  const long long end = min(static_cast<long long>(rb + 1) * rpb, prm.m);
  const long long npanels = (end - begin + kWP - 1) / kWP;
  const bool aligned = (((reinterpret_cast<uintptr_t>(prm.x.base) | reinterpret_cast<uintptr_t>(prm.x.extra)) & 15) == 0) &&
                       ((prm.x.ld & 1) == 0);
  const double* colp = prm.x.col(slot_ok ? col : 0);

  double acc[32][2];
#pragma unroll
  for (int p = 0; p < 32; ++p) acc[p][0] = acc[p][1] = 0.0;

  uint32_t phase_bits = 0, async_bits = 0;  // per stage: parity to wait for / filled by the async engine
  auto will_be_async = [&](long long pn) { return aligned && begin + pn * kWP + kWP <= end; };
  // called by all threads after a __syncthreads(); thread 0 has armed the barrier for async panels
  auto fill = [&](long long pn, int s) {
    const long long r0 = begin + pn * kWP;
    double* st = smem + s * stage_doubles;
    if (will_be_async(pn)) {
      if (slot_ok) {
        fence_async_smem();
        bulk_g2s(st + slot * kWPP, colp + r0, kWP * sizeof(double), &bars[s]);
      }
      async_bits |= 1u << s;
    } else {
      if (slot_ok) {
        for (int r = 0; r < kWP; ++r) st[slot * kWPP + r] = (r0 + r < end) ? __ldg(colp + r0 + r) : 0.0;
      }
      async_bits &= ~(1u << s);
    }
  };
  const uint32_t tx_bytes = static_cast<uint32_t>(valid_slots * kWP * sizeof(double));

  // prologue: kWStages - 1 panels in flight
  if (tid == 0) {
    for (int s = 0; s < kWStages - 1; ++s)
      if (s < npanels && will_be_async(s)) mbar_expect_tx(&bars[s], tx_bytes);
  }
  __syncthreads();
  for (int s = 0; s < kWStages - 1; ++s)
    if (s < npanels) fill(s, s);

  for (long long pn = 0; pn < npanels; ++pn) {
    const int s = static_cast<int>(pn % kWStages);
    const long long nxt = pn + kWStages - 1;
    const int sn = static_cast<int>(nxt % kWStages);
    if (tid == 0 && nxt < npanels && will_be_async(nxt)) mbar_expect_tx(&bars[sn], tx_bytes);
    __syncthreads();  // stage sn is free (panel pn-1 consumed), its barrier is armed, sync fills visible
    if (nxt < npanels) fill(nxt, sn);
    if (async_bits & (1u << s)) {
      mbar_wait(&bars[s], (phase_bits >> s) & 1u);
      phase_bits ^= 1u << s;
    }
    const double* stage = smem + s * stage_doubles;
    if (tri) {
#define SQB_TRI(WV) tri_panel<WV>(stage, acc, g, q)
      SQB_WARP_SWITCH(SQB_TRI)
#undef SQB_TRI
    } else {
      full_panel(stage, acc, warp, g, q);
    }
  }

  // ---- the CTA's partial: 128 x 128 column-major slab, element (i, j) of the chunk at [i + 128 j] ----
  double* dst = prm.partial + static_cast<long long>(blockIdx.x) * kWC * kWC;
  if (tri) {
#define SQB_TRIS(WV) tri_store<WV>(dst, acc, g, q)
    SQB_WARP_SWITCH(SQB_TRIS)
#undef SQB_TRIS
  } else {
#pragma unroll
    for (int j = 0; j < kWT; ++j) {
      double* p = dst + (8 * (2 * warp) + g) + static_cast<long long>(8 * j + 2 * q) * kWC;
      p[0] = acc[j][0];
      p[kWC] = acc[j][1];
      double* p2 = dst + (8 * (2 * warp + 1) + g) + static_cast<long long>(8 * j + 2 * q) * kWC;
      p2[0] = acc[kWT + j][0];
      p2[kWC] = acc[kWT + j][1];
    }
  }
}

// ------------------------------------------------------------------------------------------------
// Fused solve + Gram for 64 < n <= 128: the second CholQR2 sweep, C2 = (X R^-1)^T (X R^-1), with no Q
// write-back (reference tsmRttsmR -> blocked_gram(solve), src/gram.cpp:123-140, 57-62).
//
// The reference substitutes column by column inside a cache-resident panel; a column-sequential
// substitution across 128 columns would serialise the eight warps of a CTA, so here the triangular
// solve is turned into a tensor-core GEMM with the explicit inverse U = R^-1 (rinv_wide_kernel, one
// CTA, 40 us): per 32-row panel
//     Q^T tile (8 columns j x 8 rows)  =  sum_{k <= j}  U^T[8j.., 4k..] * X^T[4k.., rows]     (DMMA)
// whose accumulator fragment (lane (g,q): Q[row 2q+e, column 8j+g]) is exactly the operand layout of
// the SYRK (tri_panel), so it goes to a shared Q panel with one conflict-free 128-bit store and the
// SYRK of gram_wide_kernel runs on it unchanged.  Warp w forms tile columns w and 15-w (34 k-steps,
// the same balance as the SYRK's 17 tile pairs); its U fragments sit in shared memory in issue order.
// The Q panel is double-buffered and the SYRK runs one panel behind the GEMM: one CTA barrier per
// panel.  Same forward error class as the substitution (|dQ| <~ n eps |X| |R^-1|); deviation noted
// in DESIGN.md.
// ------------------------------------------------------------------------------------------------
// Panel geometry per variant.  The solve GEMM reads the X stage with the transposed LDS.64 pattern
// ((4k+q) * pitch + 8t + g): conflict-free for pitch = 4 or 12 (mod 16); the SYRK reads the Q panel with
// the LDS.128 pattern ((8T+g) * pitch + 8t + 2q): conflict-free for pitch = 8 (mod 16).
// `wq` (WRITEQ: Q goes to global memory, no shared Q panels and no SYRK accumulators) lets the dense
// factor afford the 32-row panels too.
__host__ __device__ constexpr int fused_rows(int op, bool wq = false) { return (op == OP_SOLVE || wq) ? 32 : 16; }
__host__ __device__ constexpr int fused_spitch(int op, bool wq = false) { return (op == OP_SOLVE || wq) ? 36 : 20; }
__host__ __device__ constexpr int fused_qpitch(int op) { return op == OP_SOLVE ? 40 : 24; }
// k4 steps per warp: triangular factor (OP_SOLVE, U = R^-1) (2w+2) + (32-2w) = 34; dense factor
// (OP_MULTIPLY, B) 32 + 32
__host__ __device__ constexpr int fused_ksteps(int op) { return op == OP_SOLVE ? 34 : 64; }
__host__ __device__ constexpr int fused_k1(int op, int w) { return op == OP_SOLVE ? 2 * w + 2 : 32; }
__host__ __device__ constexpr int fused_k2(int op, int w) { return op == OP_SOLVE ? 2 * (kWT - 1 - w) + 2 : 32; }
__host__ __device__ constexpr int fused_frag_doubles(int op) { return 8 * fused_ksteps(op) * 32; }
// panels in flight: the fused passes are far on the tensor-pipe side (a panel is ~5 us of DMMAs), so a
// two-stage ring is enough; the shared memory goes to taller panels (solve) / the dense factor's 128 KB
// of fragments (multiply) instead
__host__ __device__ constexpr int fused_stages(int) { return 2; }
__host__ __device__ constexpr size_t fused_smem_doubles(int op, bool wq = false) {
  return static_cast<size_t>(fused_stages(op)) * kWC * fused_spitch(op, wq) + (wq ? 0 : 2 * kWC * fused_qpitch(op)) +
         fused_frag_doubles(op);
}
constexpr double kEpsW = 2.220446049250313e-16;

// Factor element held by lane (g,q) of warp w at issue step f: tile column w for the first k1 steps,
// tile column 15-w after; row 4k+q, column 8j+g.
template <int OP>
__device__ __forceinline__ void fused_frag_coord(int idx, int* row, int* col) {
  const int lane = idx & 31, f = (idx >> 5) % fused_ksteps(OP), w = idx / (32 * fused_ksteps(OP));
  const int g = lane >> 2, q = lane & 3;
  const int k1 = fused_k1(OP, w);
  const int j = f < k1 ? w : kWT - 1 - w;
  const int kk = f < k1 ? f : f - k1;
  *row = 4 * kk + q;
  *col = 8 * j + g;
}

// OP_MULTIPLY: B (n x n, dense) into fragment order; tsmmttsmm validates B (gram.cpp:143-145).
__global__ void bfrag_wide_kernel(const double* __restrict__ b, int n, double* __restrict__ frags,
                                  StatusWord* status) {
  for (int idx = threadIdx.x + blockIdx.x * blockDim.x; idx < fused_frag_doubles(OP_MULTIPLY);
       idx += blockDim.x * gridDim.x) {
    int row, col;
    fused_frag_coord<OP_MULTIPLY>(idx, &row, &col);
    double v = 0.0;
    if (row < n && col < n) {
      v = b[row + static_cast<long long>(col) * n];
      if (is_nonfinite(v)) atomicExch(&status->nonfinite, 1);
    }
    frags[idx] = v;
  }
}

// Block (row0.., col0..) of a dense column-major matrix `a` (leading dimension ld; rows x cols live
// entries, zero beyond) into the fused kernel's fragment order; OP_SOLVE keeps the upper triangle of
// the block only.  Used by the 128 < n <= 256 drivers, whose factor is cut into 128 x 128 blocks.
template <int OP>
__global__ void frag_from_dense_kernel(const double* __restrict__ a, long long ld, int row0, int col0, int rows,
                                       int cols, double* __restrict__ frags) {
  for (int idx = threadIdx.x + blockIdx.x * blockDim.x; idx < fused_frag_doubles(OP); idx += blockDim.x * gridDim.x) {
    int row, col;
    fused_frag_coord<OP>(idx, &row, &col);
    const bool live = row < rows && col < cols && (OP == OP_MULTIPLY || row <= col);
    frags[idx] = live ? a[(row0 + row) + static_cast<long long>(col0 + col) * ld] : 0.0;
  }
}

// c += d (n x n): the row-slab partial sums of the 256-column drivers, added in ascending slab order
__global__ void add_square_kernel(double* __restrict__ c, const double* __restrict__ d, int count) {
  for (int idx = threadIdx.x + blockIdx.x * blockDim.x; idx < count; idx += blockDim.x * gridDim.x) c[idx] += d[idx];
}

// U = R^-1 by back substitution, thread j owns column j; written in the fused kernel's fragment order:
// warp w, step f (f < 2w+2: tile column w, k-step f; else tile column 15-w, k-step f-2w-2),
// lane (g,q): U[4k+q, 8j+g].  Also the reference's pre-check |R(j,j)| > n eps max|diag| (gram.cpp:126-134).
__global__ void __launch_bounds__(128, 1)
    rinv_wide_kernel(const double* __restrict__ r, int n, double* __restrict__ frags, StatusWord* status) {
  extern __shared__ __align__(16) double sm[];
  double* rp = sm;                       // packed upper triangle of R
  double* u = sm + tri_size(kWC);        // U[k * 128 + j]
  __shared__ double mx_s;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < kWC * kWC; idx += 128) {
    const int i = idx % kWC, j = idx / kWC;
    if (i <= j) rp[tri_index(i, j)] = (j < n) ? r[i + static_cast<long long>(j) * n] : (i == j ? 1.0 : 0.0);
    u[idx] = 0.0;
  }
  __syncthreads();
  if (tid < 32) {
    double mx = 0.0;
    for (int j = tid; j < n; j += 32) mx = fmax(mx, fabs(rp[tri_index(j, j)]));
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (tid == 0) mx_s = mx;
  }
  __syncthreads();
  if (tid == 0) {
    const double dtol = static_cast<double>(n) * kEpsW * mx_s;
    for (int j = 0; j < n; ++j)
      if (fabs(rp[tri_index(j, j)]) <= dtol) {
        raise_status(status, SQB_E_SINGULAR, j);
        break;
      }
  }
  {  // row i of U needs rows i+1.. of U only in the own column: no barrier; i is warp-uniform so the
     // R entries are broadcasts and the U reads are lane-contiguous
    const int j = tid;
    if (j < n) u[j * kWC + j] = 1.0 / rp[tri_index(j, j)];
    for (int i = n - 2; i >= 0; --i) {
      if (j > i && j < n) {
        double s0 = 0.0, s1 = 0.0;
        int k = i + 1;
        for (; k + 1 <= j; k += 2) {
          s0 = fma(rp[tri_index(i, k)], u[k * kWC + j], s0);
          s1 = fma(rp[tri_index(i, k + 1)], u[(k + 1) * kWC + j], s1);
        }
        if (k <= j) s0 = fma(rp[tri_index(i, k)], u[k * kWC + j], s0);
        u[i * kWC + j] = -(s0 + s1) / rp[tri_index(i, i)];
      }
    }
  }
  __syncthreads();
  for (int idx = tid; idx < fused_frag_doubles(OP_SOLVE); idx += 128) {
    int row, col;
    fused_frag_coord<OP_SOLVE>(idx, &row, &col);
    frags[idx] = (row <= col && col < n) ? u[row * kWC + col] : 0.0;
  }
}

// Q^T tiles of tile columns w and 15-w for the row groups of a panel.  Lane (g,q) ends up with
// Q[row 8t+2q+e, column 8J+g] in a?c[t][e].  One loop with run-time bounds for all warps (the warp index
// only sets the trip counts), so the GEMM half of the kernel is not replicated eight times in the
// instruction cache like the register-indexed SYRK has to be.
template <int OP, bool WQ = false>
__device__ __forceinline__ void solve_tiles(const double* stage, const double* rf, double (&a1c)[fused_rows(OP, WQ) / 8][2],
                                            double (&a2c)[fused_rows(OP, WQ) / 8][2], int w, int kmax, int lane, int g,
                                            int q) {
  constexpr int NT = fused_rows(OP, WQ) / 8, SP = fused_spitch(OP, WQ);
  // kmax = ceil(n / 4): columns of X beyond n are zero, so are the factor rows beyond n
  const int k1 = min(fused_k1(OP, w), kmax), k2 = min(fused_k2(OP, w), kmax);
#pragma unroll
  for (int t = 0; t < NT; ++t) a1c[t][0] = a1c[t][1] = a2c[t][0] = a2c[t][1] = 0.0;
  const double* rf1 = rf + w * fused_ksteps(OP) * 32 + lane;
  const double* rf2 = rf1 + fused_k1(OP, w) * 32;
  const double* sb = stage + q * SP + g;
  int kk = 0;
#pragma unroll 2
  for (; kk < k1; ++kk) {  // both tile columns (k1 <= k2)
    double b[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) b[t] = sb[4 * kk * SP + 8 * t];
    const double a2 = rf2[kk * 32], a1 = rf1[kk * 32];
#pragma unroll
    for (int t = 0; t < NT; ++t) dmma_w(a2c[t][0], a2c[t][1], a2, b[t]);
#pragma unroll
    for (int t = 0; t < NT; ++t) dmma_w(a1c[t][0], a1c[t][1], a1, b[t]);
  }
#pragma unroll 2
  for (; kk < k2; ++kk) {  // the longer column only (triangular factor)
    double b[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) b[t] = sb[4 * kk * SP + 8 * t];
    const double a2 = rf2[kk * 32];
#pragma unroll
    for (int t = 0; t < NT; ++t) dmma_w(a2c[t][0], a2c[t][1], a2, b[t]);
  }
}

// ... to the shared Q panel in the SYRK's operand layout (one conflict-free 128-bit store per tile)
template <int OP>
__device__ __forceinline__ void solve_panel(const double* stage, const double* rf, double* qb, int n, int w,
                                            int lane, int g, int q) {
  constexpr int NT = fused_rows(OP) / 8, QP = fused_qpitch(OP);
  const int j1 = w, j2 = kWT - 1 - w;
  double a1c[NT][2], a2c[NT][2];
  solve_tiles<OP>(stage, rf, a1c, a2c, w, (n + 3) / 4, lane, g, q);
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    *reinterpret_cast<double2*>(qb + (8 * j1 + g) * QP + 8 * t + 2 * q) = make_double2(a1c[t][0], a1c[t][1]);
    *reinterpret_cast<double2*>(qb + (8 * j2 + g) * QP + 8 * t + 2 * q) = make_double2(a2c[t][0], a2c[t][1]);
  }
}

// ... or to global memory (reconstruct_q): a lane writes two consecutive rows of one column, the four
// lanes of a column 64 contiguous bytes
template <int OP>
__device__ __forceinline__ void solve_panel_out(const double* stage, const double* rf, double* qout, long long ldq,
                                                long long r0, long long end, int n, int n_out, int accumulate,
                                                int w, int lane, int g, int q) {
  constexpr int NT = fused_rows(OP, true) / 8;
  const int j1 = w, j2 = kWT - 1 - w;
  double a1c[NT][2], a2c[NT][2];
  solve_tiles<OP, true>(stage, rf, a1c, a2c, w, (n + 3) / 4, lane, g, q);
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    const long long row = r0 + 8 * t + 2 * q;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      if (row + e < end) {
        double* p1 = qout + row + e + static_cast<long long>(8 * j1 + g) * ldq;
        double* p2 = qout + row + e + static_cast<long long>(8 * j2 + g) * ldq;
        if (8 * j1 + g < n_out) *p1 = accumulate ? *p1 + a1c[t][e] : a1c[t][e];
        if (8 * j2 + g < n_out) *p2 = accumulate ? *p2 + a2c[t][e] : a2c[t][e];
      }
    }
  }
}

struct WideSolveParams {
  MatView x;
  long long m;
  int n, kb;
  const double* frags;  // U = R^-1 (rinv_wide_kernel) or B (bfrag_wide_kernel) in fragment order
  double* partial;      // one 128 x 128 column-major slab per CTA
  double* qout;         // WRITEQ: Q = X U goes here (leading dimension ldq) and no Gram is formed
  long long ldq;
  int n_out;            // WRITEQ: live output columns (<= 128); n counts the live X columns (the K extent)
  int accumulate;       // WRITEQ: add to what qout holds (second K block of a 256-column product)
};

template <int OP, bool WRITEQ>
__global__ void __launch_bounds__(kWThreads, 1) gram_wide_fused_kernel(const WideSolveParams prm) {
  extern __shared__ __align__(128) double smem[];
  constexpr int NSTAGE = fused_stages(OP), P = fused_rows(OP, WRITEQ), SP = fused_spitch(OP, WRITEQ);
  __shared__ uint64_t bars[NSTAGE];
  constexpr int kQPitch = fused_qpitch(OP);
  constexpr int kStageDoubles = kWC * SP, kQDoubles = WRITEQ ? 0 : kWC * kQPitch;
  double* qbuf = smem + NSTAGE * kStageDoubles;  // two Q panels
  double* rf = qbuf + 2 * kQDoubles;             // factor fragments
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, q = lane & 3;
  const int rb = blockIdx.x;

  const int slot = tid;
  const bool slot_ok = slot < kWC && slot < prm.n;
  const int valid_slots = prm.n < kWC ? prm.n : kWC;

  for (int i = tid; i < NSTAGE * kStageDoubles + 2 * kQDoubles; i += kWThreads) smem[i] = 0.0;
  for (int i = tid; i < fused_frag_doubles(OP); i += kWThreads) rf[i] = prm.frags[i];
  if (tid < NSTAGE) mbar_init(&bars[tid], 1);
  mbar_fence_init();
  __syncthreads();

  long long rpb = (prm.m + prm.kb - 1) / prm.kb;
  rpb = (rpb + P - 1) / P * P;
  const long long begin = min(static_cast<long long>(rb) * rpb, prm.m);
  const long long end = min(static_cast<long long>(rb + 1) * rpb, prm.m);
  const long long npanels = (end - begin + P - 1) / P;
  const bool aligned = (((reinterpret_cast<uintptr_t>(prm.x.base) | reinterpret_cast<uintptr_t>(prm.x.extra)) & 15) == 0) &&
                       ((prm.x.ld & 1) == 0);
  const double* colp = prm.x.col(slot_ok ? slot : 0);

  double acc[32][2];
#pragma unroll
  for (int p = 0; p < 32; ++p) acc[p][0] = acc[p][1] = 0.0;

  uint32_t phase_bits = 0, async_bits = 0;
  auto will_be_async = [&](long long pn) { return aligned && begin + pn * P + P <= end; };
  auto fill = [&](long long pn, int s) {
    const long long r0 = begin + pn * P;
    double* st = smem + s * kStageDoubles;
    if (will_be_async(pn)) {
      if (slot_ok) {
        fence_async_smem();
        bulk_g2s(st + slot * SP, colp + r0, P * sizeof(double), &bars[s]);
      }
      async_bits |= 1u << s;
    } else {
      if (slot_ok) {
        for (int r = 0; r < P; ++r) st[slot * SP + r] = (r0 + r < end) ? __ldg(colp + r0 + r) : 0.0;
      }
      async_bits &= ~(1u << s);
    }
  };
  const uint32_t tx_bytes = static_cast<uint32_t>(valid_slots * P * sizeof(double));

  if (tid == 0) {
    for (int s = 0; s < NSTAGE - 1; ++s)
      if (s < npanels && will_be_async(s)) mbar_expect_tx(&bars[s], tx_bytes);
  }
  __syncthreads();
  for (int s = 0; s < NSTAGE - 1; ++s)
    if (s < npanels) fill(s, s);

  // iteration pn: SYRK of panel pn-1 (from its Q panel), then the solve GEMM of panel pn
  for (long long pn = 0; pn <= npanels; ++pn) {
    const int s = static_cast<int>(pn % NSTAGE);
    const long long nxt = pn + NSTAGE - 1;
    const int sn = static_cast<int>(nxt % NSTAGE);
    if (tid == 0 && nxt < npanels && will_be_async(nxt)) mbar_expect_tx(&bars[sn], tx_bytes);
    __syncthreads();  // GEMM(pn-1) done everywhere: stage sn free, Q panel (pn-1)&1 complete; SYRK(pn-2) done
    if (nxt < npanels) fill(nxt, sn);
    if (!WRITEQ && pn > 0) {
      const double* qp = qbuf + ((pn - 1) & 1) * kQDoubles;
#define SQB_TRI(WV) tri_panel<WV, kQPitch, P>(qp, acc, g, q)
      SQB_WARP_SWITCH(SQB_TRI)
#undef SQB_TRI
    }
    if (pn < npanels) {
      if (async_bits & (1u << s)) {
        mbar_wait(&bars[s], (phase_bits >> s) & 1u);
        phase_bits ^= 1u << s;
      }
      const double* stage = smem + s * kStageDoubles;
      if (WRITEQ)
        solve_panel_out<OP>(stage, rf, prm.qout, prm.ldq, begin + pn * P, end, prm.n, prm.n_out, prm.accumulate, warp,
                            lane, g, q);
      else solve_panel<OP>(stage, rf, qbuf + (pn & 1) * kQDoubles, prm.n, warp, lane, g, q);
    }
  }
  if (WRITEQ) return;

  double* dst = prm.partial + static_cast<long long>(blockIdx.x) * kWC * kWC;
#define SQB_TRIS(WV) tri_store<WV>(dst, acc, g, q)
  SQB_WARP_SWITCH(SQB_TRIS)
#undef SQB_TRIS
}

// Sum the row-block partials of every chunk in ascending block order, mirror (gram.cpp:81-92).
__global__ void gram_wide_reduce_kernel(const double* partial, int kb_tri, int kb_full, int n, double* c,
                                        int check_finite, StatusWord* status) {
  for (int idx = threadIdx.x + blockIdx.x * blockDim.x; idx < n * n; idx += blockDim.x * gridDim.x) {
    const int i = idx % n, j = idx / n;
    if (i > j) continue;
    const int ci = i / kWC, cj = j / kWC;
    int first, count;
    if (ci == cj) { first = ci * kb_tri; count = kb_tri; }
    else { first = 2 * kb_tri; count = kb_full; }
    const long long off = (i % kWC) + static_cast<long long>(j % kWC) * kWC;
    double s = 0.0;
    for (int b = 0; b < count; ++b) s += partial[static_cast<long long>(first + b) * kWC * kWC + off];
    c[i + static_cast<long long>(j) * n] = s;
    c[j + static_cast<long long>(i) * n] = s;
    if (check_finite && is_nonfinite(s)) atomicExch(&status->nonfinite, 1);
  }
}

}  // namespace

size_t gram_wide_partial_doubles(int n, int sm_count) {
  (void)n;
  return static_cast<size_t>(sm_count + 2) * kWC * kWC;
}

cudaError_t launch_gram_wide(const MatView& x, long long m, int n, int sm_count, double* partial,
                             double* c, int check_finite, StatusWord* status, cudaStream_t stream) {
  if (n <= 64 || n > kWideGramMaxN) return cudaErrorInvalidValue;
  WideParams prm;
  prm.x = x;
  prm.m = m;
  prm.n = n;
  prm.nchunk = (n + kWC - 1) / kWC;
  prm.partial = partial;
  int grid;
  if (prm.nchunk == 1) {
    prm.kb_tri = sm_count;
    prm.kb_full = 0;
    grid = sm_count;
  } else {
    // a full chunk costs 256 tile pairs, a triangular one 136 (and runs ~10 % faster per pair: taller
    // panels, rolled row-group loop): split the SMs in that ratio
    prm.kb_full = (sm_count * 256 + 250) / 500;
    prm.kb_tri = (sm_count - prm.kb_full) / 2;
    grid = 2 * prm.kb_tri + prm.kb_full;
  }
  const long long panels = (m + kTriP - 1) / kTriP;
  if (prm.kb_tri > panels) prm.kb_tri = static_cast<int>(panels > 0 ? panels : 1);
  if (prm.kb_full > panels) prm.kb_full = static_cast<int>(panels > 0 ? panels : 1);
  if (prm.nchunk == 1) grid = prm.kb_tri; else grid = 2 * prm.kb_tri + prm.kb_full;
  const size_t bytes = sizeof(double) * kWStages * (kWC * kTriP > 2 * kWC * kFullP ? kWC * kTriP : 2 * kWC * kFullP);
  static unsigned long long smem_ready = 0;  // per-device opt-in mask
  {
    cudaError_t e = opt_in_dynamic_smem(gram_wide_kernel, bytes, &smem_ready);
    if (e != cudaSuccess) return e;
  }
  gram_wide_kernel<<<grid, kWThreads, bytes, stream>>>(prm);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  gram_wide_reduce_kernel<<<(n * n + 255) / 256, 256, 0, stream>>>(partial, prm.kb_tri, prm.kb_full, n, c,
                                                                   check_finite, status);
  return cudaGetLastError();
}

size_t gram_wide_fused_scratch_doubles() { return fused_frag_doubles(OP_MULTIPLY); }

template <int OP, bool WRITEQ = false>
static cudaError_t launch_fused(const WideSolveParams& prm, cudaStream_t stream) {
  const size_t bytes = sizeof(double) * fused_smem_doubles(OP, WRITEQ);
  static unsigned long long smem_ready = 0;  // per-device opt-in mask
  {
    cudaError_t e = opt_in_dynamic_smem(gram_wide_fused_kernel<OP, WRITEQ>, bytes, &smem_ready);
    if (e != cudaSuccess) return e;
  }
  gram_wide_fused_kernel<OP, WRITEQ><<<prm.kb, kWThreads, bytes, stream>>>(prm);
  return cudaGetLastError();
}

static cudaError_t launch_rinv_wide(const double* r, int n, double* frags, StatusWord* status, cudaStream_t stream) {
  const size_t rinv_bytes = sizeof(double) * (tri_size(kWC) + kWC * kWC);
  static unsigned long long smem_ready = 0;  // per-device opt-in mask
  {
    cudaError_t e = opt_in_dynamic_smem(rinv_wide_kernel, rinv_bytes, &smem_ready);
    if (e != cudaSuccess) return e;
  }
  rinv_wide_kernel<<<1, 128, rinv_bytes, stream>>>(r, n, frags, status);
  return cudaGetLastError();
}

static WideSolveParams fused_params(const MatView& x, long long m, int n, const double* frags, int sm_count,
                                    int op, bool wq = false) {
  WideSolveParams prm;
  prm.x = x;
  prm.m = m;
  prm.n = n;
  prm.frags = frags;
  prm.partial = nullptr;
  prm.qout = nullptr;
  prm.ldq = 0;
  prm.n_out = n;
  prm.accumulate = 0;
  const long long panels = (m + fused_rows(op, wq) - 1) / fused_rows(op, wq);
  prm.kb = static_cast<int>(panels < sm_count ? (panels > 0 ? panels : 1) : sm_count);
  return prm;
}

cudaError_t launch_gram_wide_fused(const MatView& x, long long m, int n, int op, const double* factor,
                                   int sm_count, double* frags, double* partial, double* c, StatusWord* status,
                                   cudaStream_t stream) {
  if (n <= 64 || n > kWideFusedMaxN || (op != OP_SOLVE && op != OP_MULTIPLY)) return cudaErrorInvalidValue;
  cudaError_t e;
  if (op == OP_SOLVE) {
    e = launch_rinv_wide(factor, n, frags, status, stream);
  } else {
    bfrag_wide_kernel<<<16, 256, 0, stream>>>(factor, n, frags, status);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) return e;
  WideSolveParams prm = fused_params(x, m, n, frags, sm_count, op);
  prm.partial = partial;
  e = op == OP_SOLVE ? launch_fused<OP_SOLVE>(prm, stream) : launch_fused<OP_MULTIPLY>(prm, stream);
  if (e != cudaSuccess) return e;
  gram_wide_reduce_kernel<<<(n * n + 255) / 256, 256, 0, stream>>>(partial, prm.kb, 0, n, c, 0, status);
  return cudaGetLastError();
}

// Q = X R^-1 for 64 < n <= 128 (reference reconstruct_q, src/gram_qr.cpp:193-221): the same solve GEMM,
// tiles written straight to Q.
cudaError_t launch_apply_rinv_wide(const double* x, long long m, int n, long long ld, const double* r,
                                   int sm_count, double* frags, double* q, long long ldq, StatusWord* status,
                                   cudaStream_t stream) {
  if (n <= 64 || n > kWideFusedMaxN) return cudaErrorInvalidValue;
  cudaError_t e = launch_rinv_wide(r, n, frags, status, stream);
  if (e != cudaSuccess) return e;
  WideSolveParams prm = fused_params(MatView{x, ld, nullptr, n}, m, n, frags, sm_count, OP_SOLVE, true);
  prm.qout = q;
  prm.ldq = ldq;
  return launch_fused<OP_SOLVE, true>(prm, stream);
}

// ---- 128 < n <= 256: the Gram-based methods at BASELINE config 5's upper column count ---------------------
// At 256 columns the sweep is 64 flop per byte of X - an order of magnitude past the machine balance - and
// the factor (512 KB) no longer fits beside the stages, so Q = X F is formed explicitly, 128 output columns
// and 128 contraction columns at a time, with the same fused GEMM kernel writing to a row-slab buffer, and
// the wide SYRK runs on that slab.  The extra traffic (Q written once, read by the SYRK) is about a fifth
// of the tensor-pipe time of the sweep; no m x n intermediate ever exists, only the slab.
size_t gram_wide2_scratch_doubles(int n) {
  return 2 * static_cast<size_t>(n) * n + 4 * static_cast<size_t>(fused_frag_doubles(OP_MULTIPLY));
}

// Q(rows [0, m), 256 columns) = X F for F = R^-1 (OP_SOLVE) or B (OP_MULTIPLY); frag sets f00, f01, f10, f11
static cudaError_t wide2_apply(const MatView& x, long long m, int n, int op, const double* const f[4], int sm_count,
                               double* q, long long ldq, cudaStream_t stream) {
  const int n1 = n - kWC;
  const MatView x0{x.base, x.ld, nullptr, kWC};
  const MatView x1{x.base + static_cast<long long>(kWC) * x.ld, x.ld, nullptr, n1};
  auto run = [&](const MatView& xv, int ncols, const double* frags, bool tri, double* qo, int n_out, int acc) {
    WideSolveParams prm = fused_params(xv, m, ncols, frags, sm_count, tri ? OP_SOLVE : OP_MULTIPLY, true);
    prm.qout = qo;
    prm.ldq = ldq;
    prm.n_out = n_out;
    prm.accumulate = acc;
    return tri ? launch_fused<OP_SOLVE, true>(prm, stream) : launch_fused<OP_MULTIPLY, true>(prm, stream);
  };
  const bool tri = op == OP_SOLVE;
  cudaError_t e = run(x0, kWC, f[0], tri, q, kWC, 0);                                  // Q0  = X0 F00
  if (e == cudaSuccess && !tri) e = run(x1, n1, f[2], false, q, kWC, 1);               // Q0 += X1 F10
  if (e == cudaSuccess) e = run(x0, kWC, f[1], false, q + kWC * ldq, n1, 0);           // Q1  = X0 F01
  if (e == cudaSuccess) e = run(x1, n1, f[3], tri, q + kWC * ldq, n1, 1);              // Q1 += X1 F11
  return e;
}

// factor (n x n column-major: R or B) -> the four 128 x 128 fragment sets in `scratch`
static cudaError_t wide2_factor(const double* factor, int n, int op, double* scratch, const double* f[4],
                                StatusWord* status, cudaStream_t stream) {
  const size_t nn = static_cast<size_t>(n) * n;
  double* fr = scratch + 2 * nn;
  const size_t fd = fused_frag_doubles(OP_MULTIPLY);
  const int n1 = n - kWC;
  const double* dense = factor;
  if (op == OP_SOLVE) {
    cudaError_t e = launch_rinv_global(factor, n, scratch, scratch + nn, status, stream);
    if (e != cudaSuccess) return e;
    dense = scratch + nn;
    frag_from_dense_kernel<OP_SOLVE><<<64, 256, 0, stream>>>(dense, n, 0, 0, kWC, kWC, fr);
    frag_from_dense_kernel<OP_SOLVE><<<64, 256, 0, stream>>>(dense, n, kWC, kWC, n1, n1, fr + 3 * fd);
  } else {
    frag_from_dense_kernel<OP_MULTIPLY><<<64, 256, 0, stream>>>(dense, n, 0, 0, kWC, kWC, fr);
    frag_from_dense_kernel<OP_MULTIPLY><<<64, 256, 0, stream>>>(dense, n, kWC, 0, n1, kWC, fr + 2 * fd);
    frag_from_dense_kernel<OP_MULTIPLY><<<64, 256, 0, stream>>>(dense, n, kWC, kWC, n1, n1, fr + 3 * fd);
  }
  frag_from_dense_kernel<OP_MULTIPLY><<<64, 256, 0, stream>>>(dense, n, 0, kWC, kWC, n1, fr + fd);
  for (int i = 0; i < 4; ++i) f[i] = fr + i * fd;
  return cudaGetLastError();
}

cudaError_t launch_gram_wide2_fused(const MatView& x, long long m, int n, int op, const double* factor, int sm_count,
                                    double* scratch, double* qslab, long long slab_rows, double* partial,
                                    double* c_tmp, double* c, StatusWord* status, cudaStream_t stream,
                                    long long* launches) {
  if (n <= kWC || n > kWideGramMaxN || (op != OP_SOLVE && op != OP_MULTIPLY) || slab_rows < 8) return cudaErrorInvalidValue;
  const double* f[4];
  cudaError_t e = wide2_factor(factor, n, op, scratch, f, status, stream);
  if (e != cudaSuccess) return e;
  *launches += 6;
  e = cudaMemsetAsync(c, 0, sizeof(double) * n * n, stream);
  for (long long r0 = 0; r0 < m && e == cudaSuccess; r0 += slab_rows) {
    const long long rows = m - r0 < slab_rows ? m - r0 : slab_rows;
    const MatView xs{x.base + r0, x.ld, nullptr, n};
    e = wide2_apply(xs, rows, n, op, f, sm_count, qslab, slab_rows, stream);
    if (e != cudaSuccess) break;
    e = launch_gram_wide(MatView{qslab, slab_rows, nullptr, n}, rows, n, sm_count, partial, c_tmp, 0, status, stream);
    if (e != cudaSuccess) break;
    add_square_kernel<<<64, 256, 0, stream>>>(c, c_tmp, n * n);
    e = cudaGetLastError();
    *launches += (op == OP_SOLVE ? 3 : 4) + 3;
  }
  return e;
}

// Q = X R^-1 for 128 < n <= 256 (reference reconstruct_q, gram_qr.cpp:193-221), straight into q
cudaError_t launch_apply_rinv_wide2(const double* x, long long m, int n, long long ld, const double* r, int sm_count,
                                    double* scratch, double* q, long long ldq, StatusWord* status,
                                    cudaStream_t stream) {
  if (n <= kWC || n > kWideGramMaxN) return cudaErrorInvalidValue;
  const double* f[4];
  cudaError_t e = wide2_factor(r, n, OP_SOLVE, scratch, f, status, stream);
  if (e != cudaSuccess) return e;
  return wide2_apply(MatView{x, ld, nullptr, n}, m, n, OP_SOLVE, f, sm_count, q, ldq, stream);
}

}  // namespace sqb
