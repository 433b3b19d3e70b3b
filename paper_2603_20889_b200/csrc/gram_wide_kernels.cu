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
//   * the CTA streams P-row panels of the chunk's columns through a 4-stage shared-memory
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
constexpr int kTriP = 40;
constexpr int kFullP = 24;
constexpr int kWThreads = 256;   // 8 warps
constexpr int kWStages = 4;      // panels in flight (HBM latency is ~2 panel times)

__device__ __forceinline__ void dmma_w(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

struct WideParams {
  const double* x;
  long long ld, m;
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
template <int W>
__device__ __forceinline__ void tri_panel(const double* stage, double (&acc)[32][2], int g, int q) {
  constexpr int R1 = W, R2 = kWT - 1 - W;
#pragma unroll
  for (int t = 0; t < kTriP / 8; ++t) {
    double2 b[kWT - R1];
#pragma unroll
    for (int j = R1; j < kWT; ++j) b[j - R1] = frag<kTriP>(stage, j, t, g, q);
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
  const bool aligned = ((reinterpret_cast<uintptr_t>(prm.x) & 15) == 0) && ((prm.ld & 1) == 0);
  const double* colp = prm.x + static_cast<long long>(slot_ok ? col : 0) * prm.ld;

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

cudaError_t launch_gram_wide(const double* x, long long m, int n, long long ld, int sm_count, double* partial,
                             double* c, int check_finite, StatusWord* status, cudaStream_t stream) {
  if (n <= 64 || n > kWideGramMaxN) return cudaErrorInvalidValue;
  WideParams prm;
  prm.x = x;
  prm.ld = ld;
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
    // a full chunk costs 256 tile pairs, a triangular one 136: split the SMs in that ratio
    prm.kb_full = (sm_count * 256 + 264) / 528;
    prm.kb_tri = (sm_count - prm.kb_full) / 2;
    grid = 2 * prm.kb_tri + prm.kb_full;
  }
  const long long panels = (m + kTriP - 1) / kTriP;
  if (prm.kb_tri > panels) prm.kb_tri = static_cast<int>(panels > 0 ? panels : 1);
  if (prm.kb_full > panels) prm.kb_full = static_cast<int>(panels > 0 ? panels : 1);
  if (prm.nchunk == 1) grid = prm.kb_tri; else grid = 2 * prm.kb_tri + prm.kb_full;
  const size_t bytes = sizeof(double) * kWStages * (kWC * kTriP > 2 * kWC * kFullP ? kWC * kTriP : 2 * kWC * kFullP);
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(gram_wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(bytes));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  gram_wide_kernel<<<grid, kWThreads, bytes, stream>>>(prm);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  gram_wide_reduce_kernel<<<(n * n + 255) / 256, 256, 0, stream>>>(partial, prm.kb_tri, prm.kb_full, n, c,
                                                                   check_finite, status);
  return cudaGetLastError();
}

}  // namespace sqb
