// C ABI of the library (include/skinnyqr_b200.h): context, plans, drivers, host-pointer entry
// points and the NCCL-sharded variants.  Everything here is launch orchestration - the arithmetic
// lives in tsqr_kernels.cu / gram_kernels.cu / small_kernels.cu.  There is no CPU fallback: every
// entry point needs a CUDA device.
#include <dlfcn.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <functional>
#include <new>

#include "context.h"
#include "kernels.h"

using namespace sqb;

namespace {

#define SQB_CUDA(expr)                          \
  do {                                          \
    cudaError_t e__ = (expr);                   \
    if (e__ != cudaSuccess) return SQB_E_CUDA;  \
  } while (0)
#define SQB_TRY(expr)             \
  do {                            \
    int s__ = (expr);             \
    if (s__ != SQB_OK) return s__; \
  } while (0)

long long ceil_div(long long a, long long b) { return (a + b - 1) / b; }

int grow(double** buf, size_t* have, size_t want) {
  if (*have >= want) return SQB_OK;
  if (*buf) cudaFree(*buf);
  *buf = nullptr;
  *have = 0;
  SQB_CUDA(cudaMalloc(reinterpret_cast<void**>(buf), want * sizeof(double)));
  *have = want;
  return SQB_OK;
}

int enter(sqb_context* ctx) {
  if (!ctx) return SQB_E_ARGUMENT;
  SQB_CUDA(cudaSetDevice(ctx->device));
  return SQB_OK;
}

struct Plan {
  long long k, b, rpb;
};

// Reference partition (include/skinnyqr/plan.hpp:24-37): rows_per_block = ceil(m/(k*b))*b.
Plan make_plan(long long m, long long k, long long b) {
  Plan p{k, b, 0};
  p.rpb = ceil_div(m, k * b) * b;
  return p;
}

// B200 default for the Householder stream: one CTA per SM (the kernel owns the whole shared
// memory), b = the warp panel height; fewer CTAs when there is not even one panel per warp.
Plan tsqr_plan(const sqb_context* ctx, long long m, int n, long long k, long long b) {
  const long long P = tsqr_panel_rows(n, ctx->tsqr_kind), NW = tsqr_warps(n, ctx->tsqr_kind);
  if (b <= 0) b = P;
  if (k <= 0) k = std::max<long long>(1, std::min<long long>(ctx->sm_count, m / (P * NW)));
  return make_plan(m, k, b);
}

Plan gram_plan(const sqb_context* ctx, long long m, int n, int op, long long k, long long b) {
  const long long P = gram_panel_rows(n, op), NW = gram_warps(n);
  if (b <= 0) b = P;
  if (k <= 0)
    k = std::max<long long>(1, std::min<long long>(ctx->sm_count * gram_ctas_per_sm(n, op), m / (P * NW)));
  return make_plan(m, k, b);
}

MatView plain_view(const double* x, long long ld, int n) { return MatView{x, ld, nullptr, n}; }

int check_shape(long long m, long long n, long long ld, long long nmax) {
  if (n < 1 || m < n) return SQB_E_DIMENSION;  // validate_factorization_input, types.cpp:40-48
  if (n > nmax) return SQB_E_ARGUMENT;         // tsqr.cpp:188
  if (ld < m) return SQB_E_ARGUMENT;
  return SQB_OK;
}

// ---- TSQR on a device view -----------------------------------------------------------------
int launch_tsqr(sqb_context* ctx, const MatView& v, long long m, int n, const Plan& p, double* y,
                long long ldy, bool finalize, bool check) {
  TsqrParams prm;
  prm.x = v;
  prm.m = m;
  prm.n = n;
  prm.rows_per_block = p.rpb;
  prm.y = y;
  prm.ldy = ldy;
  prm.finalize = finalize ? 1 : 0;
  prm.check_finite = check ? 1 : 0;
  prm.status = ctx->d_status;
  prm.kind = ctx->tsqr_kind;
  SQB_CUDA(launch_tsqr_any(prm, p.k, ctx->stream));
  ctx->launches++;
  return SQB_OK;
}

// Reduce a stack of triangles (rows x n, dense column-major, leading dimension ld) to one
// triangle: the reference's stage 2 (tsqr.cpp:193-195), as a short tree of the same kernel.
int reduce_stack(sqb_context* ctx, double* stack, long long rows, long long ld, int n,
                 double* scratch, double* d_r, bool finalize) {
  const long long P = tsqr_panel_rows(n, ctx->tsqr_kind), NW = tsqr_warps(n, ctx->tsqr_kind);
  double* cur = stack;
  double* nxt = scratch;
  while (true) {
    const long long k2 = std::min<long long>(ctx->sm_count, rows / (P * NW * 4));
    if (k2 < 2) break;
    const Plan p = make_plan(rows, k2, P);
    SQB_TRY(launch_tsqr(ctx, plain_view(cur, ld, n), rows, n, p, nxt, k2 * n, false, false));
    std::swap(cur, nxt);
    rows = k2 * n;
    ld = rows;
  }
  const Plan p = make_plan(rows, 1, rows);
  return launch_tsqr(ctx, plain_view(cur, ld, n), rows, n, p, d_r, n, finalize, false);
}

int tsqr_view(sqb_context* ctx, const MatView& v, long long m, int n, long long k, long long b,
              double* d_r, bool finalize) {
  const Plan p = tsqr_plan(ctx, m, n, k, b);
  if (p.k == 1) return launch_tsqr(ctx, v, m, n, p, d_r, n, finalize, true);
  const size_t ydoubles = static_cast<size_t>(p.k) * n * n;
  SQB_TRY(grow(&ctx->work, &ctx->work_doubles, 2 * ydoubles));
  SQB_TRY(launch_tsqr(ctx, v, m, n, p, ctx->work, p.k * n, false, true));
  return reduce_stack(ctx, ctx->work, p.k * n, p.k * n, n, ctx->work + ydoubles, d_r, finalize);
}

// ---- Gram on a device view -----------------------------------------------------------------
int launch_gram_blocks(sqb_context* ctx, const MatView& v, long long m, int n, int op,
                       const double* factor, const Plan& p, double* partial, bool check) {
  GramParams prm;
  prm.x = v;
  prm.m = m;
  prm.n = n;
  prm.rows_per_block = p.rpb;
  prm.factor = factor;
  prm.partial = partial;
  prm.check_finite = check ? 1 : 0;
  prm.status = ctx->d_status;
  SQB_CUDA(launch_gram(prm, op, p.k, ctx->stream));
  ctx->launches++;
  return SQB_OK;
}

int gram_view(sqb_context* ctx, const MatView& v, long long m, int n, int op, const double* factor,
              long long k, long long b, double* d_c, bool check) {
  const Plan p = gram_plan(ctx, m, n, op, k, b);
  SQB_TRY(grow(&ctx->work, &ctx->work_doubles, static_cast<size_t>(p.k) * n * n));
  SQB_TRY(launch_gram_blocks(ctx, v, m, n, op, factor, p, ctx->work, check));
  SQB_CUDA(launch_gram_reduce(ctx->work, p.k, n, d_c, check ? 1 : 0, ctx->d_status, ctx->stream));
  ctx->launches++;
  return SQB_OK;
}

// n x n scratch slots inside ctx->small
struct Small {
  double *c1, *r1, *c2, *r2, *b1, *z1, *b2, *z2, *s2, *rr, *scratch;
  long long* rank1;
};

int small_slots(sqb_context* ctx, int n, Small* s) {
  const size_t nn = static_cast<size_t>(n) * n;
  const size_t want = 10 * nn + 4 * n + small_scratch_doubles(n) + 8;
  SQB_TRY(grow(&ctx->small, &ctx->small_doubles, want));
  double* p = ctx->small;
  s->c1 = p; p += nn;
  s->r1 = p; p += nn;
  s->c2 = p; p += nn;
  s->r2 = p; p += nn;
  s->b1 = p; p += nn;
  s->z1 = p; p += nn;
  s->b2 = p; p += nn;
  s->z2 = p; p += nn;
  s->rr = p; p += 2 * nn;
  s->s2 = p; p += 4 * n;
  s->rank1 = reinterpret_cast<long long*>(p); p += 8;
  s->scratch = p;
  return SQB_OK;
}

// CholQR2 (gram_qr.cpp:123-131): Gram, Cholesky, fused solve+Gram, Cholesky, R = R2 R1 - all
// enqueued back to back, no host round trip.  `second_pass` lets the sharded variant splice an
// all-reduce between the streaming pass and the factorisation.
int cholqr2_view(sqb_context* ctx, const MatView& v, long long m, int n, long long k, long long b,
                 double* d_r, const std::function<int(double*)>& allreduce) {
  Small s;
  SQB_TRY(small_slots(ctx, n, &s));
  SQB_TRY(gram_view(ctx, v, m, n, OP_PLAIN, nullptr, k, b, s.c1, true));
  if (allreduce) SQB_TRY(allreduce(s.c1));
  SQB_CUDA(launch_cholesky(s.c1, n, s.r1, ctx->d_status, ctx->stream));
  SQB_TRY(gram_view(ctx, v, m, n, OP_SOLVE, s.r1, k, b, s.c2, false));
  if (allreduce) SQB_TRY(allreduce(s.c2));
  SQB_CUDA(launch_cholesky(s.c2, n, s.r2, ctx->d_status, ctx->stream));
  SQB_CUDA(launch_tri_multiply(s.r2, s.r1, n, d_r, ctx->stream));
  ctx->launches += 3;
  return SQB_OK;
}

// ---- wide column counts (64 < n <= 256): plain Gram, fused solve / multiply + Gram ----
int gram_wide_view(sqb_context* ctx, const MatView& v, long long m, int n, int op, const double* factor,
                   double* d_c, bool check) {
  const size_t partial = gram_wide_partial_doubles(n, ctx->sm_count);
  if (op == OP_PLAIN) {
    if (n > kWideGramMaxN) return SQB_E_ARGUMENT;
    SQB_TRY(grow(&ctx->work, &ctx->work_doubles, partial + gram_wide_fused_scratch_doubles()));
    SQB_CUDA(launch_gram_wide(v, m, n, ctx->sm_count, ctx->work, d_c, check ? 1 : 0, ctx->d_status,
                              ctx->stream));
    ctx->launches += 2;
    return SQB_OK;
  }
  if (n > kWideGramMaxN) return SQB_E_ARGUMENT;
  if (n > kWideFusedMaxN) {
    // 129..256 columns: Q = X F per row slab (128 x 128 factor blocks), wide SYRK on the slab
    const size_t sc = gram_wide2_scratch_doubles(n), nn = static_cast<size_t>(n) * n;
    SQB_TRY(grow(&ctx->work, &ctx->work_doubles, partial + sc + nn));
    const long long slab_rows = std::min<long long>((std::max<long long>(m, 8) + 7) / 8 * 8, 1ll << 20);
    SQB_TRY(grow(&ctx->qslab, &ctx->qslab_doubles, static_cast<size_t>(slab_rows) * n));
    SQB_CUDA(launch_gram_wide2_fused(v, m, n, op, factor, ctx->sm_count, ctx->work + partial, ctx->qslab, slab_rows,
                                     ctx->work, ctx->work + partial + sc, d_c, ctx->d_status, ctx->stream,
                                     &ctx->launches));
    return SQB_OK;
  }
  SQB_TRY(grow(&ctx->work, &ctx->work_doubles, partial + gram_wide_fused_scratch_doubles()));
  SQB_CUDA(launch_gram_wide_fused(v, m, n, op, factor, ctx->sm_count, ctx->work + partial, ctx->work, d_c,
                                  ctx->d_status, ctx->stream));
  ctx->launches += 3;
  return SQB_OK;
}

// CholQR2 beyond 64 columns (the reference's cholqr2 has no column limit, gram_qr.cpp:123-131): the
// wide SYRK, Cholesky (one CTA; in global memory beyond 128 columns), the fused solve + Gram sweep, Cholesky,
// R = R2 R1; up to 256 columns.
int cholqr2_wide(sqb_context* ctx, const MatView& v, long long m, int n, double* d_r,
                 const std::function<int(double*)>& allreduce) {
  Small s;
  SQB_TRY(small_slots(ctx, n, &s));
  SQB_TRY(gram_wide_view(ctx, v, m, n, OP_PLAIN, nullptr, s.c1, true));
  if (allreduce) SQB_TRY(allreduce(s.c1));
  SQB_CUDA(launch_cholesky(s.c1, n, s.r1, ctx->d_status, ctx->stream));
  SQB_TRY(gram_wide_view(ctx, v, m, n, OP_SOLVE, s.r1, s.c2, false));
  if (allreduce) SQB_TRY(allreduce(s.c2));
  SQB_CUDA(launch_cholesky(s.c2, n, s.r2, ctx->d_status, ctx->stream));
  SQB_CUDA(launch_tri_multiply(s.r2, s.r1, n, d_r, ctx->stream));
  ctx->launches += 3;
  return SQB_OK;
}

// SVQB2 beyond 64 columns (up to the reference's own eigh_small limit of 128, gram_qr.cpp:62).
int svqb2_wide(sqb_context* ctx, const MatView& v, long long m, int n, double* d_transform, double* d_z,
               double* d_sigma, long long* d_rank, const std::function<int(double*)>& allreduce) {
  Small s;
  SQB_TRY(small_slots(ctx, n, &s));
  SQB_TRY(gram_wide_view(ctx, v, m, n, OP_PLAIN, nullptr, s.c1, true));
  if (allreduce) SQB_TRY(allreduce(s.c1));
  SQB_CUDA(launch_svqb_pass(s.c1, n, s.b1, s.z1, d_sigma, s.rank1, 1, s.scratch, ctx->d_status, ctx->stream));
  SQB_TRY(gram_wide_view(ctx, v, m, n, OP_MULTIPLY, s.b1, s.c2, false));
  if (allreduce) SQB_TRY(allreduce(s.c2));
  SQB_CUDA(launch_svqb_pass(s.c2, n, s.b2, s.z2, s.s2, d_rank, 0, s.scratch, ctx->d_status, ctx->stream));
  SQB_CUDA(launch_small_multiply(s.b1, s.b2, n, d_transform, ctx->stream));
  SQB_CUDA(launch_small_multiply(s.z2, s.z1, n, d_z, ctx->stream));
  ctx->launches += 4;
  return SQB_OK;
}

// SVQB2 (gram_qr.cpp:178-191): sigma from pass 1, rank from pass 2, B = B1 B2, Z = Z2 Z1.
int svqb2_view(sqb_context* ctx, const MatView& v, long long m, int n, long long k, long long b,
               double* d_transform, double* d_z, double* d_sigma, long long* d_rank,
               const std::function<int(double*)>& allreduce) {
  Small s;
  SQB_TRY(small_slots(ctx, n, &s));
  SQB_TRY(gram_view(ctx, v, m, n, OP_PLAIN, nullptr, k, b, s.c1, true));
  if (allreduce) SQB_TRY(allreduce(s.c1));
  SQB_CUDA(launch_svqb_pass(s.c1, n, s.b1, s.z1, d_sigma, s.rank1, 1, s.scratch, ctx->d_status,
                            ctx->stream));
  SQB_TRY(gram_view(ctx, v, m, n, OP_MULTIPLY, s.b1, k, b, s.c2, false));
  if (allreduce) SQB_TRY(allreduce(s.c2));
  SQB_CUDA(launch_svqb_pass(s.c2, n, s.b2, s.z2, s.s2, d_rank, 0, s.scratch, ctx->d_status,
                            ctx->stream));
  SQB_CUDA(launch_small_multiply(s.b1, s.b2, n, d_transform, ctx->stream));
  SQB_CUDA(launch_small_multiply(s.z2, s.z1, n, d_z, ctx->stream));
  ctx->launches += 4;
  return SQB_OK;
}

int translate_status(sqb_context* ctx) {
  const StatusWord w = *ctx->h_status;
  if (w.nonfinite) return SQB_E_ARGUMENT;  // reference validates finiteness before factorising
  if (w.code != 0) {
    ctx->last_index = w.index;
    return w.code;
  }
  return SQB_OK;
}

// ---- host-pointer plumbing -------------------------------------------------------------------
// Two ways to bring a host matrix to the GPU.
//  * upload_resident: the whole matrix lands in ctx->xbuf (leading dimension rounded up to an even
//    row count so that every column stays 16-byte aligned whatever the parity of m) - for the methods
//    that read X twice (CholQR2, SVQB2) and for explicit plans whose blocks exceed a slab.
//  * stream_slabs: single-pass methods see X as a sequence of row slabs moving through a ring of
//    ctx->kRing device buffers: slab i+1 .. i+2 are in flight over PCIe while slab i is factored, and
//    device memory stays O(slab) - the reference's streaming state is O((b+n)*n), tsqr.cpp:143-147.
long long even_up(long long v) { return (v + 1) & ~1ll; }

int upload_resident(sqb_context* ctx, const double* x, long long m, int n, long long ld, int extra_cols,
                    long long* ldx) {
  *ldx = even_up(std::max<long long>(m, 1));
  SQB_TRY(grow(&ctx->xbuf, &ctx->xbuf_doubles, static_cast<size_t>(*ldx) * (n + extra_cols)));
  const long long slab_rows = std::max<long long>(2, ctx->host_slab_bytes / (sizeof(double) * n) / 2 * 2);
  for (long long r0 = 0; r0 < m; r0 += slab_rows) {
    const long long rows = std::min(slab_rows, m - r0);
    SQB_CUDA(cudaMemcpy2DAsync(ctx->xbuf + r0, sizeof(double) * *ldx, x + r0, sizeof(double) * ld,
                               sizeof(double) * rows, n, cudaMemcpyHostToDevice, ctx->copy_stream));
  }
  SQB_CUDA(cudaEventRecord(ctx->slab_ready, ctx->copy_stream));
  SQB_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->slab_ready, 0));
  return SQB_OK;
}

using SlabFn = std::function<int(long long slab, long long r0, long long rows, const double* d_slab, long long ld_slab)>;

// rows per slab: a multiple of `row_align` (>= 2, even) that fits host_slab_bytes for n_tot columns
long long slab_rows_for(const sqb_context* ctx, int n_tot, long long row_align) {
  const long long want = ctx->host_slab_bytes / (static_cast<long long>(sizeof(double)) * n_tot);
  return std::max(row_align, want / row_align * row_align);
}

// `extra` (optional) is one more host column of m entries that travels as column n of every slab
// (least squares: the [A rhs] pencil, lstsq.cpp:24-26).
int stream_slabs(sqb_context* ctx, const double* x, const double* extra, long long m, int n, long long ld,
                 long long slab_rows, const SlabFn& on_slab) {
  const int n_tot = n + (extra ? 1 : 0);
  const long long lds = even_up(slab_rows);
  const size_t slab_doubles = static_cast<size_t>(lds) * n_tot;
  SQB_TRY(grow(&ctx->ring, &ctx->ring_doubles, slab_doubles * sqb_context::kRing));
  // the ring may still be read by kernels of an earlier call on this stream
  SQB_CUDA(cudaEventRecord(ctx->slab_ready, ctx->stream));
  SQB_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->slab_ready, 0));
  long long slab = 0;
  for (long long r0 = 0; r0 < m; r0 += slab_rows, ++slab) {
    const long long rows = std::min(slab_rows, m - r0);
    const int slot = static_cast<int>(slab % sqb_context::kRing);
    double* dst = ctx->ring + slab_doubles * slot;
    if (slab >= sqb_context::kRing) SQB_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->ring_free[slot], 0));
    SQB_CUDA(cudaMemcpy2DAsync(dst, sizeof(double) * lds, x + r0, sizeof(double) * ld, sizeof(double) * rows, n,
                               cudaMemcpyHostToDevice, ctx->copy_stream));
    if (extra)
      SQB_CUDA(cudaMemcpyAsync(dst + static_cast<size_t>(lds) * n, extra + r0, sizeof(double) * rows,
                               cudaMemcpyHostToDevice, ctx->copy_stream));
    SQB_CUDA(cudaEventRecord(ctx->slab_ready, ctx->copy_stream));
    SQB_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->slab_ready, 0));
    SQB_TRY(on_slab(slab, r0, rows, dst, lds));
    SQB_CUDA(cudaEventRecord(ctx->ring_free[slot], ctx->stream));
  }
  return SQB_OK;
}

// Every *_host call starts from a clean status word: an error left behind by an un-synchronised
// *_dev call must not be attributed to this call.
int enter_host(sqb_context* ctx) {
  SQB_TRY(enter(ctx));
  SQB_CUDA(cudaMemsetAsync(ctx->d_status, 0, sizeof(StatusWord), ctx->stream));
  return SQB_OK;
}

int upload_small(sqb_context* ctx, const double* h, size_t count, double* d) {
  SQB_CUDA(cudaMemcpyAsync(d, h, count * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  return SQB_OK;
}

int download(sqb_context* ctx, void* h, const void* d, size_t bytes) {
  SQB_CUDA(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  return SQB_OK;
}

// ---- NCCL through dlopen -----------------------------------------------------------------------
struct NcclId {
  char bytes[128];
};
struct NcclApi {
  void* lib = nullptr;
  int (*GetUniqueId)(NcclId*) = nullptr;
  int (*CommInitRank)(void**, int, NcclId, int) = nullptr;
  int (*CommDestroy)(void*) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  bool ok = false;
};
constexpr int kNcclFloat64 = 8;  // ncclDouble
constexpr int kNcclSum = 0;      // ncclSum

NcclApi& nccl() {
  static NcclApi api;
  if (api.lib) return api;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* nm : names) {
    api.lib = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (api.lib) break;
  }
  if (!api.lib) return api;
  api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(api.lib, "ncclGetUniqueId"));
  api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(api.lib, "ncclCommInitRank"));
  api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(api.lib, "ncclCommDestroy"));
  api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(api.lib, "ncclAllGather"));
  api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(api.lib, "ncclAllReduce"));
  api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather && api.AllReduce;
  return api;
}

// ---- the n x n exchange of the row-sharded drivers ---------------------------------------------------
bool is_sharded(const sqb_context* ctx) { return ctx->world > 1 || ctx->nccl_comm || ctx->gather_fn; }

// `count` doubles per rank: send -> recv (world blocks in rank order).  One implementation of the
// protocol, two transports: a caller-supplied all-gather or NCCL.
int allgather_blocks(sqb_context* ctx, const double* send, double* recv, size_t count) {
  if (ctx->gather_fn)
    return ctx->gather_fn(ctx->gather_user, send, recv, static_cast<int64_t>(count)) == 0 ? SQB_OK : SQB_E_NCCL;
  NcclApi& api = nccl();
  if (!api.ok || !ctx->nccl_comm) return SQB_E_NCCL;
  return api.AllGather(send, recv, count, kNcclFloat64, ctx->nccl_comm, ctx->stream) == 0 ? SQB_OK : SQB_E_NCCL;
}

// gathered: world blocks of n x n (column-major, leading dimension n) -> (world*n) x n stack
__global__ void pack_stack_kernel(const double* __restrict__ gathered, int world, int n,
                                  double* __restrict__ stack) {
  const long long total = static_cast<long long>(world) * n * n;
  for (long long t = threadIdx.x + static_cast<long long>(blockIdx.x) * blockDim.x; t < total;
       t += static_cast<long long>(blockDim.x) * gridDim.x) {
    const int g = static_cast<int>(t / (n * n));
    const int rem = static_cast<int>(t % (n * n));
    const int i = rem % n, j = rem / n;
    stack[(static_cast<long long>(g) * n + i) + static_cast<long long>(j) * world * n] = gathered[t];
  }
}

// out = sum over ranks, ascending rank order (the reference's ascending block order, gram.cpp:81-92):
// every rank computes the same sum bit for bit, whatever the transport's internal order is
__global__ void sum_ranks_kernel(const double* __restrict__ gathered, int world, long long count,
                                 double* __restrict__ out) {
  for (long long t = threadIdx.x + static_cast<long long>(blockIdx.x) * blockDim.x; t < count;
       t += static_cast<long long>(blockDim.x) * gridDim.x) {
    double acc = gathered[t];
    for (int g = 1; g < world; ++g) acc += gathered[t + g * count];
    out[t] = acc;
  }
}

// Stage 2 with k = world (tsqr.cpp:193-195): stack the gathered triangles, fold, sign-normalise.
int tsqr_combine(sqb_context* ctx, const double* gathered, int world, int n, double* stack, double* d_r) {
  pack_stack_kernel<<<8, 256, 0, ctx->stream>>>(gathered, world, n, stack);
  SQB_CUDA(cudaGetLastError());
  ctx->launches++;
  const long long rows = static_cast<long long>(world) * n;
  return launch_tsqr(ctx, plain_view(stack, rows, n), rows, n, make_plan(rows, 1, rows), d_r, n, true, false);
}

int gram_combine(sqb_context* ctx, const double* gathered, int world, int n, double* d_c) {
  const long long count = static_cast<long long>(n) * n;
  sum_ranks_kernel<<<static_cast<unsigned>(std::min<long long>((count + 255) / 256, 64)), 256, 0, ctx->stream>>>(
      gathered, world, count, d_c);
  SQB_CUDA(cudaGetLastError());
  ctx->launches++;
  return SQB_OK;
}

// scratch of the exchange: [gathered: world*n*n][stack: world*n*n]
int exchange_scratch(sqb_context* ctx, int n, double** gathered, double** stack) {
  const size_t nn = static_cast<size_t>(n) * n;
  SQB_TRY(grow(&ctx->gen, &ctx->gen_doubles, 2 * nn * ctx->world));
  *gathered = ctx->gen;
  *stack = ctx->gen + nn * ctx->world;
  return SQB_OK;
}

// Partial Gram of this rank's slab (in place in d) -> the sum over all ranks, identical everywhere.
int allreduce_square(sqb_context* ctx, double* d, int n) {
  if (!is_sharded(ctx)) return SQB_OK;
  double *gathered, *stack;
  SQB_TRY(exchange_scratch(ctx, n, &gathered, &stack));
  SQB_TRY(allgather_blocks(ctx, d, gathered, static_cast<size_t>(n) * n));
  return gram_combine(ctx, gathered, ctx->world, n, d);
}

// This rank's un-normalised triangle; a rank may own fewer than n rows (or none): its triangle is
// then that of a zero-padded slab.
int tsqr_local_view(sqb_context* ctx, const MatView& v, long long m_local, int n, double* d_r_local) {
  if (m_local > 0) return tsqr_view(ctx, v, m_local, n, 0, 0, d_r_local, false);
  SQB_CUDA(cudaMemsetAsync(d_r_local, 0, sizeof(double) * n * n, ctx->stream));
  return SQB_OK;
}

// Local triangle -> all-gather -> redundant final combine on every rank (stage 2 with k = world).
int tsqr_sharded_view(sqb_context* ctx, const MatView& v, long long m_local, int n, double* d_r) {
  if (!is_sharded(ctx)) return tsqr_view(ctx, v, m_local, n, 0, 0, d_r, true);
  Small s;
  SQB_TRY(small_slots(ctx, n, &s));
  SQB_TRY(tsqr_local_view(ctx, v, m_local, n, s.c1));
  double *gathered, *stack;
  SQB_TRY(exchange_scratch(ctx, n, &gathered, &stack));
  SQB_TRY(allgather_blocks(ctx, s.c1, gathered, static_cast<size_t>(n) * n));
  return tsqr_combine(ctx, gathered, ctx->world, n, stack, d_r);
}

}  // namespace

// =================================================================================================
extern "C" {

int sqb_create(sqb_context** out, int device) {
  if (!out) return SQB_E_ARGUMENT;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || device < 0 || device >= count) return SQB_E_CUDA;
  SQB_CUDA(cudaSetDevice(device));
  sqb_context* ctx = new (std::nothrow) sqb_context();
  if (!ctx) return SQB_E_CUDA;
  ctx->device = device;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major < 10) {
    delete ctx;
    return SQB_E_CUDA;  // sm_100a kernels only
  }
  ctx->sm_count = prop.multiProcessorCount;
  bool ok = cudaStreamCreateWithFlags(&ctx->own_stream_handle, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&ctx->slab_ready, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&ctx->ring_free[0], cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&ctx->ring_free[1], cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&ctx->ring_free[2], cudaEventDisableTiming) == cudaSuccess &&
            cudaMalloc(reinterpret_cast<void**>(&ctx->d_status), sizeof(StatusWord)) == cudaSuccess &&
            cudaMallocHost(reinterpret_cast<void**>(&ctx->h_status), sizeof(StatusWord)) == cudaSuccess;
  if (ok) ok = cudaMemset(ctx->d_status, 0, sizeof(StatusWord)) == cudaSuccess;
  if (!ok) {
    sqb_destroy(ctx);
    return SQB_E_CUDA;
  }
  ctx->stream = ctx->own_stream_handle;
  std::memset(ctx->h_status, 0, sizeof(StatusWord));
  *out = ctx;
  return SQB_OK;
}

int sqb_destroy(sqb_context* ctx) {
  if (!ctx) return SQB_OK;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->own_comm && ctx->nccl_comm && nccl().ok) nccl().CommDestroy(ctx->nccl_comm);
  cudaFree(ctx->work);
  cudaFree(ctx->small);
  cudaFree(ctx->xbuf);
  cudaFree(ctx->ring);
  cudaFree(ctx->qslab);
  for (cudaEvent_t e : ctx->ring_free)
    if (e) cudaEventDestroy(e);
  cudaFree(ctx->gen);
  cudaFree(ctx->d_status);
  if (ctx->h_status) cudaFreeHost(ctx->h_status);
  if (ctx->slab_ready) cudaEventDestroy(ctx->slab_ready);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->own_stream_handle) cudaStreamDestroy(ctx->own_stream_handle);
  delete ctx;
  return SQB_OK;
}

int sqb_set_stream(sqb_context* ctx, void* cuda_stream) {
  SQB_TRY(enter(ctx));
  ctx->stream = static_cast<cudaStream_t>(cuda_stream);  // NULL is the CUDA default stream
  ctx->own_stream = false;
  return SQB_OK;
}

int sqb_use_own_stream(sqb_context* ctx) {
  SQB_TRY(enter(ctx));
  ctx->stream = ctx->own_stream_handle;
  ctx->own_stream = true;
  return SQB_OK;
}

void* sqb_get_stream(sqb_context* ctx) { return ctx ? ctx->stream : nullptr; }

int sqb_set_tsqr_kernel(sqb_context* ctx, int kind) {
  if (!ctx || kind < kTsqrAuto || kind > kTsqrMma) return SQB_E_ARGUMENT;
  ctx->tsqr_kind = kind;
  return SQB_OK;
}

int sqb_set_host_slab_bytes(sqb_context* ctx, int64_t bytes) {
  if (!ctx || bytes < (1ll << 20)) return SQB_E_ARGUMENT;
  ctx->host_slab_bytes = bytes;
  return SQB_OK;
}

int sqb_copy_h2d(sqb_context* ctx, void* d_dst, const void* h_src, int64_t bytes) {
  SQB_TRY(enter(ctx));
  if (bytes < 0 || (bytes > 0 && (!d_dst || !h_src))) return SQB_E_ARGUMENT;
  SQB_CUDA(cudaMemcpyAsync(d_dst, h_src, static_cast<size_t>(bytes), cudaMemcpyHostToDevice, ctx->stream));
  SQB_CUDA(cudaStreamSynchronize(ctx->stream));
  return SQB_OK;
}

int sqb_device_alloc(sqb_context* ctx, int64_t bytes, void** d_ptr) {
  SQB_TRY(enter(ctx));
  if (!d_ptr || bytes < 0) return SQB_E_ARGUMENT;
  *d_ptr = nullptr;
  if (bytes == 0) return SQB_OK;
  SQB_CUDA(cudaMalloc(d_ptr, static_cast<size_t>(bytes)));
  return SQB_OK;
}

int sqb_device_free(sqb_context* ctx, void* d_ptr) {
  SQB_TRY(enter(ctx));
  if (d_ptr) {
    SQB_CUDA(cudaStreamSynchronize(ctx->stream));  // nothing enqueued on this context may still use it
    SQB_CUDA(cudaFree(d_ptr));
  }
  return SQB_OK;
}

int sqb_copy_d2h(sqb_context* ctx, void* h_dst, const void* d_src, int64_t bytes) {
  SQB_TRY(enter(ctx));
  if (bytes < 0 || (bytes > 0 && (!h_dst || !d_src))) return SQB_E_ARGUMENT;
  SQB_CUDA(cudaMemcpyAsync(h_dst, d_src, static_cast<size_t>(bytes), cudaMemcpyDeviceToHost, ctx->stream));
  SQB_CUDA(cudaStreamSynchronize(ctx->stream));
  return SQB_OK;
}

int sqb_sync(sqb_context* ctx) {
  SQB_TRY(enter(ctx));
  SQB_CUDA(cudaMemcpyAsync(ctx->h_status, ctx->d_status, sizeof(StatusWord), cudaMemcpyDeviceToHost,
                           ctx->stream));
  SQB_CUDA(cudaMemsetAsync(ctx->d_status, 0, sizeof(StatusWord), ctx->stream));
  SQB_CUDA(cudaStreamSynchronize(ctx->stream));
  return translate_status(ctx);
}

long long sqb_last_error_index(const sqb_context* ctx) { return ctx ? ctx->last_index : -1; }

const char* sqb_status_string(int status) {
  switch (status) {
    case SQB_OK: return "ok";
    case SQB_E_DIMENSION: return "DimensionError";
    case SQB_E_ARGUMENT: return "ArgumentError";
    case SQB_E_BREAKDOWN: return "BreakdownError";
    case SQB_E_SINGULAR: return "SingularFactorError";
    case SQB_E_ZERO_MATRIX: return "ZeroMatrixError";
    case SQB_E_RANK_DEFICIENT: return "RankDeficiencyError";
    case SQB_E_NO_CONVERGENCE: return "Error (eigensolver did not converge)";
    case SQB_E_CUDA: return "CUDA failure or no sm_100 device";
    case SQB_E_NCCL: return "NCCL failure";
    default: return "unknown status";
  }
}

int sqb_device_sm_count(const sqb_context* ctx) { return ctx ? ctx->sm_count : 0; }
long long sqb_launch_count(const sqb_context* ctx) { return ctx ? ctx->launches : 0; }

int sqb_default_tsqr_plan(const sqb_context* ctx, int64_t m, int64_t n, int64_t* num_blocks,
                          int64_t* panel_rows) {
  if (!ctx || n < 1 || n > 64) return SQB_E_ARGUMENT;  // plan.cpp:20-21
  const Plan p = tsqr_plan(ctx, m, static_cast<int>(n), 0, 0);
  if (num_blocks) *num_blocks = p.k;
  if (panel_rows) *panel_rows = p.b;
  return SQB_OK;
}

int sqb_default_gram_plan(const sqb_context* ctx, int64_t m, int64_t n, int64_t* num_blocks,
                          int64_t* panel_rows) {
  if (!ctx || n < 1 || n > kWideGramMaxN) return SQB_E_ARGUMENT;  // plan.cpp:9-17 has no column limit
  if (n > 64) {  // the wide kernel partitions rows itself: report its shape (one row block per SM, 56-row panels)
    if (num_blocks) *num_blocks = ctx->sm_count;
    if (panel_rows) *panel_rows = 56;
    return SQB_OK;
  }
  const Plan p = gram_plan(ctx, m, static_cast<int>(n), OP_PLAIN, 0, 0);
  if (num_blocks) *num_blocks = p.k;
  if (panel_rows) *panel_rows = p.b;
  return SQB_OK;
}

// ---- device-pointer entry points ---------------------------------------------------------------
int sqb_tsqr_qless_dev(sqb_context* ctx, const double* d_x, int64_t m, int64_t n, int64_t ld,
                       int64_t num_blocks, int64_t panel_rows, double* d_r) {
  SQB_TRY(enter(ctx));
  SQB_TRY(check_shape(m, n, ld, 64));
  return tsqr_view(ctx, plain_view(d_x, ld, static_cast<int>(n)), m, static_cast<int>(n), num_blocks,
                   panel_rows, d_r, true);
}

int sqb_tsqr_stage1_dev(sqb_context* ctx, const double* d_x, int64_t m, int64_t n, int64_t ld,
                        int64_t num_blocks, int64_t panel_rows, double* d_y) {
  SQB_TRY(enter(ctx));
  if (n < 1 || n > 64 || ld < m || m < 0) return SQB_E_ARGUMENT;
  const Plan p = tsqr_plan(ctx, m, static_cast<int>(n), num_blocks, panel_rows);
  return launch_tsqr(ctx, plain_view(d_x, ld, static_cast<int>(n)), m, static_cast<int>(n), p, d_y,
                     p.k * n, false, true);
}

int sqb_block_qless_qr_dev(sqb_context* ctx, const double* d_x, int64_t m, int64_t n, int64_t ld,
                           int64_t panel_rows, double* d_r) {
  SQB_TRY(enter(ctx));
  if (n < 1 || n > 64 || ld < m || m < 0) return SQB_E_ARGUMENT;
  const int64_t b = panel_rows > 0 ? panel_rows : tsqr_panel_rows(static_cast<int>(n), ctx->tsqr_kind);
  Plan p{1, b, ceil_div(std::max<int64_t>(m, 1), b) * b};
  return launch_tsqr(ctx, plain_view(d_x, ld, static_cast<int>(n)), m, static_cast<int>(n), p, d_r, n,
                     false, true);
}

static int gram_entry(sqb_context* ctx, const double* d_x, int64_t m, int64_t n, int64_t ld, int op,
                      const double* factor, int64_t k, int64_t b, double* d_c) {
  SQB_TRY(enter(ctx));
  if (n < 1 || m < 0) return SQB_E_DIMENSION;
  if (ld < m) return SQB_E_ARGUMENT;
  if (op == OP_MULTIPLY) {  // tsmmttsmm checks B for finiteness at any n (gram.cpp:143-145)
    if (n > kWideGramMaxN) return SQB_E_ARGUMENT;
    SQB_CUDA(launch_check_finite(factor, n * n, ctx->d_status, ctx->stream));
    ctx->launches++;
  }
  if (n > 64) {
    // the reference's Gram kernels have no column limit (gram.cpp:113-151); here the plain Gram goes
    // up to 256 columns, like the fused solve / multiply + Gram (one launch up to 128, per row slab beyond)
    return gram_wide_view(ctx, plain_view(d_x, ld, static_cast<int>(n)), m, static_cast<int>(n), op, factor, d_c,
                          op == OP_PLAIN);
  }
  return gram_view(ctx, plain_view(d_x, ld, static_cast<int>(n)), m, static_cast<int>(n), op, factor, k,
                   b, d_c, op == OP_PLAIN);
}

int sqb_tsmttsm_dev(sqb_context* ctx, const double* d_x, int64_t m, int64_t n, int64_t ld,
                    int64_t num_blocks, int64_t panel_rows, double* d_c) {
  return gram_entry(ctx, d_x, m, n, ld, OP_PLAIN, nullptr, num_blocks, panel_rows, d_c);
}

int sqb_tsmRttsmR_dev(sqb_context* ctx, const double* d_x, int64_t m, int64_t n, int64_t ld,
                      const double* d_r, int64_t num_blocks, int64_t panel_rows, double* d_c) {
  return gram_entry(ctx, d_x, m, n, ld, OP_SOLVE, d_r, num_blocks, panel_rows, d_c);
}

int sqb_tsmmttsmm_dev(sqb_context* ctx, const double* d_x, int64_t m, int64_t n, int64_t ld,
                      const double* d_b, int64_t num_blocks, int64_t panel_rows, double* d_c) {
  return gram_entry(ctx, d_x, m, n, ld, OP_MULTIPLY, d_b, num_blocks, panel_rows, d_c);
}

int sqb_cholesky_dev(sqb_context* ctx, const double* d_c, int64_t n, double* d_r) {
  SQB_TRY(enter(ctx));
  if (n < 1) return SQB_E_DIMENSION;
  if (n > kWideGramMaxN) return SQB_E_ARGUMENT;  // the reference has no limit (gram_qr.cpp:36-58); 256 = config 5
  SQB_CUDA(launch_cholesky(d_c, static_cast<int>(n), d_r, ctx->d_status, ctx->stream));
  ctx->launches++;
  return SQB_OK;
}

int sqb_eigh_small_dev(sqb_context* ctx, const double* d_c, int64_t n, double* d_values,
                       double* d_vectors) {
  SQB_TRY(enter(ctx));
  if (n < 1) return SQB_E_DIMENSION;
  if (n > kSmallMaxN) return SQB_E_ARGUMENT;  // gram_qr.cpp:62
  Small s;
  SQB_TRY(small_slots(ctx, static_cast<int>(n), &s));
  SQB_CUDA(launch_eigh(d_c, static_cast<int>(n), d_values, d_vectors, s.scratch, ctx->d_status,
                       ctx->stream));
  ctx->launches++;
  return SQB_OK;
}

int sqb_cholqr2_dev(sqb_context* ctx, const double* d_x, int64_t m, int64_t n, int64_t ld,
                    int64_t num_blocks, int64_t panel_rows, double* d_r) {
  SQB_TRY(enter(ctx));
  SQB_TRY(check_shape(m, n, ld, kWideGramMaxN));
  if (n > 64) return cholqr2_wide(ctx, plain_view(d_x, ld, static_cast<int>(n)), m, static_cast<int>(n), d_r, nullptr);
  return cholqr2_view(ctx, plain_view(d_x, ld, static_cast<int>(n)), m, static_cast<int>(n), num_blocks,
                      panel_rows, d_r, nullptr);
}

int sqb_svqb2_dev(sqb_context* ctx, const double* d_x, int64_t m, int64_t n, int64_t ld,
                  int64_t num_blocks, int64_t panel_rows, double* d_transform, double* d_z,
                  double* d_sigma, int64_t* d_rank) {
  SQB_TRY(enter(ctx));
  SQB_TRY(check_shape(m, n, ld, kWideFusedMaxN));
  if (n > 64)
    return svqb2_wide(ctx, plain_view(d_x, ld, static_cast<int>(n)), m, static_cast<int>(n), d_transform, d_z,
                      d_sigma, reinterpret_cast<long long*>(d_rank), nullptr);
  return svqb2_view(ctx, plain_view(d_x, ld, static_cast<int>(n)), m, static_cast<int>(n), num_blocks,
                    panel_rows, d_transform, d_z, d_sigma, reinterpret_cast<long long*>(d_rank),
                    nullptr);
}

int sqb_svqb_pass_dev(sqb_context* ctx, const double* d_c, int64_t n, double* d_b, double* d_z,
                      double* d_sigma, int64_t* d_rank) {
  SQB_TRY(enter(ctx));
  if (n < 1) return SQB_E_DIMENSION;
  if (n > kSmallMaxN) return SQB_E_ARGUMENT;
  Small s;
  SQB_TRY(small_slots(ctx, static_cast<int>(n), &s));
  SQB_CUDA(launch_svqb_pass(d_c, static_cast<int>(n), d_b, d_z, d_sigma,
                            reinterpret_cast<long long*>(d_rank), 1, s.scratch, ctx->d_status,
                            ctx->stream));
  ctx->launches++;
  return SQB_OK;
}

int sqb_reconstruct_q_dev(sqb_context* ctx, const double* d_x, int64_t m, int64_t n, int64_t ld,
                          const double* d_r, double* d_q, int64_t ldq) {
  SQB_TRY(enter(ctx));
  if (n < 1 || m < 0) return SQB_E_DIMENSION;
  if (n > kWideGramMaxN || ld < m || ldq < m) return SQB_E_ARGUMENT;
  if (n > kWideFusedMaxN) {
    SQB_TRY(grow(&ctx->work, &ctx->work_doubles, gram_wide2_scratch_doubles(static_cast<int>(n))));
    SQB_CUDA(launch_apply_rinv_wide2(d_x, m, static_cast<int>(n), ld, d_r, ctx->sm_count, ctx->work, d_q, ldq,
                                     ctx->d_status, ctx->stream));
    ctx->launches += 9;
    return SQB_OK;
  }
  if (n > 64) {
    SQB_TRY(grow(&ctx->work, &ctx->work_doubles, gram_wide_partial_doubles(static_cast<int>(n), ctx->sm_count) +
                                                     gram_wide_fused_scratch_doubles()));
    SQB_CUDA(launch_apply_rinv_wide(d_x, m, static_cast<int>(n), ld, d_r, ctx->sm_count, ctx->work, d_q, ldq,
                                    ctx->d_status, ctx->stream));
    ctx->launches += 2;
    return SQB_OK;
  }
  SQB_CUDA(launch_apply_rinv(d_x, m, static_cast<int>(n), ld, d_r, d_q, ldq, ctx->d_status,
                             ctx->stream));
  ctx->launches += 2;
  return SQB_OK;
}

static int lstsq_view(sqb_context* ctx, const MatView& v, int64_t m, int ne, int method,
                      double* d_xsol, double* d_residual, bool sharded) {
  // [A rhs] may have up to 64 columns on the TSQR route (tsqr.cpp:188), up to 128 on the Gram routes
  if (ne > (method == SQB_METHOD_TSQR ? 64 : kWideFusedMaxN)) return SQB_E_ARGUMENT;
  Small s;
  SQB_TRY(small_slots(ctx, ne, &s));
  double* r = s.rr;
  std::function<int(double*)> ar;
  if (sharded) ar = [ctx, ne](double* d) { return allreduce_square(ctx, d, ne); };
  if (method == SQB_METHOD_TSQR) {
    if (sharded) SQB_TRY(tsqr_sharded_view(ctx, v, m, ne, r));
    else SQB_TRY(tsqr_view(ctx, v, m, ne, 0, 0, r, true));
  } else if (method == SQB_METHOD_CHOLQR2) {
    if (ne > 64) SQB_TRY(cholqr2_wide(ctx, v, m, ne, r, ar));  // the Gram route has no 64-column limit
    else SQB_TRY(cholqr2_view(ctx, v, m, ne, 0, 0, r, ar));
  } else if (method == SQB_METHOD_SVQB2) {
    // Z -> rr[0, ne^2), transform -> rr[ne^2, 2 ne^2) (svqb2_view owns every other slot)
    double* tr = s.rr + static_cast<size_t>(ne) * ne;
    if (ne > 64) {
      SQB_TRY(svqb2_wide(ctx, v, m, ne, tr, r, s.s2 + ne, s.rank1 + 1, ar));
      SQB_CUDA(cudaMemcpyAsync(tr, r, sizeof(double) * ne * ne, cudaMemcpyDeviceToDevice, ctx->stream));
      SQB_CUDA(launch_hhqr_small(tr, ne, r, ctx->stream));  // hhqr_small, lstsq.cpp:37-39
      SQB_CUDA(launch_backsolve(r, ne, d_xsol, d_residual, ctx->d_status, ctx->stream));
      ctx->launches += 2;
      return SQB_OK;
    }
    SQB_TRY(svqb2_view(ctx, v, m, ne, 0, 0, tr, r, s.s2 + ne, s.rank1 + 1, ar));
    // triangularise Z with the Householder kernel (reference hhqr_small, lstsq.cpp:37-39);
    // in-place is safe: the kernel stages Z on chip before writing its triangle.
    SQB_CUDA(cudaMemcpyAsync(tr, r, sizeof(double) * ne * ne, cudaMemcpyDeviceToDevice, ctx->stream));
    SQB_TRY(launch_tsqr(ctx, plain_view(tr, ne, ne), ne, ne, make_plan(ne, 1, ne), r, ne, true, false));
  } else {
    return SQB_E_ARGUMENT;
  }
  SQB_CUDA(launch_backsolve(r, ne, d_xsol, d_residual, ctx->d_status, ctx->stream));
  ctx->launches++;
  return SQB_OK;
}

int sqb_solve_lstsq_dev(sqb_context* ctx, const double* d_a, int64_t m, int64_t n, int64_t lda,
                        const double* d_rhs, int method, double* d_xsol, double* d_residual) {
  SQB_TRY(enter(ctx));
  if (n < 1 || m < n + 1) return SQB_E_DIMENSION;  // lstsq.cpp:16-17
  if (n + 1 > kWideFusedMaxN || lda < m) return SQB_E_ARGUMENT;
  const MatView v{d_a, lda, d_rhs, static_cast<int>(n)};
  return lstsq_view(ctx, v, m, static_cast<int>(n) + 1, method, d_xsol, d_residual, false);
}

// ---- host-pointer entry points -------------------------------------------------------------------
// Slab layout for a single-pass call under a plan.  Default plan (k = b = 0): every slab is cut into
// its own blocks.  Explicit plan: the reference partition (plan.hpp:24-37) is reproduced exactly by
// making every slab a whole number of plan blocks; *resident is set when one block alone exceeds the
// slab budget (then X is uploaded whole).
struct SlabPlan {
  long long slab_rows;   // rows per slab
  long long blocks;      // kernel blocks (CTAs) per full slab
  long long rpb;         // rows per block inside a slab
  bool resident;
};

SlabPlan slab_plan(const sqb_context* ctx, long long m, int n_tot, long long k, long long b, long long P,
                   long long NW, int ctas_per_sm) {
  SlabPlan sp{0, 0, 0, false};
  if (k > 0 || b > 0) {
    if (k <= 0) k = 1;
    if (b <= 0) b = P;
    sp.rpb = make_plan(m, k, b).rpb;
    const long long budget = ctx->host_slab_bytes / (static_cast<long long>(sizeof(double)) * n_tot);
    sp.blocks = std::min(k, budget / std::max<long long>(sp.rpb, 1));
    if (sp.blocks < 1 || (sp.rpb & 1)) {  // odd block heights would leave later blocks unaligned inside a slab
      sp.resident = true;
      return sp;
    }
    sp.slab_rows = sp.blocks * sp.rpb;
    return sp;
  }
  sp.slab_rows = slab_rows_for(ctx, n_tot, even_up(P));
  sp.blocks = std::max<long long>(1, std::min<long long>(ctx->sm_count * ctas_per_sm, sp.slab_rows / (P * NW)));
  sp.rpb = make_plan(sp.slab_rows, sp.blocks, P).rpb;
  return sp;
}

// Q-less TSQR of a host matrix (optionally with one extra host column): slabs are factored as they
// land, all block triangles are stacked in ctx->work and reduced by the stage-2 tree.
int tsqr_host_stream(sqb_context* ctx, const double* x, const double* extra, long long m, int n, long long ld,
                     long long k, long long b, double* d_r, bool finalize) {
  const int nt = n + (extra ? 1 : 0);
  const long long P = tsqr_panel_rows(nt, ctx->tsqr_kind), NW = tsqr_warps(nt, ctx->tsqr_kind);
  const SlabPlan sp = slab_plan(ctx, m, nt, k, b, P, NW, 1);
  if (sp.resident) {
    long long ldx = 0;
    SQB_TRY(upload_resident(ctx, x, m, n, ld, extra ? 1 : 0, &ldx));
    MatView v = plain_view(ctx->xbuf, ldx, nt);
    if (extra) {
      SQB_CUDA(cudaMemcpyAsync(ctx->xbuf + static_cast<size_t>(ldx) * n, extra, sizeof(double) * m,
                               cudaMemcpyHostToDevice, ctx->stream));
    }
    return tsqr_view(ctx, v, m, nt, k, b, d_r, finalize);
  }
  const long long nslabs = std::max<long long>(1, ceil_div(m, sp.slab_rows));
  const long long ldy = nslabs * sp.blocks * nt;
  const size_t ymax = static_cast<size_t>(ldy) * nt;
  SQB_TRY(grow(&ctx->work, &ctx->work_doubles, 2 * ymax));
  SQB_CUDA(cudaMemsetAsync(ctx->work, 0, ymax * sizeof(double), ctx->stream));
  SQB_TRY(stream_slabs(ctx, x, extra, m, n, ld, sp.slab_rows,
                       [&](long long slab, long long, long long rows, const double* d_slab, long long lds) {
                         Plan p{std::min(sp.blocks, std::max<long long>(1, ceil_div(rows, sp.rpb))), 0, sp.rpb};
                         return launch_tsqr(ctx, plain_view(d_slab, lds, nt), rows, nt, p,
                                            ctx->work + slab * sp.blocks * nt, ldy, false, true);
                       }));
  return reduce_stack(ctx, ctx->work, ldy, ldy, nt, ctx->work + ymax, d_r, finalize);
}

int sqb_tsqr_qless_host(sqb_context* ctx, const double* x, int64_t m, int64_t n, int64_t ld,
                        int64_t num_blocks, int64_t panel_rows, double* r) {
  SQB_TRY(enter_host(ctx));
  SQB_TRY(check_shape(m, n, ld, 64));
  const int nn = static_cast<int>(n);
  Small s;
  SQB_TRY(small_slots(ctx, nn, &s));
  SQB_TRY(tsqr_host_stream(ctx, x, nullptr, m, nn, ld, num_blocks, panel_rows, s.rr, true));
  SQB_TRY(download(ctx, r, s.rr, sizeof(double) * nn * nn));
  return sqb_sync(ctx);
}

int sqb_tsqr_stage1_host(sqb_context* ctx, const double* x, int64_t m, int64_t n, int64_t ld,
                         int64_t num_blocks, int64_t panel_rows, double* y) {
  SQB_TRY(enter_host(ctx));
  if (n < 1 || n > 64 || ld < m || m < 0) return SQB_E_ARGUMENT;
  const int nn = static_cast<int>(n);
  const Plan p = tsqr_plan(ctx, m, nn, num_blocks, panel_rows);
  const size_t yd = static_cast<size_t>(p.k) * nn * nn;
  SQB_TRY(grow(&ctx->work, &ctx->work_doubles, yd));
  const long long budget = ctx->host_slab_bytes / (static_cast<long long>(sizeof(double)) * nn);
  const long long per_slab = std::min(p.k, budget / std::max<long long>(p.rpb, 1));
  if (per_slab < 1 || (p.rpb & 1)) {
    long long ldx = 0;
    SQB_TRY(upload_resident(ctx, x, m, nn, ld, 0, &ldx));
    SQB_TRY(launch_tsqr(ctx, plain_view(ctx->xbuf, ldx, nn), m, nn, p, ctx->work, p.k * nn, false, true));
  } else {
    // block i of the plan is block (i mod per_slab) of slab i / per_slab; blocks past the end of X are empty
    SQB_CUDA(cudaMemsetAsync(ctx->work, 0, yd * sizeof(double), ctx->stream));
    SQB_TRY(stream_slabs(ctx, x, nullptr, m, nn, ld, per_slab * p.rpb,
                         [&](long long slab, long long, long long rows, const double* d_slab, long long lds) {
                           Plan ps{std::min(per_slab, p.k - slab * per_slab), 0, p.rpb};
                           return launch_tsqr(ctx, plain_view(d_slab, lds, nn), rows, nn, ps,
                                              ctx->work + slab * per_slab * nn, p.k * nn, false, true);
                         }));
  }
  SQB_TRY(download(ctx, y, ctx->work, yd * sizeof(double)));
  return sqb_sync(ctx);
}

int sqb_block_qless_qr_host(sqb_context* ctx, const double* x, int64_t m, int64_t n, int64_t ld,
                            int64_t panel_rows, double* r) {
  SQB_TRY(enter_host(ctx));
  if (n < 1 || n > 64 || ld < m || m < 0) return SQB_E_ARGUMENT;
  const int nn = static_cast<int>(n);
  Small s;
  SQB_TRY(small_slots(ctx, nn, &s));
  long long ldx = 0;  // one block = one CTA walking all of X: resident copy
  SQB_TRY(upload_resident(ctx, x, m, nn, ld, 0, &ldx));
  SQB_TRY(sqb_block_qless_qr_dev(ctx, ctx->xbuf, m, n, ldx, panel_rows, s.rr));
  SQB_TRY(download(ctx, r, s.rr, sizeof(double) * nn * nn));
  return sqb_sync(ctx);
}

static int gram_host(sqb_context* ctx, const double* x, int64_t m, int64_t n, int64_t ld, int op,
                     const double* factor, int64_t k, int64_t b, double* c) {
  SQB_TRY(enter_host(ctx));
  if (n < 1 || m < 0) return SQB_E_DIMENSION;
  if (n > kWideGramMaxN || ld < m) return SQB_E_ARGUMENT;
  const int nn = static_cast<int>(n);
  Small s;
  SQB_TRY(small_slots(ctx, nn, &s));
  if (factor) SQB_TRY(upload_small(ctx, factor, static_cast<size_t>(nn) * nn, s.r1));
  const double* d_factor = factor ? s.r1 : nullptr;
  SlabPlan sp{0, 0, 0, true};
  if (nn <= 64) sp = slab_plan(ctx, m, nn, k, b, gram_panel_rows(nn, op), gram_warps(nn), gram_ctas_per_sm(nn, op));
  if (sp.resident) {  // wide kernels (own row partition) and oversized explicit blocks
    long long ldx = 0;
    SQB_TRY(upload_resident(ctx, x, m, nn, ld, 0, &ldx));
    SQB_TRY(gram_entry(ctx, ctx->xbuf, m, n, ldx, op, d_factor, k, b, s.rr));
  } else {
    if (op == OP_MULTIPLY) {  // tsmmttsmm checks B for finiteness (gram.cpp:143-145)
      SQB_CUDA(launch_check_finite(d_factor, n * n, ctx->d_status, ctx->stream));
      ctx->launches++;
    }
    // per-block partial Grams of all slabs, summed in ascending block order by one reduce launch
    const long long nslabs = std::max<long long>(1, ceil_div(m, sp.slab_rows));
    const size_t pd = static_cast<size_t>(nslabs) * sp.blocks * nn * nn;
    SQB_TRY(grow(&ctx->work, &ctx->work_doubles, pd));
    SQB_CUDA(cudaMemsetAsync(ctx->work, 0, pd * sizeof(double), ctx->stream));
    SQB_TRY(stream_slabs(ctx, x, nullptr, m, nn, ld, sp.slab_rows,
                         [&](long long slab, long long, long long rows, const double* d_slab, long long lds) {
                           Plan p{std::min(sp.blocks, std::max<long long>(1, ceil_div(rows, sp.rpb))), 0, sp.rpb};
                           return launch_gram_blocks(ctx, plain_view(d_slab, lds, nn), rows, nn, op, d_factor, p,
                                                     ctx->work + static_cast<size_t>(slab) * sp.blocks * nn * nn,
                                                     op == OP_PLAIN);
                         }));
    SQB_CUDA(launch_gram_reduce(ctx->work, nslabs * sp.blocks, nn, s.rr, op == OP_PLAIN ? 1 : 0, ctx->d_status,
                                ctx->stream));
    ctx->launches++;
  }
  SQB_TRY(download(ctx, c, s.rr, sizeof(double) * nn * nn));
  return sqb_sync(ctx);
}

int sqb_tsmttsm_host(sqb_context* ctx, const double* x, int64_t m, int64_t n, int64_t ld,
                     int64_t num_blocks, int64_t panel_rows, double* c) {
  return gram_host(ctx, x, m, n, ld, OP_PLAIN, nullptr, num_blocks, panel_rows, c);
}
int sqb_tsmRttsmR_host(sqb_context* ctx, const double* x, int64_t m, int64_t n, int64_t ld,
                       const double* r, int64_t num_blocks, int64_t panel_rows, double* c) {
  return gram_host(ctx, x, m, n, ld, OP_SOLVE, r, num_blocks, panel_rows, c);
}
int sqb_tsmmttsmm_host(sqb_context* ctx, const double* x, int64_t m, int64_t n, int64_t ld,
                       const double* b, int64_t num_blocks, int64_t panel_rows, double* c) {
  return gram_host(ctx, x, m, n, ld, OP_MULTIPLY, b, num_blocks, panel_rows, c);
}

int sqb_cholesky_host(sqb_context* ctx, const double* c, int64_t n, double* r) {
  SQB_TRY(enter_host(ctx));
  if (n < 1) return SQB_E_DIMENSION;
  if (n > kWideGramMaxN) return SQB_E_ARGUMENT;
  Small s;
  SQB_TRY(small_slots(ctx, static_cast<int>(n), &s));
  SQB_TRY(upload_small(ctx, c, static_cast<size_t>(n) * n, s.c1));
  SQB_TRY(sqb_cholesky_dev(ctx, s.c1, n, s.r1));
  SQB_TRY(download(ctx, r, s.r1, sizeof(double) * n * n));
  return sqb_sync(ctx);
}

int sqb_eigh_small_host(sqb_context* ctx, const double* c, int64_t n, double* values,
                        double* vectors) {
  SQB_TRY(enter_host(ctx));
  if (n < 1) return SQB_E_DIMENSION;
  if (n > kSmallMaxN) return SQB_E_ARGUMENT;
  Small s;
  SQB_TRY(small_slots(ctx, static_cast<int>(n), &s));
  SQB_TRY(upload_small(ctx, c, static_cast<size_t>(n) * n, s.c1));
  SQB_TRY(sqb_eigh_small_dev(ctx, s.c1, n, s.s2, s.r1));
  SQB_TRY(download(ctx, values, s.s2, sizeof(double) * n));
  SQB_TRY(download(ctx, vectors, s.r1, sizeof(double) * n * n));
  return sqb_sync(ctx);
}

int sqb_cholqr2_host(sqb_context* ctx, const double* x, int64_t m, int64_t n, int64_t ld,
                     int64_t num_blocks, int64_t panel_rows, double* r) {
  SQB_TRY(enter_host(ctx));
  SQB_TRY(check_shape(m, n, ld, kWideGramMaxN));
  const int nn = static_cast<int>(n);
  Small s;
  SQB_TRY(small_slots(ctx, nn, &s));
  long long ldx = 0;  // X is read twice: resident copy
  SQB_TRY(upload_resident(ctx, x, m, nn, ld, 0, &ldx));
  if (nn > 64) SQB_TRY(cholqr2_wide(ctx, plain_view(ctx->xbuf, ldx, nn), m, nn, s.rr, nullptr));
  else SQB_TRY(cholqr2_view(ctx, plain_view(ctx->xbuf, ldx, nn), m, nn, num_blocks, panel_rows, s.rr, nullptr));
  SQB_TRY(download(ctx, r, s.rr, sizeof(double) * nn * nn));
  return sqb_sync(ctx);
}

int sqb_svqb_pass_host(sqb_context* ctx, const double* c, int64_t n, double* b, double* z,
                       double* sigma, int64_t* rank) {
  SQB_TRY(enter_host(ctx));
  if (n < 1) return SQB_E_DIMENSION;
  if (n > kSmallMaxN) return SQB_E_ARGUMENT;
  Small s;
  SQB_TRY(small_slots(ctx, static_cast<int>(n), &s));
  SQB_TRY(upload_small(ctx, c, static_cast<size_t>(n) * n, s.c1));
  SQB_TRY(sqb_svqb_pass_dev(ctx, s.c1, n, s.b1, s.z1, s.s2, reinterpret_cast<int64_t*>(s.rank1)));
  SQB_TRY(download(ctx, b, s.b1, sizeof(double) * n * n));
  SQB_TRY(download(ctx, z, s.z1, sizeof(double) * n * n));
  SQB_TRY(download(ctx, sigma, s.s2, sizeof(double) * n));
  SQB_TRY(download(ctx, rank, s.rank1, sizeof(int64_t)));
  return sqb_sync(ctx);
}

int sqb_svqb2_host(sqb_context* ctx, const double* x, int64_t m, int64_t n, int64_t ld,
                   int64_t num_blocks, int64_t panel_rows, double* transform, double* z,
                   double* sigma, int64_t* rank) {
  SQB_TRY(enter_host(ctx));
  SQB_TRY(check_shape(m, n, ld, kWideFusedMaxN));
  const int nn = static_cast<int>(n);
  const size_t sq = static_cast<size_t>(nn) * nn;
  Small s;
  SQB_TRY(small_slots(ctx, nn, &s));
  long long ldx = 0;
  SQB_TRY(upload_resident(ctx, x, m, nn, ld, 0, &ldx));
  if (nn > 64)
    SQB_TRY(svqb2_wide(ctx, plain_view(ctx->xbuf, ldx, nn), m, nn, s.rr, s.rr + sq, s.s2 + nn, s.rank1 + 1, nullptr));
  else
    SQB_TRY(svqb2_view(ctx, plain_view(ctx->xbuf, ldx, nn), m, nn, num_blocks, panel_rows, s.rr, s.rr + sq,
                       s.s2 + nn, s.rank1 + 1, nullptr));
  SQB_TRY(download(ctx, transform, s.rr, sizeof(double) * sq));
  SQB_TRY(download(ctx, z, s.rr + sq, sizeof(double) * sq));
  SQB_TRY(download(ctx, sigma, s.s2 + nn, sizeof(double) * nn));
  SQB_TRY(download(ctx, rank, s.rank1 + 1, sizeof(int64_t)));
  return sqb_sync(ctx);
}

int sqb_reconstruct_q_host(sqb_context* ctx, const double* x, int64_t m, int64_t n, int64_t ld,
                           const double* r, double* q, int64_t ldq) {
  SQB_TRY(enter_host(ctx));
  if (n < 1 || m < 0) return SQB_E_DIMENSION;
  if (n > kWideGramMaxN || ld < m || ldq < m) return SQB_E_ARGUMENT;
  const int nn = static_cast<int>(n);
  Small s;
  SQB_TRY(small_slots(ctx, nn, &s));
  SQB_TRY(upload_small(ctx, r, static_cast<size_t>(nn) * nn, s.r1));
  long long ldx = 0;
  SQB_TRY(upload_resident(ctx, x, m, nn, ld, 0, &ldx));
  SQB_TRY(grow(&ctx->gen, &ctx->gen_doubles, static_cast<size_t>(ldx) * nn));
  SQB_TRY(sqb_reconstruct_q_dev(ctx, ctx->xbuf, m, n, ldx, s.r1, ctx->gen, ldx));
  SQB_CUDA(cudaMemcpy2DAsync(q, sizeof(double) * ldq, ctx->gen, sizeof(double) * ldx, sizeof(double) * m,
                             nn, cudaMemcpyDeviceToHost, ctx->stream));
  return sqb_sync(ctx);
}

int sqb_solve_lstsq_host(sqb_context* ctx, const double* a, int64_t m, int64_t n, int64_t lda,
                         const double* rhs, int method, double* xsol, double* residual) {
  SQB_TRY(enter_host(ctx));
  if (n < 1 || m < n + 1) return SQB_E_DIMENSION;
  if (n + 1 > kWideFusedMaxN || lda < m) return SQB_E_ARGUMENT;
  const int nn = static_cast<int>(n);
  Small s;
  SQB_TRY(small_slots(ctx, nn + 1, &s));
  double* d_out = s.s2 + 2 * (nn + 1);
  if (method == SQB_METHOD_TSQR) {
    // single pass: [A rhs] streams through the slab ring, rhs travelling as the last column
    if (nn + 1 > 64) return SQB_E_ARGUMENT;  // tsqr.cpp:188
    SQB_TRY(tsqr_host_stream(ctx, a, rhs, m, nn, lda, 0, 0, s.rr, true));
    SQB_CUDA(launch_backsolve(s.rr, nn + 1, d_out, d_out + nn, ctx->d_status, ctx->stream));
    ctx->launches++;
  } else {
    // two passes: [A rhs] lands as one resident (n+1)-column matrix, rhs in the last column
    long long ldx = 0;
    SQB_TRY(upload_resident(ctx, a, m, nn, lda, 1, &ldx));
    double* d_rhs = ctx->xbuf + static_cast<size_t>(ldx) * nn;
    SQB_CUDA(cudaMemcpyAsync(d_rhs, rhs, sizeof(double) * m, cudaMemcpyHostToDevice, ctx->stream));
    const MatView v{ctx->xbuf, ldx, d_rhs, nn};
    SQB_TRY(lstsq_view(ctx, v, m, nn + 1, method, d_out, d_out + nn, false));
  }
  SQB_TRY(download(ctx, xsol, d_out, sizeof(double) * nn));
  SQB_TRY(download(ctx, residual, d_out + nn, sizeof(double)));
  return sqb_sync(ctx);
}

// ---- synthetic inputs ------------------------------------------------------------------------------
int sqb_fill_gaussian_dev(sqb_context* ctx, double* d_x, int64_t m, int64_t n, int64_t ld,
                          uint64_t seed, int64_t row_offset, int64_t m_total) {
  SQB_TRY(enter(ctx));
  if (m < 0 || n < 1 || ld < m) return SQB_E_ARGUMENT;
  SQB_CUDA(launch_fill_gaussian(d_x, m, static_cast<int>(n), ld, seed, row_offset, m_total, ctx->stream));
  ctx->launches++;
  return SQB_OK;
}

int sqb_generate_dev(sqb_context* ctx, double* d_x, int64_t m, int64_t n, int64_t ld, double kappa,
                     int linear_decay, uint64_t seed) {
  SQB_TRY(enter(ctx));
  // matgen.cpp:78-83
  if (n < 1 || m < n || n > 64 || ld < m || !(kappa >= 1.0) || (n == 1 && kappa != 1.0))
    return SQB_E_ARGUMENT;
  SQB_TRY(grow(&ctx->gen, &ctx->gen_doubles, generate_scratch_doubles(m, static_cast<int>(n))));
  SQB_CUDA(launch_generate(d_x, m, static_cast<int>(n), ld, kappa, linear_decay, seed, ctx->gen,
                           ctx->stream));
  ctx->launches += 3 * n + 3;
  return SQB_OK;
}

// ---- multi-GPU ----------------------------------------------------------------------------------------
int sqb_attach_nccl(sqb_context* ctx, void* nccl_comm, int rank, int world) {
  SQB_TRY(enter(ctx));
  if (world < 1 || rank < 0 || rank >= world) return SQB_E_ARGUMENT;
  if (world > 1 && (!nccl_comm || !nccl().ok)) return SQB_E_NCCL;
  ctx->nccl_comm = nccl_comm;
  ctx->own_comm = false;
  ctx->rank = rank;
  ctx->world = world;
  return SQB_OK;
}

int sqb_set_allgather(sqb_context* ctx, sqb_allgather_fn fn, void* user, int rank, int world) {
  SQB_TRY(enter(ctx));
  if (world < 1 || rank < 0 || rank >= world || (world > 1 && !fn)) return SQB_E_ARGUMENT;
  ctx->gather_fn = fn;
  ctx->gather_user = user;
  ctx->rank = rank;
  ctx->world = world;
  return SQB_OK;
}

int sqb_tsqr_local_dev(sqb_context* ctx, const double* d_x, int64_t m_local, int64_t n, int64_t ld,
                       double* d_r_local) {
  SQB_TRY(enter(ctx));
  if (n < 1 || m_local < 0) return SQB_E_DIMENSION;
  if (n > 64 || ld < m_local) return SQB_E_ARGUMENT;
  return tsqr_local_view(ctx, plain_view(d_x, ld, static_cast<int>(n)), m_local, static_cast<int>(n), d_r_local);
}

int sqb_tsqr_combine_dev(sqb_context* ctx, const double* d_gathered, int64_t world, int64_t n, double* d_r) {
  SQB_TRY(enter(ctx));
  if (n < 1 || world < 1) return SQB_E_DIMENSION;
  if (n > 64 || world > (1 << 20)) return SQB_E_ARGUMENT;
  const size_t nn = static_cast<size_t>(n) * n;
  SQB_TRY(grow(&ctx->gen, &ctx->gen_doubles, nn * world));
  return tsqr_combine(ctx, d_gathered, static_cast<int>(world), static_cast<int>(n), ctx->gen, d_r);
}

int sqb_gram_combine_dev(sqb_context* ctx, const double* d_gathered, int64_t world, int64_t n, double* d_c) {
  SQB_TRY(enter(ctx));
  if (n < 1 || world < 1) return SQB_E_DIMENSION;
  if (world > (1 << 20)) return SQB_E_ARGUMENT;
  return gram_combine(ctx, d_gathered, static_cast<int>(world), static_cast<int>(n), d_c);
}

int sqb_nccl_unique_id(void* out128) {
  if (!out128 || !nccl().ok) return SQB_E_NCCL;
  return nccl().GetUniqueId(static_cast<NcclId*>(out128)) == 0 ? SQB_OK : SQB_E_NCCL;
}

int sqb_init_nccl(sqb_context* ctx, const void* unique_id128, int rank, int world) {
  SQB_TRY(enter(ctx));
  if (world < 1 || rank < 0 || rank >= world || !unique_id128) return SQB_E_ARGUMENT;
  if (!nccl().ok) return SQB_E_NCCL;
  NcclId id;
  std::memcpy(&id, unique_id128, sizeof(id));
  void* comm = nullptr;
  if (nccl().CommInitRank(&comm, world, id, rank) != 0) return SQB_E_NCCL;
  ctx->nccl_comm = comm;
  ctx->own_comm = true;
  ctx->rank = rank;
  ctx->world = world;
  return SQB_OK;
}

int sqb_tsqr_qless_sharded_dev(sqb_context* ctx, const double* d_x, int64_t m_local, int64_t n,
                               int64_t ld, double* d_r) {
  SQB_TRY(enter(ctx));
  if (n < 1 || m_local < 0) return SQB_E_DIMENSION;
  if (n > 64 || ld < m_local) return SQB_E_ARGUMENT;
  return tsqr_sharded_view(ctx, plain_view(d_x, ld, static_cast<int>(n)), m_local, static_cast<int>(n),
                           d_r);
}

// Host slab of this rank -> slab ring -> local triangle -> exchange -> combine -> host R.
int sqb_tsqr_qless_sharded_host(sqb_context* ctx, const double* x, int64_t m_local, int64_t n, int64_t ld,
                                double* r) {
  SQB_TRY(enter_host(ctx));
  if (n < 1 || m_local < 0) return SQB_E_DIMENSION;
  if (n > 64 || ld < m_local) return SQB_E_ARGUMENT;
  const int nn = static_cast<int>(n);
  Small s;
  SQB_TRY(small_slots(ctx, nn, &s));
  if (!is_sharded(ctx)) {
    SQB_TRY(tsqr_host_stream(ctx, x, nullptr, m_local, nn, ld, 0, 0, s.rr, true));
  } else {
    if (m_local > 0) SQB_TRY(tsqr_host_stream(ctx, x, nullptr, m_local, nn, ld, 0, 0, s.c1, false));
    else SQB_CUDA(cudaMemsetAsync(s.c1, 0, sizeof(double) * nn * nn, ctx->stream));
    double *gathered, *stack;
    SQB_TRY(exchange_scratch(ctx, nn, &gathered, &stack));
    SQB_TRY(allgather_blocks(ctx, s.c1, gathered, static_cast<size_t>(nn) * nn));
    SQB_TRY(tsqr_combine(ctx, gathered, ctx->world, nn, stack, s.rr));
  }
  SQB_TRY(download(ctx, r, s.rr, sizeof(double) * nn * nn));
  return sqb_sync(ctx);
}

int sqb_cholqr2_sharded_dev(sqb_context* ctx, const double* d_x, int64_t m_local, int64_t n,
                            int64_t ld, double* d_r) {
  SQB_TRY(enter(ctx));
  if (n < 1 || m_local < 0) return SQB_E_DIMENSION;
  if (n > kWideGramMaxN || ld < m_local) return SQB_E_ARGUMENT;
  const int nn = static_cast<int>(n);
  if (nn > 64)
    return cholqr2_wide(ctx, plain_view(d_x, ld, nn), m_local, nn, d_r,
                        [ctx, nn](double* d) { return allreduce_square(ctx, d, nn); });
  return cholqr2_view(ctx, plain_view(d_x, ld, nn), m_local, nn, 0, 0, d_r,
                      [ctx, nn](double* d) { return allreduce_square(ctx, d, nn); });
}

int sqb_svqb2_sharded_dev(sqb_context* ctx, const double* d_x, int64_t m_local, int64_t n,
                          int64_t ld, double* d_transform, double* d_z, double* d_sigma,
                          int64_t* d_rank) {
  SQB_TRY(enter(ctx));
  if (n < 1 || m_local < 0) return SQB_E_DIMENSION;
  if (n > kWideFusedMaxN || ld < m_local) return SQB_E_ARGUMENT;
  const int nn = static_cast<int>(n);
  if (nn > 64)
    return svqb2_wide(ctx, plain_view(d_x, ld, nn), m_local, nn, d_transform, d_z, d_sigma,
                      reinterpret_cast<long long*>(d_rank),
                      [ctx, nn](double* d) { return allreduce_square(ctx, d, nn); });
  return svqb2_view(ctx, plain_view(d_x, ld, nn), m_local, nn, 0, 0, d_transform, d_z, d_sigma,
                    reinterpret_cast<long long*>(d_rank),
                    [ctx, nn](double* d) { return allreduce_square(ctx, d, nn); });
}

int sqb_solve_lstsq_sharded_dev(sqb_context* ctx, const double* d_a, int64_t m_local, int64_t n,
                                int64_t lda, const double* d_rhs, double* d_xsol,
                                double* d_residual) {
  SQB_TRY(enter(ctx));
  if (n < 1 || m_local < 0) return SQB_E_DIMENSION;
  if (n + 1 > 64 || lda < m_local) return SQB_E_ARGUMENT;  // sharded least squares is the TSQR route
  const MatView v{d_a, lda, d_rhs, static_cast<int>(n)};
  return lstsq_view(ctx, v, m_local, static_cast<int>(n) + 1, SQB_METHOD_TSQR, d_xsol, d_residual,
                    true);
}

}  // extern "C"
