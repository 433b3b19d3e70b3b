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
  const long long P = tsqr_panel_rows(n), NW = tsqr_warps(n);
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
  SQB_CUDA(launch_tsqr_any(prm, p.k, ctx->stream));
  ctx->launches++;
  return SQB_OK;
}

// Reduce a stack of triangles (rows x n, dense column-major, leading dimension ld) to one
// triangle: the reference's stage 2 (tsqr.cpp:193-195), as a short tree of the same kernel.
int reduce_stack(sqb_context* ctx, double* stack, long long rows, long long ld, int n,
                 double* scratch, double* d_r, bool finalize) {
  const long long P = tsqr_panel_rows(n), NW = tsqr_warps(n);
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
  const size_t want = 10 * nn + 4 * n + (nn + 3 * n + 16) + 8;
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

// ---- wide column counts (64 < n): plain Gram up to 256 columns, fused solve + Gram up to 128 ----
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
  if (n > kWideFusedMaxN) return SQB_E_ARGUMENT;
  SQB_TRY(grow(&ctx->work, &ctx->work_doubles, partial + gram_wide_fused_scratch_doubles()));
  SQB_CUDA(launch_gram_wide_fused(v, m, n, op, factor, ctx->sm_count, ctx->work + partial, ctx->work, d_c,
                                  ctx->d_status, ctx->stream));
  ctx->launches += 3;
  return SQB_OK;
}

// CholQR2 beyond 64 columns (the reference's cholqr2 has no column limit, gram_qr.cpp:123-131): the
// wide SYRK, the one-CTA Cholesky (n <= 128), the fused solve + Gram sweep, Cholesky, R = R2 R1.
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
// Streams X into a resident device buffer in row slabs (copy stream) and hands every slab, as soon
// as it has landed, to `on_slab(row0, rows)` which enqueues work on the compute stream.
constexpr size_t kSlabBytes = 256u << 20;

int upload_slabs(sqb_context* ctx, const double* x, long long m, int n, long long ld,
                 long long row_align, const std::function<int(long long, long long)>& on_slab) {
  SQB_TRY(grow(&ctx->xbuf, &ctx->xbuf_doubles, static_cast<size_t>(m) * n + 2));
  long long slab_rows = static_cast<long long>(kSlabBytes / (sizeof(double) * n));
  slab_rows = std::max(row_align, slab_rows / row_align * row_align);
  for (long long r0 = 0; r0 < m; r0 += slab_rows) {
    const long long rows = std::min(slab_rows, m - r0);
    SQB_CUDA(cudaMemcpy2DAsync(ctx->xbuf + r0, sizeof(double) * m, x + r0, sizeof(double) * ld,
                               sizeof(double) * rows, n, cudaMemcpyHostToDevice, ctx->copy_stream));
    SQB_CUDA(cudaEventRecord(ctx->slab_ready, ctx->copy_stream));
    SQB_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->slab_ready, 0));
    if (on_slab) SQB_TRY(on_slab(r0, rows));
  }
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

int allreduce_square(sqb_context* ctx, double* d, int n) {
  if (ctx->world <= 1 && !ctx->nccl_comm) return SQB_OK;  // an attached 1-rank communicator is used
  NcclApi& api = nccl();
  if (!api.ok || !ctx->nccl_comm) return SQB_E_NCCL;
  const int rc = api.AllReduce(d, d, static_cast<size_t>(n) * n, kNcclFloat64, kNcclSum,
                               ctx->nccl_comm, ctx->stream);
  return rc == 0 ? SQB_OK : SQB_E_NCCL;
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

// Local triangle -> all-gather -> redundant final combine on every rank (stage 2 with k = world).
int tsqr_sharded_view(sqb_context* ctx, const MatView& v, long long m_local, int n, double* d_r) {
  if (ctx->world <= 1 && !ctx->nccl_comm) return tsqr_view(ctx, v, m_local, n, 0, 0, d_r, true);
  NcclApi& api = nccl();
  if (!api.ok || !ctx->nccl_comm) return SQB_E_NCCL;
  Small s;
  SQB_TRY(small_slots(ctx, n, &s));
  const size_t nn = static_cast<size_t>(n) * n;
  // a rank may own fewer than n rows (or none): its triangle is then that of a zero-padded slab
  if (m_local > 0) {
    SQB_TRY(tsqr_view(ctx, v, m_local, n, 0, 0, s.c1, false));
  } else {
    SQB_CUDA(cudaMemsetAsync(s.c1, 0, nn * sizeof(double), ctx->stream));
  }
  const size_t need = 2 * nn * ctx->world;
  SQB_TRY(grow(&ctx->gen, &ctx->gen_doubles, need));
  double* gathered = ctx->gen;
  double* stack = ctx->gen + nn * ctx->world;
  if (api.AllGather(s.c1, gathered, nn, kNcclFloat64, ctx->nccl_comm, ctx->stream) != 0)
    return SQB_E_NCCL;
  pack_stack_kernel<<<8, 256, 0, ctx->stream>>>(gathered, ctx->world, n, stack);
  ctx->launches++;
  const long long rows = static_cast<long long>(ctx->world) * n;
  return launch_tsqr(ctx, plain_view(stack, rows, n), rows, n, make_plan(rows, 1, rows), d_r, n, true,
                     false);
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
  const int64_t b = panel_rows > 0 ? panel_rows : tsqr_panel_rows(static_cast<int>(n));
  Plan p{1, b, ceil_div(std::max<int64_t>(m, 1), b) * b};
  return launch_tsqr(ctx, plain_view(d_x, ld, static_cast<int>(n)), m, static_cast<int>(n), p, d_r, n,
                     false, true);
}

static int gram_entry(sqb_context* ctx, const double* d_x, int64_t m, int64_t n, int64_t ld, int op,
                      const double* factor, int64_t k, int64_t b, double* d_c) {
  SQB_TRY(enter(ctx));
  if (n < 1 || m < 0) return SQB_E_DIMENSION;
  if (ld < m) return SQB_E_ARGUMENT;
  if (n > 64) {
    // the reference's Gram kernels have no column limit (gram.cpp:113-151); here the plain Gram goes
    // up to 256 columns and the fused solve + Gram up to 128; the fused multiply stays at n <= 64
    return gram_wide_view(ctx, plain_view(d_x, ld, static_cast<int>(n)), m, static_cast<int>(n), op, factor, d_c,
                          op == OP_PLAIN);
  }
  if (op == OP_MULTIPLY) {  // tsmmttsmm checks B for finiteness (gram.cpp:143-145)
    SQB_CUDA(launch_check_finite(factor, n * n, ctx->d_status, ctx->stream));
    ctx->launches++;
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
  if (n > kSmallMaxN) return SQB_E_ARGUMENT;
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
  SQB_TRY(check_shape(m, n, ld, kWideFusedMaxN));
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
  if (n > kWideFusedMaxN || ld < m || ldq < m) return SQB_E_ARGUMENT;
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
int sqb_tsqr_qless_host(sqb_context* ctx, const double* x, int64_t m, int64_t n, int64_t ld,
                        int64_t num_blocks, int64_t panel_rows, double* r) {
  SQB_TRY(enter(ctx));
  SQB_TRY(check_shape(m, n, ld, 64));
  const int nn = static_cast<int>(n);
  Small s;
  SQB_TRY(small_slots(ctx, nn, &s));
  if (num_blocks > 0 || panel_rows > 0) {
    // explicit plan: reproduce the reference partition exactly on the resident copy
    SQB_TRY(upload_slabs(ctx, x, m, nn, ld, 2, nullptr));
    SQB_TRY(tsqr_view(ctx, plain_view(ctx->xbuf, m, nn), m, nn, num_blocks, panel_rows, s.rr, true));
  } else {
    // default plan: every slab is factored as soon as it lands; all slab triangles are stacked
    const long long P = tsqr_panel_rows(nn), NW = tsqr_warps(nn);
    long long slab_rows = static_cast<long long>(kSlabBytes / (sizeof(double) * n));
    slab_rows = std::max(P, slab_rows / P * P);
    const long long nslabs = ceil_div(m, slab_rows);
    const long long kmax = std::max<long long>(1, std::min<long long>(ctx->sm_count, slab_rows / (P * NW)));
    const size_t ymax = static_cast<size_t>(nslabs) * kmax * nn * nn;
    SQB_TRY(grow(&ctx->work, &ctx->work_doubles, 2 * ymax));
    const long long ldy = nslabs * kmax * nn;
    SQB_CUDA(cudaMemsetAsync(ctx->work, 0, ymax * sizeof(double), ctx->stream));
    long long slab = 0;
    SQB_TRY(upload_slabs(ctx, x, m, nn, ld, P, [&](long long r0, long long rows) {
      const long long k = std::max<long long>(1, std::min<long long>(kmax, rows / (P * NW)));
      const Plan p = make_plan(rows, k, P);
      const int st = launch_tsqr(ctx, plain_view(ctx->xbuf + r0, m, nn), rows, nn, p,
                                 ctx->work + slab * kmax * nn, ldy, false, true);
      ++slab;
      return st;
    }));
    SQB_TRY(reduce_stack(ctx, ctx->work, ldy, ldy, nn, ctx->work + ymax, s.rr, true));
  }
  SQB_TRY(download(ctx, r, s.rr, sizeof(double) * nn * nn));
  return sqb_sync(ctx);
}

int sqb_tsqr_stage1_host(sqb_context* ctx, const double* x, int64_t m, int64_t n, int64_t ld,
                         int64_t num_blocks, int64_t panel_rows, double* y) {
  SQB_TRY(enter(ctx));
  if (n < 1 || n > 64 || ld < m || m < 0) return SQB_E_ARGUMENT;
  const int nn = static_cast<int>(n);
  const Plan p = tsqr_plan(ctx, m, nn, num_blocks, panel_rows);
  SQB_TRY(upload_slabs(ctx, x, m, nn, ld, 2, nullptr));
  const size_t yd = static_cast<size_t>(p.k) * nn * nn;
  SQB_TRY(grow(&ctx->work, &ctx->work_doubles, yd));
  SQB_TRY(launch_tsqr(ctx, plain_view(ctx->xbuf, m, nn), m, nn, p, ctx->work, p.k * nn, false, true));
  SQB_TRY(download(ctx, y, ctx->work, yd * sizeof(double)));
  return sqb_sync(ctx);
}

int sqb_block_qless_qr_host(sqb_context* ctx, const double* x, int64_t m, int64_t n, int64_t ld,
                            int64_t panel_rows, double* r) {
  SQB_TRY(enter(ctx));
  if (n < 1 || n > 64 || ld < m || m < 0) return SQB_E_ARGUMENT;
  const int nn = static_cast<int>(n);
  Small s;
  SQB_TRY(small_slots(ctx, nn, &s));
  SQB_TRY(upload_slabs(ctx, x, m, nn, ld, 2, nullptr));
  SQB_TRY(sqb_block_qless_qr_dev(ctx, ctx->xbuf, m, n, m, panel_rows, s.rr));
  SQB_TRY(download(ctx, r, s.rr, sizeof(double) * nn * nn));
  return sqb_sync(ctx);
}

static int gram_host(sqb_context* ctx, const double* x, int64_t m, int64_t n, int64_t ld, int op,
                     const double* factor, int64_t k, int64_t b, double* c) {
  SQB_TRY(enter(ctx));
  if (n < 1 || m < 0) return SQB_E_DIMENSION;
  if (n > (op == OP_PLAIN ? kWideGramMaxN : kWideFusedMaxN) || ld < m) return SQB_E_ARGUMENT;
  const int nn = static_cast<int>(n);
  Small s;
  SQB_TRY(small_slots(ctx, nn, &s));
  if (factor) SQB_TRY(upload_small(ctx, factor, static_cast<size_t>(nn) * nn, s.r1));
  SQB_TRY(upload_slabs(ctx, x, m, nn, ld, 2, nullptr));
  SQB_TRY(gram_entry(ctx, ctx->xbuf, m, n, m, op, factor ? s.r1 : nullptr, k, b, s.rr));
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
  SQB_TRY(enter(ctx));
  if (n < 1) return SQB_E_DIMENSION;
  if (n > kSmallMaxN) return SQB_E_ARGUMENT;
  Small s;
  SQB_TRY(small_slots(ctx, static_cast<int>(n), &s));
  SQB_TRY(upload_small(ctx, c, static_cast<size_t>(n) * n, s.c1));
  SQB_TRY(sqb_cholesky_dev(ctx, s.c1, n, s.r1));
  SQB_TRY(download(ctx, r, s.r1, sizeof(double) * n * n));
  return sqb_sync(ctx);
}

int sqb_eigh_small_host(sqb_context* ctx, const double* c, int64_t n, double* values,
                        double* vectors) {
  SQB_TRY(enter(ctx));
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
  SQB_TRY(enter(ctx));
  SQB_TRY(check_shape(m, n, ld, kWideFusedMaxN));
  const int nn = static_cast<int>(n);
  Small s;
  SQB_TRY(small_slots(ctx, nn, &s));
  SQB_TRY(upload_slabs(ctx, x, m, nn, ld, 2, nullptr));
  if (nn > 64) SQB_TRY(cholqr2_wide(ctx, plain_view(ctx->xbuf, m, nn), m, nn, s.rr, nullptr));
  else SQB_TRY(cholqr2_view(ctx, plain_view(ctx->xbuf, m, nn), m, nn, num_blocks, panel_rows, s.rr, nullptr));
  SQB_TRY(download(ctx, r, s.rr, sizeof(double) * nn * nn));
  return sqb_sync(ctx);
}

int sqb_svqb_pass_host(sqb_context* ctx, const double* c, int64_t n, double* b, double* z,
                       double* sigma, int64_t* rank) {
  SQB_TRY(enter(ctx));
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
  SQB_TRY(enter(ctx));
  SQB_TRY(check_shape(m, n, ld, kWideFusedMaxN));
  const int nn = static_cast<int>(n);
  const size_t sq = static_cast<size_t>(nn) * nn;
  Small s;
  SQB_TRY(small_slots(ctx, nn, &s));
  SQB_TRY(upload_slabs(ctx, x, m, nn, ld, 2, nullptr));
  if (nn > 64)
    SQB_TRY(svqb2_wide(ctx, plain_view(ctx->xbuf, m, nn), m, nn, s.rr, s.rr + sq, s.s2 + nn, s.rank1 + 1, nullptr));
  else
    SQB_TRY(svqb2_view(ctx, plain_view(ctx->xbuf, m, nn), m, nn, num_blocks, panel_rows, s.rr, s.rr + sq,
                       s.s2 + nn, s.rank1 + 1, nullptr));
  SQB_TRY(download(ctx, transform, s.rr, sizeof(double) * sq));
  SQB_TRY(download(ctx, z, s.rr + sq, sizeof(double) * sq));
  SQB_TRY(download(ctx, sigma, s.s2 + nn, sizeof(double) * nn));
  SQB_TRY(download(ctx, rank, s.rank1 + 1, sizeof(int64_t)));
  return sqb_sync(ctx);
}

int sqb_reconstruct_q_host(sqb_context* ctx, const double* x, int64_t m, int64_t n, int64_t ld,
                           const double* r, double* q, int64_t ldq) {
  SQB_TRY(enter(ctx));
  if (n < 1 || m < 0) return SQB_E_DIMENSION;
  if (n > kWideFusedMaxN || ld < m || ldq < m) return SQB_E_ARGUMENT;
  const int nn = static_cast<int>(n);
  Small s;
  SQB_TRY(small_slots(ctx, nn, &s));
  SQB_TRY(upload_small(ctx, r, static_cast<size_t>(nn) * nn, s.r1));
  SQB_TRY(upload_slabs(ctx, x, m, nn, ld, 2, nullptr));
  SQB_TRY(grow(&ctx->gen, &ctx->gen_doubles, static_cast<size_t>(m) * nn));
  SQB_TRY(sqb_reconstruct_q_dev(ctx, ctx->xbuf, m, n, m, s.r1, ctx->gen, m));
  SQB_CUDA(cudaMemcpy2DAsync(q, sizeof(double) * ldq, ctx->gen, sizeof(double) * m, sizeof(double) * m,
                             nn, cudaMemcpyDeviceToHost, ctx->stream));
  return sqb_sync(ctx);
}

int sqb_solve_lstsq_host(sqb_context* ctx, const double* a, int64_t m, int64_t n, int64_t lda,
                         const double* rhs, int method, double* xsol, double* residual) {
  SQB_TRY(enter(ctx));
  if (n < 1 || m < n + 1) return SQB_E_DIMENSION;
  if (n + 1 > kWideFusedMaxN || lda < m) return SQB_E_ARGUMENT;
  const int nn = static_cast<int>(n);
  Small s;
  SQB_TRY(small_slots(ctx, nn + 1, &s));
  // [A rhs] lands as one resident (n+1)-column matrix: rhs is simply the last column's slab
  SQB_TRY(grow(&ctx->xbuf, &ctx->xbuf_doubles, static_cast<size_t>(m) * (nn + 1) + 2));
  SQB_TRY(upload_slabs(ctx, a, m, nn, lda, 2, nullptr));
  SQB_CUDA(cudaMemcpyAsync(ctx->xbuf + static_cast<size_t>(m) * nn, rhs, sizeof(double) * m,
                           cudaMemcpyHostToDevice, ctx->stream));
  const MatView v{ctx->xbuf, m, ctx->xbuf + static_cast<size_t>(m) * nn, nn};
  double* d_out = s.s2 + 2 * (nn + 1);
  SQB_TRY(lstsq_view(ctx, v, m, nn + 1, method, d_out, d_out + nn, false));
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

int sqb_cholqr2_sharded_dev(sqb_context* ctx, const double* d_x, int64_t m_local, int64_t n,
                            int64_t ld, double* d_r) {
  SQB_TRY(enter(ctx));
  if (n < 1 || m_local < 0) return SQB_E_DIMENSION;
  if (n > kWideFusedMaxN || ld < m_local) return SQB_E_ARGUMENT;
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
