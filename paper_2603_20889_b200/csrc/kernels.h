// Internal launcher declarations shared between the kernel translation units and the C ABI.
#pragma once

#include <cuda_runtime.h>

#include "warp_pipe.cuh"

namespace sqb {

// ---- TSQR streaming kernels ------------------------------------------------------------------
struct TsqrParams {
  MatView x;
  long long m;
  int n;
  long long rows_per_block;
  double* y;         // block blk's triangle goes to rows [blk*n, blk*n+n), leading dim ldy
  long long ldy;
  int finalize;      // sign-normalise (reference sign_normalize, src/types.cpp:8-14)
  int check_finite;  // raise StatusWord::nonfinite when an Inf/NaN is streamed
  StatusWord* status;
  int kind = -1;     // kernel family (TsqrKind); -1 = the measured selection table
};

// ---- tsqr_thread_kernels.cu (n <= 16: every thread is a leaf of the reduction tree) --------
constexpr int kThreadTsqrMaxN = 16;
cudaError_t launch_tsqr_thread(const TsqrParams& prm, long long num_blocks, cudaStream_t stream);
int tsqr_thread_chunk_rows(int n);
int tsqr_thread_warps(int n);

// ---- tsqr_fold_kernels.cu (3 <= n <= 64: lookahead lane-group kernel with retire loads) -------
constexpr int kFoldTsqrMinN = 3;   // smallest column count the family is instantiated for
constexpr int kFoldTsqrAutoMinN = 3;  // ... and the smallest one the selection table gives it
cudaError_t launch_tsqr_fold(const TsqrParams& prm, long long num_blocks, cudaStream_t stream);
int tsqr_fold_chunk_rows(int n);
int tsqr_fold_warps(int n);

// ---- tsqr_mma_kernels.cu (blocked compact-WY Householder on the FP64 tensor cores) ----------
constexpr int kMmaTsqrMinN = 9;
cudaError_t launch_tsqr_mma(const TsqrParams& prm, long long num_blocks, cudaStream_t stream);
int tsqr_mma_panel_rows(int n);
int tsqr_mma_warps(int n);

// Kernel selection by column count (measured on B200, profiles/README.md): register-resident thread
// kernel up to 2 columns, lookahead fold kernel for 3..28, DMMA blocked kernel for 29..64.  A
// context may force one family where the column count allows it (sqb_set_tsqr_kernel: A/B timing
// and the kernel-family parity test); a family that cannot run this n falls back to the table.
enum TsqrKind { kTsqrAuto = -1, kTsqrThread = 0, kTsqrFold = 1, kTsqrMma = 2 };
inline int tsqr_kernel_kind(int n, int forced) {
  if (forced == kTsqrThread && n <= kThreadTsqrMaxN) return kTsqrThread;
  if (forced == kTsqrFold && n >= kFoldTsqrMinN) return kTsqrFold;
  if (forced == kTsqrMma && n >= kMmaTsqrMinN) return kTsqrMma;
  if (n < kFoldTsqrAutoMinN) return kTsqrThread;
  if (n <= 28) return kTsqrFold;
  return kTsqrMma;
}
inline cudaError_t launch_tsqr_any(const TsqrParams& prm, long long num_blocks, cudaStream_t stream) {
  switch (tsqr_kernel_kind(prm.n, prm.kind)) {
    case kTsqrThread: return launch_tsqr_thread(prm, num_blocks, stream);
    case kTsqrFold: return launch_tsqr_fold(prm, num_blocks, stream);
    default: return launch_tsqr_mma(prm, num_blocks, stream);
  }
}
inline int tsqr_panel_rows(int n, int forced) {
  switch (tsqr_kernel_kind(n, forced)) {
    case kTsqrThread: return tsqr_thread_chunk_rows(n);
    case kTsqrFold: return tsqr_fold_chunk_rows(n);
    default: return tsqr_mma_panel_rows(n);
  }
}
inline int tsqr_warps(int n, int forced) {
  switch (tsqr_kernel_kind(n, forced)) {
    case kTsqrThread: return tsqr_thread_warps(n);
    case kTsqrFold: return tsqr_fold_warps(n);
    default: return tsqr_mma_warps(n);
  }
}

// ---- gram_kernels.cu ---------------------------------------------------------------------
enum { OP_PLAIN = 0, OP_SOLVE = 1, OP_MULTIPLY = 2 };
struct GramParams {
  MatView x;
  long long m;
  int n;
  long long rows_per_block;
  const double* factor;  // n x n column-major: R (OP_SOLVE) or B (OP_MULTIPLY); null for OP_PLAIN
  double* partial;       // num_blocks x (n*n): each block's upper-triangle partial
  int check_finite;
  StatusWord* status;
};
cudaError_t launch_gram(const GramParams& prm, int op, long long num_blocks, cudaStream_t stream);
cudaError_t launch_gram_reduce(const double* partial, long long num_blocks, int n, double* c,
                               int check_finite, StatusWord* status, cudaStream_t stream);
int gram_panel_rows(int n, int op);
int gram_warps(int n);
int gram_ctas_per_sm(int n, int op);

// ---- gram_wide_kernels.cu (64 < n <= 256: BASELINE config 5) ----------------------------------
constexpr int kWideGramMaxN = 256;
size_t gram_wide_partial_doubles(int n, int sm_count);
cudaError_t launch_gram_wide(const MatView& x, long long m, int n, int sm_count, double* partial,
                             double* c, int check_finite, StatusWord* status, cudaStream_t stream);

// fused solve / multiply + Gram (the second CholQR2 / SVQB2 sweep) for 64 < n <= 128;
// frags: gram_wide_fused_scratch_doubles() doubles of device scratch
constexpr int kWideFusedMaxN = 128;
size_t gram_wide_fused_scratch_doubles();
cudaError_t launch_gram_wide_fused(const MatView& x, long long m, int n, int op, const double* factor,
                                   int sm_count, double* frags, double* partial, double* c, StatusWord* status,
                                   cudaStream_t stream);

cudaError_t launch_apply_rinv_wide(const double* x, long long m, int n, long long ld, const double* r,
                                   int sm_count, double* frags, double* q, long long ldq, StatusWord* status,
                                   cudaStream_t stream);

// the same for 128 < n <= 256 (BASELINE config 5): Q = X F formed per row slab (128 x 128 factor blocks,
// explicit R^-1), the wide SYRK on the slab.  scratch: gram_wide2_scratch_doubles(n); qslab: slab_rows x n
// (leading dimension slab_rows, even); c_tmp: n x n
size_t gram_wide2_scratch_doubles(int n);
cudaError_t launch_gram_wide2_fused(const MatView& x, long long m, int n, int op, const double* factor, int sm_count,
                                    double* scratch, double* qslab, long long slab_rows, double* partial,
                                    double* c_tmp, double* c, StatusWord* status, cudaStream_t stream,
                                    long long* launches);
cudaError_t launch_apply_rinv_wide2(const double* x, long long m, int n, long long ld, const double* r, int sm_count,
                                    double* scratch, double* q, long long ldq, StatusWord* status,
                                    cudaStream_t stream);

// ---- gram_thread_kernels.cu (n <= 12: register-resident rows and accumulators) -------------
constexpr int kThreadGramMaxN = 12;
// measured on B200 (profiles/README.md): the register-resident kernel wins the plain pass up to 10 columns,
// the fused multiply pass up to 11 and the fused solve pass up to 12; beyond, the DMMA kernel
inline bool gram_use_thread(int n, int op) { return n <= (op == OP_PLAIN ? 10 : (op == OP_MULTIPLY ? 11 : kThreadGramMaxN)); }
cudaError_t launch_gram_thread(const GramParams& prm, int op, long long num_blocks,
                               cudaStream_t stream);
int gram_thread_chunk_rows(int n, int op);
int gram_thread_warps();
int gram_thread_ctas_per_sm(int n, int op);

// ---- small_kernels.cu (n x n work, one CTA each) -------------------------------------------
constexpr int kSmallMaxN = 128;
// n <= 128: one CTA, matrix in shared memory; beyond: in place in global memory (any n)
cudaError_t launch_cholesky(const double* c, int n, double* r, StatusWord* status,
                            cudaStream_t stream);
// U = R^-1 (n x n column-major) for any n; scratch_rowmajor: n x n doubles
cudaError_t launch_rinv_global(const double* r, int n, double* scratch_rowmajor, double* u, StatusWord* status,
                               cudaStream_t stream);
// doubles of global scratch launch_eigh / launch_svqb_pass / the Cholesky kernels need at n columns
size_t small_scratch_doubles(int n);
cudaError_t launch_eigh(const double* c, int n, double* values, double* vectors, double* scratch,
                        StatusWord* status, cudaStream_t stream);
// scratch: at least 2*n doubles of device memory (the two diagonal scalings; A and U live in shared memory).
// want_sigma adds a second CTA that solves the unscaled Gram matrix for sigma beside the scaled solve.
cudaError_t launch_svqb_pass(const double* c, int n, double* b, double* z, double* sigma,
                             long long* rank, int want_sigma, double* scratch, StatusWord* status,
                             cudaStream_t stream);
cudaError_t launch_tri_multiply(const double* a, const double* b, int n, double* out,
                                cudaStream_t stream);
cudaError_t launch_small_multiply(const double* a, const double* b, int n, double* out,
                                  cudaStream_t stream);
// Householder QR of an n x n matrix, n <= 128 (reference hhqr_small in solve_lstsq's SVQB2 route, lstsq.cpp:37-39)
cudaError_t launch_hhqr_small(const double* z, int n, double* r, cudaStream_t stream);
cudaError_t launch_backsolve(const double* r, int ne, double* xsol, double* residual,
                             StatusWord* status, cudaStream_t stream);
cudaError_t launch_check_finite(const double* a, long long count, StatusWord* status,
                                cudaStream_t stream);
// Q = X R^-1 (reference reconstruct_q, src/gram_qr.cpp:193-221)
cudaError_t launch_apply_rinv(const double* x, long long m, int n, long long ld, const double* r,
                              double* q, long long ldq, StatusWord* status, cudaStream_t stream);

// ---- matgen_kernels.cu -----------------------------------------------------------------------
cudaError_t launch_fill_gaussian(double* x, long long m, int n, long long ld, unsigned long long seed,
                                 long long row_offset, long long m_total, cudaStream_t stream);
cudaError_t launch_generate(double* x, long long m, int n, long long ld, double kappa,
                            int linear_decay, unsigned long long seed, double* scratch,
                            cudaStream_t stream);
size_t generate_scratch_doubles(long long m, int n);

}  // namespace sqb
