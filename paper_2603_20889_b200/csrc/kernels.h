// Internal launcher declarations shared between the kernel translation units and the C ABI.
#pragma once

#include <cuda_runtime.h>

#include "tsqr_warp.cuh"

namespace sqb {

// ---- tsqr_kernels.cu ---------------------------------------------------------------------
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
  int tune = 0;      // experiment switches (SQB_FOLD_TUNE), 0 in production
};
cudaError_t launch_tsqr_warp(const TsqrParams& prm, long long num_blocks, cudaStream_t stream);
int tsqr_warp_panel_rows(int n);
int tsqr_warp_warps(int n);

// ---- tsqr_thread_kernels.cu (n <= 16: every thread is a leaf of the reduction tree) --------
constexpr int kThreadTsqrMaxN = 16;
cudaError_t launch_tsqr_thread(const TsqrParams& prm, long long num_blocks, cudaStream_t stream);
int tsqr_thread_chunk_rows(int n);
int tsqr_thread_warps(int n);

// ---- tsqr_group_kernels.cu (8 < n <= 64: a group of G lanes is a leaf of the tree) ---------
cudaError_t launch_tsqr_group(const TsqrParams& prm, long long num_blocks, cudaStream_t stream);
int tsqr_group_chunk_rows(int n);
int tsqr_group_warps(int n);

// ---- tsqr_fold_kernels.cu (5 <= n <= 64: lookahead lane-group kernel with retire loads) -------
constexpr int kFoldTsqrMinN = 5;
cudaError_t launch_tsqr_fold(const TsqrParams& prm, long long num_blocks, cudaStream_t stream);
int tsqr_fold_chunk_rows(int n);
int tsqr_fold_warps(int n);

// ---- tsqr_mma_kernels.cu (blocked compact-WY Householder on the FP64 tensor cores) ----------
constexpr int kMmaTsqrMinN = 9;
cudaError_t launch_tsqr_mma(const TsqrParams& prm, long long num_blocks, cudaStream_t stream);
int tsqr_mma_panel_rows(int n);
int tsqr_mma_warps(int n);

// Kernel selection by column count (measured on B200, profiles/README.md): register-resident thread
// kernel up to 4 columns, lookahead fold kernel for 5..28, DMMA blocked kernel for 29..64.
// SQB_TSQR_KERNEL=0..4 forces thread / lane-group / warp-panel / fold / DMMA where the column count
// allows it (tuning, A/B tests and the kernel-family parity test only).
int tsqr_forced_kind();
inline int tsqr_kernel_kind(int n) {
  const int f = tsqr_forced_kind();
  if (f == 0 && n <= kThreadTsqrMaxN) return 0;
  if (f == 1 && n > 8) return 1;
  if (f == 2) return 2;
  if (f == 3 && n >= kFoldTsqrMinN) return 3;
  if (f == 4 && n >= kMmaTsqrMinN) return 4;
  if (f >= 0 && f <= 4) {  // forced kind not available for this n: fall back to the legacy table
    if (n <= 14) return 0;
    if (n <= 24) return 1;
    if (n <= 32) return 2;
    return 1;
  }
  if (n < kFoldTsqrMinN) return 0;
  if (n <= 28) return 3;
  return 4;
}
inline cudaError_t launch_tsqr_any(const TsqrParams& prm, long long num_blocks, cudaStream_t stream) {
  switch (tsqr_kernel_kind(prm.n)) {
    case 0: return launch_tsqr_thread(prm, num_blocks, stream);
    case 1: return launch_tsqr_group(prm, num_blocks, stream);
    case 3: return launch_tsqr_fold(prm, num_blocks, stream);
    case 4: return launch_tsqr_mma(prm, num_blocks, stream);
    default: return launch_tsqr_warp(prm, num_blocks, stream);
  }
}
inline int tsqr_panel_rows(int n) {
  switch (tsqr_kernel_kind(n)) {
    case 0: return tsqr_thread_chunk_rows(n);
    case 1: return tsqr_group_chunk_rows(n);
    case 3: return tsqr_fold_chunk_rows(n);
    case 4: return tsqr_mma_panel_rows(n);
    default: return tsqr_warp_panel_rows(n);
  }
}
inline int tsqr_warps(int n) {
  switch (tsqr_kernel_kind(n)) {
    case 0: return tsqr_thread_warps(n);
    case 1: return tsqr_group_warps(n);
    case 3: return tsqr_fold_warps(n);
    case 4: return tsqr_mma_warps(n);
    default: return tsqr_warp_warps(n);
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

// ---- gram_wide_kernels.cu (64 < n <= 256, plain Gram only: BASELINE config 5) -----------------
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

// ---- gram_thread_kernels.cu (n <= 8: register-resident rows and accumulators) --------------
constexpr int kThreadGramMaxN = 8;
cudaError_t launch_gram_thread(const GramParams& prm, int op, long long num_blocks,
                               cudaStream_t stream);
int gram_thread_chunk_rows(int n, int op);
int gram_thread_warps();
int gram_thread_ctas_per_sm(int n, int op);

// ---- small_kernels.cu (n x n work, one CTA each) -------------------------------------------
constexpr int kSmallMaxN = 128;
cudaError_t launch_cholesky(const double* c, int n, double* r, StatusWord* status,
                            cudaStream_t stream);
cudaError_t launch_eigh(const double* c, int n, double* values, double* vectors, double* scratch,
                        StatusWord* status, cudaStream_t stream);
// scratch: at least 4*n*n + 4*n doubles of device memory
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
