/*
 * skinnyqr_b200 -- C ABI of the B200-native Q-less tall-skinny QR library.
 *
 * This is the drop-in boundary.  Each entry point names the reference interface it replaces
 * (paths relative to the reference's proj/ directory).  Everything is FP64, column-major:
 * element (i,j) of an m x n matrix with leading dimension ld lives at x[j*ld + i]
 * (reference: include/skinnyqr/types.hpp:79-94).
 *
 * Two families:
 *   *_dev   X (and outputs) are DEVICE pointers; the call is enqueued on the context's stream
 *           and returns without synchronising.  Numerical failures are recorded in the
 *           context's device status word and reported by sqb_sync().
 *   *_host  X and outputs are HOST pointers; the call streams X to the device in slabs
 *           (copy/compute overlapped), synchronises and returns the final status.  These are
 *           what the C++ entry points in paper_2603_20889_b200/include/skinnyqr bind to.
 *
 * Status codes mirror the reference's exception classes (include/skinnyqr/types.hpp:11-77).
 * There is no CPU fallback anywhere behind this ABI: without a CUDA device every call fails
 * with SQB_E_CUDA.
 */
#ifndef SKINNYQR_B200_H_
#define SKINNYQR_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SQB_OK = 0,
  SQB_E_DIMENSION = -1,      /* skinnyqr::DimensionError                                  */
  SQB_E_ARGUMENT = -2,       /* skinnyqr::ArgumentError (non-finite input, n > 64, ...)    */
  SQB_E_BREAKDOWN = -3,      /* skinnyqr::BreakdownError      + pivot index                */
  SQB_E_SINGULAR = -4,       /* skinnyqr::SingularFactorError + diagonal index             */
  SQB_E_ZERO_MATRIX = -5,    /* skinnyqr::ZeroMatrixError                                  */
  SQB_E_RANK_DEFICIENT = -6, /* skinnyqr::RankDeficiencyError + diagonal index             */
  SQB_E_NO_CONVERGENCE = -7, /* skinnyqr::Error from eigh_small (30 sweeps)                */
  SQB_E_CUDA = -8,           /* CUDA runtime failure / no device                           */
  SQB_E_NCCL = -9            /* communicator failure                                       */
};

enum { SQB_METHOD_TSQR = 0, SQB_METHOD_CHOLQR2 = 1, SQB_METHOD_SVQB2 = 2 };

typedef struct sqb_context sqb_context;

/* ---- context ------------------------------------------------------------------------- */
/* Creates a context on `device` with its own stream, workspace (stacked triangles / partial
 * Grams, n x n scratch) and status word.  The reference has no such object: its workspaces
 * are allocated per call (src/tsqr.cpp:142, src/gram.cpp:44-47).                           */
int sqb_create(sqb_context** ctx, int device);
int sqb_destroy(sqb_context* ctx);
/* Use a caller-owned cudaStream_t instead of the context's own (NULL = the CUDA default
 * stream); sqb_use_own_stream switches back.                                               */
int sqb_set_stream(sqb_context* ctx, void* cuda_stream);
int sqb_use_own_stream(sqb_context* ctx);
void* sqb_get_stream(sqb_context* ctx);
/* Synchronise the stream and return the first error recorded since the last sync (0 = ok). */
int sqb_sync(sqb_context* ctx);
/* Index attached to the last BREAKDOWN / SINGULAR / RANK_DEFICIENT status.                  */
long long sqb_last_error_index(const sqb_context* ctx);
const char* sqb_status_string(int status);
/* Device facts the default plans are derived from.                                         */
int sqb_device_sm_count(const sqb_context* ctx);
/* Number of kernels launched through this context since creation (bench bookkeeping).      */
long long sqb_launch_count(const sqb_context* ctx);

/* Test / tuning hook: force one TSQR kernel family for this context (0 = thread-private leaves,
 * 1 = lookahead fold, 2 = FP64 tensor-core blocked kernel, -1 = the measured selection table).
 * A family that cannot run a given column count falls back to the table.                     */
int sqb_set_tsqr_kernel(sqb_context* ctx, int kind);
/* Slab size (bytes, >= 1 MiB) of the host-pointer entry points: single-pass calls stream X
 * through a three-slab ring, so device memory stays O(slab) however large m*n is (the reference
 * keeps O((b+n)*n) state, src/tsqr.cpp:143-147).                                              */
int sqb_set_host_slab_bytes(sqb_context* ctx, int64_t bytes);
/* Stream-ordered copies between host memory and device buffers of this context's device; both
 * synchronise the stream before returning (used by caller-supplied exchanges, below).         */
int sqb_copy_h2d(sqb_context* ctx, void* d_dst, const void* h_src, int64_t bytes);
int sqb_copy_d2h(sqb_context* ctx, void* h_dst, const void* d_src, int64_t bytes);
/* Device memory on the context's device, for host code that owns device-resident matrices without
 * including CUDA headers (the C++ mirror's DeviceMatrix, paper_2603_20889_b200/include/skinnyqr/device.hpp). */
int sqb_device_alloc(sqb_context* ctx, int64_t bytes, void** d_ptr);
int sqb_device_free(sqb_context* ctx, void* d_ptr);

/* ---- plans (replaces default_tsqr_plan / default_gram_plan, src/plan.cpp:9-32) ---------- */
/* num_blocks = CTAs of the streaming kernel (reference: worker threads), panel_rows = rows
 * one warp stages per TMA transaction group (reference: cache-resident panel height).       */
int sqb_default_tsqr_plan(const sqb_context* ctx, int64_t m, int64_t n, int64_t* num_blocks,
                          int64_t* panel_rows);
int sqb_default_gram_plan(const sqb_context* ctx, int64_t m, int64_t n, int64_t* num_blocks,
                          int64_t* panel_rows);

/* ---- Q-less Householder TSQR ---------------------------------------------------------- */
/* Replaces tsqr_qless (include/skinnyqr/tsqr.hpp:65, src/tsqr.cpp:186-197).  d_r receives the
 * n x n upper triangle (full square, exact zeros below the diagonal, diagonal >= 0).
 * num_blocks / panel_rows = 0 select the default plan.  n <= 64.                           */
int sqb_tsqr_qless_dev(sqb_context* ctx, const double* d_x, int64_t m, int64_t n, int64_t ld,
                       int64_t num_blocks, int64_t panel_rows, double* d_r);
/* Replaces tsqr_stage1 (tsqr.hpp:68, tsqr.cpp:168-184): d_y is (num_blocks*n) x n, block i's
 * un-normalised triangle at rows [i*n, i*n+n); row partition = PanelPlan::block_begin/end
 * (include/skinnyqr/plan.hpp:24-37).                                                       */
int sqb_tsqr_stage1_dev(sqb_context* ctx, const double* d_x, int64_t m, int64_t n, int64_t ld,
                        int64_t num_blocks, int64_t panel_rows, double* d_y);
/* Replaces block_qless_qr (tsqr.hpp:59, tsqr.cpp:162-166): one block, no sign normalisation. */
int sqb_block_qless_qr_dev(sqb_context* ctx, const double* d_x, int64_t m, int64_t n,
                           int64_t ld, int64_t panel_rows, double* d_r);

/* ---- Gram kernels (include/skinnyqr/gram.hpp:12-21, src/gram.cpp:113-151) ----------------- */
/* C = X^T X (tsmttsm); n <= 256: the reference has no column limit here, 65..256 columns run
 * the wide FP64 tensor-core kernel and ignore num_blocks / panel_rows (BASELINE config 5)   */
int sqb_tsmttsm_dev(sqb_context* ctx, const double* d_x, int64_t m, int64_t n, int64_t ld,
                    int64_t num_blocks, int64_t panel_rows, double* d_c);
/* C = (X R^-1)^T (X R^-1), R upper triangular n x n on device (tsmRttsmR); n <= 128: the
 * reference has no column limit; 65..128 columns run the wide fused kernel (explicit R^-1 as a
 * tensor-core GEMM feeding the SYRK) and ignore num_blocks / panel_rows                       */
int sqb_tsmRttsmR_dev(sqb_context* ctx, const double* d_x, int64_t m, int64_t n, int64_t ld,
                      const double* d_r, int64_t num_blocks, int64_t panel_rows, double* d_c);
/* C = (X B)^T (X B), B dense n x n on device (tsmmttsmm); n <= 128, as above               */
int sqb_tsmmttsmm_dev(sqb_context* ctx, const double* d_x, int64_t m, int64_t n, int64_t ld,
                      const double* d_b, int64_t num_blocks, int64_t panel_rows, double* d_c);

/* ---- n x n factorisations on device (include/skinnyqr/gram_qr.hpp:37-41) ------------------ */
int sqb_cholesky_dev(sqb_context* ctx, const double* d_c, int64_t n, double* d_r);
int sqb_eigh_small_dev(sqb_context* ctx, const double* d_c, int64_t n, double* d_values,
                       double* d_vectors);

/* ---- Gram-based drivers (gram_qr.hpp:46-59, src/gram_qr.cpp:123-221) ----------------------- */
/* cholqr2: two streaming passes, both Cholesky factorisations and R2*R1 stay on the device.
 * n <= 128 (the reference has no column limit; 65..128 columns take the wide kernels).       */
int sqb_cholqr2_dev(sqb_context* ctx, const double* d_x, int64_t m, int64_t n, int64_t ld,
                    int64_t num_blocks, int64_t panel_rows, double* d_r);
/* svqb2: d_transform (B), d_z are n x n, d_sigma has n entries, d_rank one int64.
 * n <= 128 = the reference's own limit (eigh_small, gram_qr.cpp:62).                         */
int sqb_svqb2_dev(sqb_context* ctx, const double* d_x, int64_t m, int64_t n, int64_t ld,
                  int64_t num_blocks, int64_t panel_rows, double* d_transform, double* d_z,
                  double* d_sigma, int64_t* d_rank);
/* One SVQB pass on a device Gram matrix (svqb_pass, gram_qr.cpp:133-176).                    */
int sqb_svqb_pass_dev(sqb_context* ctx, const double* d_c, int64_t n, double* d_b, double* d_z,
                      double* d_sigma, int64_t* d_rank);
/* Q = X R^-1 written to d_q (ldq) (reconstruct_q, gram_qr.cpp:193-221); n <= 128.           */
int sqb_reconstruct_q_dev(sqb_context* ctx, const double* d_x, int64_t m, int64_t n, int64_t ld,
                          const double* d_r, double* d_q, int64_t ldq);

/* ---- least squares (include/skinnyqr/lstsq.hpp:21, src/lstsq.cpp:13-61) -------------------- */
/* A (m x n, lda) and rhs (m) stay separate device arrays: column n of the [A rhs] pencil is
 * read straight from d_rhs, so the reference's m*(n+1) assembly copy (lstsq.cpp:24-26) never
 * happens.  d_xsol gets n entries, d_residual one.  n + 1 <= 64 on the TSQR route (tsqr.cpp:188),
 * n + 1 <= 128 on the CholQR2 / SVQB2 routes.                                                 */
int sqb_solve_lstsq_dev(sqb_context* ctx, const double* d_a, int64_t m, int64_t n, int64_t lda,
                        const double* d_rhs, int method, double* d_xsol, double* d_residual);

/* ---- host-pointer entry points (what the C++ API binds to) --------------------------------- */
int sqb_tsqr_qless_host(sqb_context* ctx, const double* x, int64_t m, int64_t n, int64_t ld,
                        int64_t num_blocks, int64_t panel_rows, double* r);
int sqb_tsqr_stage1_host(sqb_context* ctx, const double* x, int64_t m, int64_t n, int64_t ld,
                         int64_t num_blocks, int64_t panel_rows, double* y);
int sqb_block_qless_qr_host(sqb_context* ctx, const double* x, int64_t m, int64_t n, int64_t ld,
                            int64_t panel_rows, double* r);
int sqb_tsmttsm_host(sqb_context* ctx, const double* x, int64_t m, int64_t n, int64_t ld,
                     int64_t num_blocks, int64_t panel_rows, double* c);
int sqb_tsmRttsmR_host(sqb_context* ctx, const double* x, int64_t m, int64_t n, int64_t ld,
                       const double* r, int64_t num_blocks, int64_t panel_rows, double* c);
int sqb_tsmmttsmm_host(sqb_context* ctx, const double* x, int64_t m, int64_t n, int64_t ld,
                       const double* b, int64_t num_blocks, int64_t panel_rows, double* c);
int sqb_cholesky_host(sqb_context* ctx, const double* c, int64_t n, double* r);
int sqb_eigh_small_host(sqb_context* ctx, const double* c, int64_t n, double* values,
                        double* vectors);
int sqb_cholqr2_host(sqb_context* ctx, const double* x, int64_t m, int64_t n, int64_t ld,
                     int64_t num_blocks, int64_t panel_rows, double* r);
int sqb_svqb_pass_host(sqb_context* ctx, const double* c, int64_t n, double* b, double* z,
                       double* sigma, int64_t* rank);
int sqb_svqb2_host(sqb_context* ctx, const double* x, int64_t m, int64_t n, int64_t ld,
                   int64_t num_blocks, int64_t panel_rows, double* transform, double* z,
                   double* sigma, int64_t* rank);
int sqb_reconstruct_q_host(sqb_context* ctx, const double* x, int64_t m, int64_t n, int64_t ld,
                           const double* r, double* q, int64_t ldq);
int sqb_solve_lstsq_host(sqb_context* ctx, const double* a, int64_t m, int64_t n, int64_t lda,
                         const double* rhs, int method, double* xsol, double* residual);

/* ---- synthetic inputs on device (harness; reference: src/matgen.cpp:8-109) ------------------ */
/* Gaussian: element e = j*m + i draws u1 = uniform01(seed, 2e), u2 = uniform01(seed, 2e+1)
 * and x = sqrt(-2 ln max(u1, 2^-53)) cos(2 pi u2); `row_offset` shifts i so that row slabs of
 * one logical matrix can be generated independently (m_total is the logical row count).      */
int sqb_fill_gaussian_dev(sqb_context* ctx, double* d_x, int64_t m, int64_t n, int64_t ld,
                          uint64_t seed, int64_t row_offset, int64_t m_total);
/* Controlled-spectrum matrix X = U diag(sigma) V^T (generate, matgen.cpp:77-109).            */
int sqb_generate_dev(sqb_context* ctx, double* d_x, int64_t m, int64_t n, int64_t ld,
                     double kappa, int linear_decay, uint64_t seed);

/* ---- multi-GPU (one process per GPU; rows sharded, only n x n data crosses NVLink) ----------
 * The protocol is the reference's own block structure one level up: rank g plays the part of
 * block g.  TSQR: every rank reduces its slab to an n x n triangle, the triangles are all-gathered
 * and every rank runs stage 2 over the (world*n) x n stack (src/tsqr.cpp:175-195 with k = world).
 * Gram methods: every rank forms its partial n x n Gram, the partials are all-gathered and summed
 * in ascending rank order (src/gram.cpp:81-92), so all ranks hold bit-identical matrices.  The
 * exchange is NCCL (sqb_init_nccl / sqb_attach_nccl) or any caller-supplied all-gather
 * (sqb_set_allgather: MPI, torch.distributed, a test harness) - the same driver code runs over
 * either.  The two halves are also exported on their own (sqb_tsqr_local_dev + sqb_*_combine_dev).   */
/* All-gather of `count` doubles per rank: d_send (this rank's block) -> d_recv (world blocks in
 * rank order), both device pointers on the context's device.  It is called between kernel
 * launches on the context's stream (sqb_get_stream); d_send is ready in stream order and d_recv
 * must be valid for work enqueued on that stream afterwards.  Return 0 on success.               */
typedef int (*sqb_allgather_fn)(void* user, const double* d_send, double* d_recv, int64_t count);
int sqb_set_allgather(sqb_context* ctx, sqb_allgather_fn fn, void* user, int rank, int world);
/* This rank's triangle: Q-less TSQR of its slab WITHOUT sign normalisation (block_qless_qr of
 * block `rank`, src/tsqr.cpp:178-181); m_local may be smaller than n or zero (zero triangle).    */
int sqb_tsqr_local_dev(sqb_context* ctx, const double* d_x, int64_t m_local, int64_t n, int64_t ld,
                       double* d_r_local);
/* Stage 2 over `world` gathered triangles (d_gathered: world blocks of n x n, leading dimension
 * n): stack, fold, sign-normalise (src/tsqr.cpp:193-195, src/types.cpp:8-14).                     */
int sqb_tsqr_combine_dev(sqb_context* ctx, const double* d_gathered, int64_t world, int64_t n,
                         double* d_r);
/* Sum of `world` gathered n x n Gram partials in ascending rank order (src/gram.cpp:81-92).      */
int sqb_gram_combine_dev(sqb_context* ctx, const double* d_gathered, int64_t world, int64_t n,
                         double* d_c);
/* Attach an ncclComm_t created by the caller (e.g. from torch.distributed's unique id).      */
int sqb_attach_nccl(sqb_context* ctx, void* nccl_comm, int rank, int world);
/* Create a communicator from a 128-byte ncclUniqueId (all ranks call collectively).          */
int sqb_nccl_unique_id(void* out128);
int sqb_init_nccl(sqb_context* ctx, const void* unique_id128, int rank, int world);
/* Row-sharded variants: d_x is this rank's slab (m_local rows).  Every rank ends with the
 * same R.  TSQR: all-gather of the per-rank triangles + redundant final combine;
 * CholQR2/SVQB2: all-reduce of each n x n Gram.                                              */
int sqb_tsqr_qless_sharded_dev(sqb_context* ctx, const double* d_x, int64_t m_local, int64_t n,
                               int64_t ld, double* d_r);
/* Host-pointer form: this rank's slab lives in host memory and streams through the slab ring.  */
int sqb_tsqr_qless_sharded_host(sqb_context* ctx, const double* x, int64_t m_local, int64_t n,
                                int64_t ld, double* r);
int sqb_cholqr2_sharded_dev(sqb_context* ctx, const double* d_x, int64_t m_local, int64_t n,
                            int64_t ld, double* d_r);
int sqb_svqb2_sharded_dev(sqb_context* ctx, const double* d_x, int64_t m_local, int64_t n,
                          int64_t ld, double* d_transform, double* d_z, double* d_sigma,
                          int64_t* d_rank);
int sqb_solve_lstsq_sharded_dev(sqb_context* ctx, const double* d_a, int64_t m_local, int64_t n,
                                int64_t lda, const double* d_rhs, double* d_xsol,
                                double* d_residual);

#ifdef __cplusplus
}
#endif

#endif /* SKINNYQR_B200_H_ */
