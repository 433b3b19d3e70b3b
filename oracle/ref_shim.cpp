// TEST INFRASTRUCTURE ONLY -- not part of the shipped product.
//
// C-ABI shim around the UNMODIFIED reference sources under
// /root/reference/proj (namespace skinnyqr). The Makefile in this directory
// compiles those sources where they lie and links them with this file into
// oracle/_ref/libskinnyqr_ref.so.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load that library.
//
// Every entry point returns 0 on success or a negative status mirroring the
// reference's exception type (see REF_E_* below); index-carrying exceptions
// report the index through *err_index.  All matrices are column-major FP64.
//
// Timing: the *_timed entry points take a matrix handle (a DenseMatrix built
// outside the timed region) and return the wall time of the reference call
// alone, measured with steady_clock, as SURVEY.md section 8(d) prescribes.

#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "skinnyqr/counters.hpp"
#include "skinnyqr/gram.hpp"
#include "skinnyqr/gram_qr.hpp"
#include "skinnyqr/kernels.hpp"
#include "skinnyqr/lstsq.hpp"
#include "skinnyqr/matgen.hpp"
#include "skinnyqr/parallel.hpp"
#include "skinnyqr/plan.hpp"
#include "skinnyqr/small.hpp"
#include "skinnyqr/tsqr.hpp"
#include "skinnyqr/types.hpp"

namespace sq = skinnyqr;

enum {
  REF_OK = 0,
  REF_E_DIMENSION = -1,
  REF_E_ARGUMENT = -2,
  REF_E_BREAKDOWN = -3,
  REF_E_SINGULAR = -4,
  REF_E_ZERO_MATRIX = -5,
  REF_E_RANK_DEFICIENT = -6,
  REF_E_OTHER = -7,
};

namespace {

thread_local std::string g_last_message;

template <class Fn>
int guarded(long long* err_index, Fn&& fn) {
  if (err_index) *err_index = -1;
  try {
    fn();
    return REF_OK;
  } catch (const sq::BreakdownError& e) {
    if (err_index) *err_index = static_cast<long long>(e.pivot_index);
    g_last_message = e.what();
    return REF_E_BREAKDOWN;
  } catch (const sq::SingularFactorError& e) {
    if (err_index) *err_index = static_cast<long long>(e.diagonal_index);
    g_last_message = e.what();
    return REF_E_SINGULAR;
  } catch (const sq::RankDeficiencyError& e) {
    if (err_index) *err_index = static_cast<long long>(e.diagonal_index);
    g_last_message = e.what();
    return REF_E_RANK_DEFICIENT;
  } catch (const sq::ZeroMatrixError& e) {
    g_last_message = e.what();
    return REF_E_ZERO_MATRIX;
  } catch (const sq::DimensionError& e) {
    g_last_message = e.what();
    return REF_E_DIMENSION;
  } catch (const sq::ArgumentError& e) {
    g_last_message = e.what();
    return REF_E_ARGUMENT;
  } catch (const std::exception& e) {
    g_last_message = e.what();
    return REF_E_OTHER;
  }
}

sq::DenseMatrix dense_from(const double* x, long long m, long long n) {
  sq::DenseMatrix d(static_cast<std::size_t>(m), static_cast<std::size_t>(n));
  if (m * n > 0) std::memcpy(d.data(), x, sizeof(double) * m * n);
  return d;
}

sq::PanelPlan plan_from(long long k, long long b, bool tsqr, std::size_t m, std::size_t n) {
  sq::PanelPlan p = tsqr ? sq::default_tsqr_plan(m, n) : sq::default_gram_plan(m, n);
  if (k > 0) p.num_blocks = static_cast<std::size_t>(k);
  if (b > 0) p.panel_rows = static_cast<std::size_t>(b);
  return p;
}

template <class Square>
void square_out(const Square& s, std::size_t n, double* out) {
  std::memcpy(out, s.data(), sizeof(double) * n * n);
}

sq::UpperTriangular upper_from(const double* r, long long n) {
  sq::UpperTriangular u(static_cast<std::size_t>(n));
  std::memcpy(u.data(), r, sizeof(double) * n * n);
  return u;
}

sq::GramMatrix gram_from(const double* c, long long n) {
  sq::GramMatrix g(static_cast<std::size_t>(n));
  std::memcpy(g.data(), c, sizeof(double) * n * n);
  return g;
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

extern "C" {

const char* ref_last_message() { return g_last_message.c_str(); }
const char* ref_kernel_table_name() { return sq::kernels::active().name; }
long long ref_max_threads() { return static_cast<long long>(sq::max_threads()); }
void ref_set_max_threads(long long n) { sq::set_max_threads(static_cast<std::size_t>(n)); }

// 0 = scalar, 1 = avx2 (if available). Returns 0 on success.
int ref_select_kernel_table(int which) {
  if (which == 0) {
    sq::kernels::set_active(sq::kernels::scalar_table());
    return 0;
  }
  if (const sq::kernels::KernelTable* t = sq::kernels::avx2_table()) {
    sq::kernels::set_active(*t);
    return 0;
  }
  return -1;
}

void ref_counters_reset() { sq::counters().reset(); }
void ref_counters_read(unsigned long long out[4]) {
  const sq::CounterSnapshot s = sq::counters().snapshot();
  out[0] = s.large_reads;
  out[1] = s.large_writes;
  out[2] = s.flops;
  out[3] = s.flops_actual;
}

// ---- plans ---------------------------------------------------------------
int ref_default_tsqr_plan(long long m, long long n, long long* k, long long* b) {
  return guarded(nullptr, [&] {
    const sq::PanelPlan p = sq::default_tsqr_plan(m, n);
    *k = static_cast<long long>(p.num_blocks);
    *b = static_cast<long long>(p.panel_rows);
  });
}
int ref_default_gram_plan(long long m, long long n, long long* k, long long* b) {
  return guarded(nullptr, [&] {
    const sq::PanelPlan p = sq::default_gram_plan(m, n);
    *k = static_cast<long long>(p.num_blocks);
    *b = static_cast<long long>(p.panel_rows);
  });
}
void ref_plan_block_range(long long m, long long k, long long b, long long block,
                          long long* begin, long long* end) {
  sq::PanelPlan p;
  p.num_blocks = static_cast<std::size_t>(k);
  p.panel_rows = static_cast<std::size_t>(b);
  *begin = static_cast<long long>(p.block_begin(m, block));
  *end = static_cast<long long>(p.block_end(m, block));
}

// ---- generator -------------------------------------------------------------
unsigned long long ref_mix64(unsigned long long seed, unsigned long long index) {
  return sq::mix64(seed, index);
}
double ref_uniform01(unsigned long long seed, unsigned long long index) {
  return sq::uniform01(seed, index);
}
int ref_generate(long long m, long long n, double kappa, int linear_decay,
                 unsigned long long seed, double* out) {
  return guarded(nullptr, [&] {
    sq::SpectrumSpec spec;
    spec.kappa = kappa;
    spec.decay = linear_decay ? sq::SpectrumDecay::linear : sq::SpectrumDecay::geometric;
    spec.seed = seed;
    const sq::DenseMatrix x = sq::generate(m, n, spec);
    std::memcpy(out, x.data(), sizeof(double) * m * n);
  });
}

// ---- TSQR ------------------------------------------------------------------
int ref_tsqr_qless(const double* x, long long m, long long n, long long k, long long b,
                   double* r_out) {
  return guarded(nullptr, [&] {
    const sq::DenseMatrix d = dense_from(x, m, n);
    const sq::UpperTriangular r = sq::tsqr_qless(d, plan_from(k, b, true, m, n));
    square_out(r, n, r_out);
  });
}
int ref_tsqr_stage1(const double* x, long long m, long long n, long long k, long long b,
                    double* y_out /* (k*n) x n */) {
  return guarded(nullptr, [&] {
    const sq::DenseMatrix d = dense_from(x, m, n);
    const sq::PanelPlan p = plan_from(k, b, true, m, n);
    const sq::DenseMatrix y = sq::tsqr_stage1(d, p);
    std::memcpy(y_out, y.data(), sizeof(double) * y.rows() * y.cols());
  });
}
int ref_block_qless_qr(const double* x, long long m, long long n, long long b, double* r_out) {
  return guarded(nullptr, [&] {
    const sq::DenseMatrix d = dense_from(x, m, n);
    const sq::UpperTriangular r = sq::block_qless_qr(d, static_cast<std::size_t>(b));
    square_out(r, n, r_out);
  });
}
int ref_reference_hhqr(const double* x, long long m, long long n, double* r_out) {
  return guarded(nullptr, [&] {
    const sq::DenseMatrix d = dense_from(x, m, n);
    const sq::UpperTriangular r = sq::reference_hhqr(d);
    square_out(r, n, r_out);
  });
}
// One pencil step on a fresh workspace (zero running triangle): loads the
// p x n panel w (ld = p) and factors it; returns the whole (b+n) x n pencil.
int ref_factor_trapezoidal(const double* w, long long p, long long n, long long b,
                           double* pencil_out) {
  return guarded(nullptr, [&] {
    sq::TrapezoidalWorkspace ws(static_cast<std::size_t>(b), static_cast<std::size_t>(n));
    ws.load_panel(w, static_cast<std::size_t>(p), static_cast<std::size_t>(p));
    sq::factor_trapezoidal(ws);
    for (long long j = 0; j < n; ++j)
      for (long long i = 0; i < b + n; ++i) pencil_out[j * (b + n) + i] = ws.at(i, j);
  });
}

// ---- Gram kernels ----------------------------------------------------------
int ref_tsmttsm(const double* x, long long m, long long n, long long k, long long b,
                int deterministic, double* c_out) {
  return guarded(nullptr, [&] {
    const sq::DenseMatrix d = dense_from(x, m, n);
    sq::PanelPlan p = plan_from(k, b, false, m, n);
    p.deterministic = deterministic != 0;
    square_out(sq::tsmttsm(d, p), n, c_out);
  });
}
int ref_tsmRttsmR(const double* x, long long m, long long n, const double* r, long long k,
                  long long b, double* c_out, long long* err_index) {
  return guarded(err_index, [&] {
    const sq::DenseMatrix d = dense_from(x, m, n);
    square_out(sq::tsmRttsmR(d, upper_from(r, n), plan_from(k, b, false, m, n)), n, c_out);
  });
}
int ref_tsmmttsmm(const double* x, long long m, long long n, const double* bmat, long long k,
                  long long b, double* c_out) {
  return guarded(nullptr, [&] {
    const sq::DenseMatrix d = dense_from(x, m, n);
    const sq::DenseMatrix bm = dense_from(bmat, n, n);
    square_out(sq::tsmmttsmm(d, bm, plan_from(k, b, false, m, n)), n, c_out);
  });
}

// ---- n x n factorizations ----------------------------------------------------
int ref_cholesky(const double* c, long long n, double* r_out, long long* err_index) {
  return guarded(err_index, [&] { square_out(sq::cholesky(gram_from(c, n)), n, r_out); });
}
int ref_eigh_small(const double* c, long long n, double* values, double* vectors) {
  return guarded(nullptr, [&] {
    const sq::EigenDecomp e = sq::eigh_small(gram_from(c, n));
    std::memcpy(values, e.values.data(), sizeof(double) * n);
    std::memcpy(vectors, e.vectors.data(), sizeof(double) * n * n);
  });
}
int ref_triangular_multiply(const double* a, const double* b, long long n, double* out) {
  return guarded(nullptr, [&] {
    square_out(sq::triangular_multiply(upper_from(a, n), upper_from(b, n)), n, out);
  });
}
int ref_hhqr_small(const double* a, long long m, long long n, double* r_out) {
  return guarded(nullptr, [&] { square_out(sq::hhqr_small(dense_from(a, m, n)), n, r_out); });
}

// ---- Gram-based drivers ----------------------------------------------------
int ref_cholqr2(const double* x, long long m, long long n, long long k, long long b,
                double* r_out, long long* err_index) {
  return guarded(err_index, [&] {
    const sq::DenseMatrix d = dense_from(x, m, n);
    square_out(sq::cholqr2(d, plan_from(k, b, false, m, n)), n, r_out);
  });
}
int ref_svqb_pass(const double* c, long long n, double* b_out, double* z_out, double* sigma,
                  long long* rank) {
  return guarded(nullptr, [&] {
    // svqb_pass only inspects x.cols(); hand it an n x n placeholder.
    const sq::DenseMatrix x(static_cast<std::size_t>(n), static_cast<std::size_t>(n));
    const sq::SvqbPassResult p = sq::svqb_pass(x, gram_from(c, n));
    std::memcpy(b_out, p.b.data(), sizeof(double) * n * n);
    std::memcpy(z_out, p.z.data(), sizeof(double) * n * n);
    std::memcpy(sigma, p.sigma.data(), sizeof(double) * n);
    *rank = static_cast<long long>(p.rank);
  });
}
int ref_svqb2(const double* x, long long m, long long n, long long k, long long b,
              double* transform, double* z, double* sigma, long long* rank) {
  return guarded(nullptr, [&] {
    const sq::DenseMatrix d = dense_from(x, m, n);
    const sq::QzResult q = sq::svqb2(d, plan_from(k, b, false, m, n));
    std::memcpy(transform, q.transform.data(), sizeof(double) * n * n);
    std::memcpy(z, q.z.data(), sizeof(double) * n * n);
    std::memcpy(sigma, q.singular_values.data(), sizeof(double) * n);
    *rank = static_cast<long long>(q.rank);
  });
}
int ref_reconstruct_q(const double* x, long long m, long long n, const double* r, double* q_out,
                      long long* err_index) {
  return guarded(err_index, [&] {
    const sq::DenseMatrix d = dense_from(x, m, n);
    const sq::DenseMatrix q = sq::reconstruct_q(d, upper_from(r, n));
    std::memcpy(q_out, q.data(), sizeof(double) * m * n);
  });
}

// ---- least squares ---------------------------------------------------------
int ref_solve_lstsq(const double* a, long long m, long long n, const double* rhs, int method,
                    double* x_out, double* residual, long long* err_index) {
  return guarded(err_index, [&] {
    const sq::DenseMatrix d = dense_from(a, m, n);
    const std::vector<double> b(rhs, rhs + m);
    const sq::LstsqResult res =
        sq::solve_lstsq(d, b, static_cast<sq::LstsqMethod>(method));
    std::memcpy(x_out, res.x.data(), sizeof(double) * n);
    *residual = res.residual_norm;
  });
}

// ---- timed handles (CPU baseline) ---------------------------------------------
void* ref_matrix_create(const double* x, long long m, long long n) {
  return new sq::DenseMatrix(dense_from(x, m, n));
}
void* ref_matrix_create_uninit(long long m, long long n) {
  return new sq::DenseMatrix(static_cast<std::size_t>(m), static_cast<std::size_t>(n));
}
double* ref_matrix_data(void* h) { return static_cast<sq::DenseMatrix*>(h)->data(); }
void ref_matrix_destroy(void* h) { delete static_cast<sq::DenseMatrix*>(h); }

// method: 0 tsqr_qless, 1 cholqr2, 2 svqb2, 3 tsqr_stage1 + stage-2 block QR (no validation
// scan), 4 reference_hhqr, 5 tsmttsm.  r_out may be null.  Returns status; *seconds = wall
// time of the reference call alone.
int ref_timed_factor(void* h, int method, long long k, long long b, double* r_out,
                     double* seconds) {
  const sq::DenseMatrix& x = *static_cast<sq::DenseMatrix*>(h);
  const std::size_t m = x.rows(), n = x.cols();
  return guarded(nullptr, [&] {
    const auto t0 = std::chrono::steady_clock::now();
    switch (method) {
      case 0: {
        const sq::UpperTriangular r = sq::tsqr_qless(x, plan_from(k, b, true, m, n));
        *seconds = seconds_since(t0);
        if (r_out) square_out(r, n, r_out);
        break;
      }
      case 1: {
        const sq::UpperTriangular r = sq::cholqr2(x, plan_from(k, b, false, m, n));
        *seconds = seconds_since(t0);
        if (r_out) square_out(r, n, r_out);
        break;
      }
      case 2: {
        const sq::QzResult q = sq::svqb2(x, plan_from(k, b, false, m, n));
        *seconds = seconds_since(t0);
        if (r_out) std::memcpy(r_out, q.z.data(), sizeof(double) * n * n);
        break;
      }
      case 3: {
        const sq::PanelPlan p = plan_from(k, b, true, m, n);
        const sq::DenseMatrix y = sq::tsqr_stage1(x, p);
        sq::UpperTriangular r = sq::block_qless_qr(y, p.panel_rows);
        sq::sign_normalize(r);
        *seconds = seconds_since(t0);
        if (r_out) square_out(r, n, r_out);
        break;
      }
      case 4: {
        const sq::UpperTriangular r = sq::reference_hhqr(x);
        *seconds = seconds_since(t0);
        if (r_out) square_out(r, n, r_out);
        break;
      }
      case 5: {
        const sq::GramMatrix c = sq::tsmttsm(x, plan_from(k, b, false, m, n));
        *seconds = seconds_since(t0);
        if (r_out) square_out(c, n, r_out);
        break;
      }
      default:
        throw sq::ArgumentError("ref_timed_factor: unknown method");
    }
  });
}

}  // extern "C"
