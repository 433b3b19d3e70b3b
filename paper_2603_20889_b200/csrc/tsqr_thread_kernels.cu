// Thread-private Q-less Householder TSQR for narrow matrices (n <= 16).
//
// Reference semantics: block_qless_qr_core / factor_trapezoidal / make_reflector
// (reference src/tsqr.cpp:51-158) - fold row panels into a running upper triangle with Householder
// reflectors, discard Q.  TSQR lets the rows be partitioned any way we like, so here EVERY THREAD
// is its own leaf of the reduction tree: it streams its own rows (two adjacent rows per 128-bit
// load, a warp reads 512 contiguous bytes per column), keeps its own running triangle
// (registers for n <= 8, a bank-conflict-free interleaved shared-memory slot for n <= 16) and
// never talks to another thread until the end.  No shuffles, no barriers, no broadcast in the
// streaming loop; the per-reflector work is fully unrolled with static register indices.
// The CTA's triangles are then merged by a shared-memory tree with the same folding routine and one
// triangle per CTA goes to Y, exactly where tsqr_stage1 puts it (reference src/tsqr.cpp:168-184).
#include <cstdlib>
#include <type_traits>

#include "kernels.h"

namespace sqb {

namespace {

// Compile-time loop: nvcc stops honouring "#pragma unroll" on the column loops once n > 8, and a
// partially unrolled loop would push the register panel into local memory.
template <int B, int E, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

template <int N>
struct ThreadCfg {
  static constexpr int kTri = N * (N + 1) / 2;
  static constexpr bool kRegR = N <= 8;                 // running triangle in registers
  static constexpr int P = N == 1 ? 32 : (N == 2 ? 16 : (N <= 8 ? 8 : 4));  // rows folded per step
  static constexpr int kMaxT = (220 * 1024) / (kTri * 8) / 32 * 32;
  static constexpr int T = kMaxT >= 256 ? 256 : kMaxT;  // threads per CTA
  static constexpr size_t kSmemBytes = sizeof(double) * kTri * T;
  static constexpr int kChunk = 32 * P;                 // rows a warp consumes per step
};

// Running triangle accessor: packed row-major (row c holds (c, c..N-1)); registers or an
// interleaved shared-memory slot (element e of thread t at rs[e*T + t]).
template <int N, bool REG, int T>
struct Tri {
  double r[REG ? N * (N + 1) / 2 : 1];
  double* rs;
  static __device__ __forceinline__ constexpr int idx(int c, int j) {
    return c * N - (c * (c - 1)) / 2 + (j - c);
  }
  __device__ __forceinline__ double get(int c, int j) const {
    if constexpr (REG) return r[idx(c, j)];
    else return rs[idx(c, j) * T];
  }
  __device__ __forceinline__ void set(int c, int j, double v) {
    if constexpr (REG) r[idx(c, j)] = v;
    else rs[idx(c, j) * T] = v;
  }
};

// Fold P dense rows (w[col][row]) into the thread's triangle.
template <int N, int P, bool REG, int T>
__device__ __forceinline__ void fold_rows(double (&w)[N][P], Tri<N, REG, T>& tri) {
  static_for<0, N>([&](auto cc) {
    constexpr int c = decltype(cc)::value;
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int i = 0; i < P; i += 2) {
      s0 = fma(w[c][i], w[c][i], s0);
      s1 = fma(w[c][i + 1], w[c][i + 1], s1);
    }
    const double pivot = tri.get(c, c);
    const Reflector h = make_reflector(pivot, s0 + s1);
    static_for<c + 1, N>([&](auto jj) {
      constexpr int j = decltype(jj)::value;
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int i = 0; i < P; i += 2) {
        d0 = fma(w[c][i], w[j][i], d0);
        d1 = fma(w[c][i + 1], w[j][i + 1], d1);
      }
      const double rcj = tri.get(c, j);
      const double s = h.gamma * fma(h.u0, rcj, d0 + d1);
      tri.set(c, j, fma(-h.u0, s, rcj));
#pragma unroll
      for (int i = 0; i < P; ++i) w[j][i] = fma(-w[c][i], s, w[j][i]);
    });
    tri.set(c, c, h.beta);
  });
}

template <int N>
__global__ void __launch_bounds__(ThreadCfg<N>::T, 1) tsqr_thread_kernel(const TsqrParams prm) {
  using Cfg = ThreadCfg<N>;
  constexpr int P = Cfg::P, T = Cfg::T, NW = T / 32, CH = Cfg::kChunk;
  constexpr bool REG = Cfg::kRegR;
  extern __shared__ __align__(16) double rs_all[];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  Tri<N, REG, T> tri;
  tri.rs = rs_all + tid;
#pragma unroll
  for (int e = 0; e < Cfg::kTri; ++e) {
    if constexpr (REG) tri.r[e] = 0.0;
    else tri.rs[e * T] = 0.0;
  }

  const long long blk = blockIdx.x;
  const long long begin = min(blk * prm.rows_per_block, prm.m);
  const long long end = min((blk + 1) * prm.rows_per_block, prm.m);
  const long long nchunks = (end - begin + CH - 1) / CH;
  const bool aligned = view_bulk_aligned(prm.x, N, begin);

  double w[N][P];
  for (long long ch = warp; ch < nchunks; ch += NW) {
    const long long r0 = begin + ch * CH;
    // pull the warp's next chunk towards L2 while this one is folded
    if (aligned && ch + NW < nchunks && lane < N && r0 + static_cast<long long>(NW + 1) * CH <= end) {
      const double* nxt = prm.x.col(lane) + r0 + static_cast<long long>(NW) * CH;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nxt), "r"(CH * 8) : "memory");
    }
    if (aligned && r0 + CH <= end) {
      static_for<0, N>([&](auto jj) {
        constexpr int j = decltype(jj)::value;
        const double* cp = prm.x.col(j) + r0 + 2 * lane;
#pragma unroll
        for (int k = 0; k < P / 2; ++k) {
          const double2 v = __ldcs(reinterpret_cast<const double2*>(cp + 64 * k));
          w[j][2 * k] = v.x;
          w[j][2 * k + 1] = v.y;
        }
      });
    } else {
      static_for<0, N>([&](auto jj) {
        constexpr int j = decltype(jj)::value;
        const double* cp = prm.x.col(j);
#pragma unroll
        for (int i = 0; i < P; ++i) {
          const long long row = r0 + 64 * (i >> 1) + 2 * lane + (i & 1);
          w[j][i] = row < end ? __ldg(cp + row) : 0.0;
        }
      });
    }
    fold_rows<N, P, REG, T>(w, tri);
  }

  // ---- merge the CTA's triangles: shared-memory tree, same folding routine -----------------------
  if constexpr (REG) {
#pragma unroll
    for (int e = 0; e < Cfg::kTri; ++e) tri.rs[e * T] = tri.r[e];
  }
  int active = T;
  while (active > 1) {
    const int half = (active + 1) / 2;
    __syncthreads();
    if (tid < active - half) {
      const double* other = rs_all + tid + half;
#pragma unroll 1
      for (int base = 0; base < N; base += P) {
        static_for<0, N>([&](auto jj) {
          constexpr int j = decltype(jj)::value;
#pragma unroll
          for (int i = 0; i < P; ++i) {
            const int row = base + i;  // runtime row, static register indices
            w[j][i] = (row <= j) ? other[(row * N - (row * (row - 1)) / 2 + (j - row)) * T] : 0.0;
          }
        });
        fold_rows<N, P, REG, T>(w, tri);
      }
      if constexpr (REG) {
#pragma unroll
        for (int e = 0; e < Cfg::kTri; ++e) tri.rs[e * T] = tri.r[e];
      }
    }
    active = half;
  }
  __syncthreads();

  // ---- CTA triangle -> rows [blk*n, blk*n+n) of Y (full square, zeros below the diagonal) ---------
  double* dst = prm.y + blk * N;
  bool bad = false;
  for (int idx = tid; idx < N * N; idx += T) {
    const int i = idx % N, j = idx / N;
    double val = 0.0;
    if (i <= j) {
      val = rs_all[Tri<N, REG, T>::idx(i, j) * T];
      bad = bad || is_nonfinite(val);
      if (prm.finalize && rs_all[Tri<N, REG, T>::idx(i, i) * T] < 0.0) val = -val;
    }
    dst[i + j * prm.ldy] = val;
  }
  if (prm.check_finite && bad) atomicExch(&prm.status->nonfinite, 1);
}

template <int N>
cudaError_t launch_n(const TsqrParams& prm, long long num_blocks, cudaStream_t stream) {
  using Cfg = ThreadCfg<N>;
  static unsigned long long smem_ready = 0;  // per-device opt-in mask
  {
    cudaError_t e = opt_in_dynamic_smem(tsqr_thread_kernel<N>, Cfg::kSmemBytes, &smem_ready);
    if (e != cudaSuccess) return e;
  }
  tsqr_thread_kernel<N><<<static_cast<unsigned>(num_blocks), Cfg::T, Cfg::kSmemBytes, stream>>>(prm);
  return cudaGetLastError();
}

}  // namespace

#define SQB_N_SWITCH(EXPR)       \
  switch (n) {                   \
    case 1: return EXPR(1);      \
    case 2: return EXPR(2);      \
    case 3: return EXPR(3);      \
    case 4: return EXPR(4);      \
    case 5: return EXPR(5);      \
    case 6: return EXPR(6);      \
    case 7: return EXPR(7);      \
    case 8: return EXPR(8);      \
    case 9: return EXPR(9);      \
    case 10: return EXPR(10);    \
    case 11: return EXPR(11);    \
    case 12: return EXPR(12);    \
    case 13: return EXPR(13);    \
    case 14: return EXPR(14);    \
    case 15: return EXPR(15);    \
    default: return EXPR(16);    \
  }

cudaError_t launch_tsqr_thread(const TsqrParams& prm, long long num_blocks, cudaStream_t stream) {
  const int n = prm.n;
  if (n < 1 || n > kThreadTsqrMaxN) return cudaErrorInvalidValue;
#define LN(NV) launch_n<NV>(prm, num_blocks, stream)
  SQB_N_SWITCH(LN)
#undef LN
}

int tsqr_thread_chunk_rows(int n) {
#define CN(NV) ThreadCfg<NV>::kChunk
  SQB_N_SWITCH(CN)
#undef CN
}

int tsqr_thread_warps(int n) {
#define WN(NV) (ThreadCfg<NV>::T / 32)
  SQB_N_SWITCH(WN)
#undef WN
}

}  // namespace sqb
