// Thread-private fused Gram kernels for narrow matrices (n <= 12).
//
//   OP_PLAIN     C = X^T X                      reference tsmttsm    (src/gram.cpp:113-121)
//   OP_SOLVE     C = (X R^-1)^T (X R^-1)        reference tsmRttsmR  (src/gram.cpp:123-140)
//   OP_MULTIPLY  C = (X B)^T (X B)              reference tsmmttsmm  (src/gram.cpp:142-151)
//
// Every thread streams its own rows (two adjacent rows per 128-bit load; a warp reads 512
// contiguous bytes per column), applies R^-1 (substitution in the reference's column order,
// src/kernels_scalar.cpp:19-32) or B to the row IN REGISTERS and accumulates the n(n+1)/2 upper
// triangle entries in registers.  At n <= 8 that is at most 100 FMAs per row against 64 bytes of
// HBM traffic, so these kernels sit on the memory roofline; up to 12 columns (78 accumulators, one CTA per
// SM) they still beat the DMMA kernels (gram_kernels.cu), whose padded 16-column tiles do 2.4x the useful
// work at 9 columns - the crossover is per operation (kernels.h: gram_use_thread).  Per-CTA partials are
// reduced in fixed order (deterministic, gram.cpp:81-92).
#include <type_traits>

#include "kernels.h"

namespace sqb {

namespace {

template <int B, int E, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

constexpr int kGT = 256;  // threads per CTA

// Rows per thread per step and resident CTAs per SM: two CTAs (<= 128 registers) wherever the
// accumulators + rows fit, which doubles the loads in flight.
template <int N, int OP>
struct GtCfg {
  // 9..12 columns: up to 78 accumulators + 2 rows of the panel per thread - one CTA per SM, 255 registers
  static constexpr int MINB = ((OP == OP_MULTIPLY && N >= 5) || N >= 9) ? 1 : 2;
  static constexpr int P = ((N >= 7 && OP != OP_MULTIPLY) || N >= 9) ? 2 : 4;
  static constexpr int kChunk = 32 * P;  // rows a warp consumes per step
};

template <int N, int OP>
__global__ void __launch_bounds__(kGT, GtCfg<N, OP>::MINB) gram_thread_kernel(const GramParams prm) {
  constexpr int TRI = N * (N + 1) / 2, NW = kGT / 32;
  constexpr int kGP = GtCfg<N, OP>::P, kGChunk = GtCfg<N, OP>::kChunk;
  __shared__ double fac[N * N];
  __shared__ double inv[N];
  __shared__ double red[NW][TRI];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (OP != OP_PLAIN) {
    for (int i = tid; i < N * N; i += kGT) fac[i] = prm.factor[i];
    __syncthreads();
    if (OP == OP_SOLVE && tid == 0) {
      // reference tsmRttsmR pre-check (gram.cpp:126-134)
      double mx = 0.0;
      for (int j = 0; j < N; ++j) mx = fmax(mx, fabs(fac[j + j * N]));
      const double dtol = static_cast<double>(N) * 2.220446049250313e-16 * mx;
      int bad = -1;
      for (int j = 0; j < N; ++j) {
        const double d = fac[j + j * N];
        if (bad < 0 && !(fabs(d) > dtol)) bad = j;
        inv[j] = 1.0 / d;
      }
      if (bad >= 0 && blockIdx.x == 0) raise_status(prm.status, SQB_E_SINGULAR, bad);
    }
    __syncthreads();
  }

  const long long blk = blockIdx.x;
  const long long begin = min(blk * prm.rows_per_block, prm.m);
  const long long end = min((blk + 1) * prm.rows_per_block, prm.m);
  const long long nchunks = (end - begin + kGChunk - 1) / kGChunk;
  const bool aligned = view_bulk_aligned(prm.x, N, begin);

  double acc[TRI];
#pragma unroll
  for (int e = 0; e < TRI; ++e) acc[e] = 0.0;

  for (long long ch = warp; ch < nchunks; ch += NW) {
    const long long r0 = begin + ch * kGChunk;
    if (aligned && lane < N && r0 + static_cast<long long>(NW + 1) * kGChunk <= end) {
      const double* nxt = prm.x.col(lane) + r0 + static_cast<long long>(NW) * kGChunk;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nxt), "r"(kGChunk * 8) : "memory");
    }
    double w[N][kGP];
    if (aligned && r0 + kGChunk <= end) {
      static_for<0, N>([&](auto jj) {
        constexpr int j = decltype(jj)::value;
        const double* cp = prm.x.col(j) + r0 + 2 * lane;
#pragma unroll
        for (int k = 0; k < kGP / 2; ++k) {
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
        for (int i = 0; i < kGP; ++i) {
          const long long row = r0 + 64 * (i >> 1) + 2 * lane + (i & 1);
          w[j][i] = row < end ? __ldg(cp + row) : 0.0;
        }
      });
    }
    if (OP == OP_SOLVE) {
      static_for<0, N>([&](auto jj) {
        constexpr int j = decltype(jj)::value;
        static_for<0, j>([&](auto ii) {
          constexpr int i2 = decltype(ii)::value;
          const double rij = fac[i2 + j * N];
#pragma unroll
          for (int i = 0; i < kGP; ++i) w[j][i] = fma(-rij, w[i2][i], w[j][i]);
        });
        const double d = inv[j];
#pragma unroll
        for (int i = 0; i < kGP; ++i) w[j][i] *= d;
      });
    } else if (OP == OP_MULTIPLY) {
      double y[N][kGP];
      static_for<0, N>([&](auto jj) {
        constexpr int j = decltype(jj)::value;
#pragma unroll
        for (int i = 0; i < kGP; ++i) y[j][i] = 0.0;
        static_for<0, N>([&](auto kk) {
          constexpr int k = decltype(kk)::value;
          const double bkj = fac[k + j * N];
#pragma unroll
          for (int i = 0; i < kGP; ++i) y[j][i] = fma(bkj, w[k][i], y[j][i]);
        });
      });
      static_for<0, N>([&](auto jj) {
        constexpr int j = decltype(jj)::value;
#pragma unroll
        for (int i = 0; i < kGP; ++i) w[j][i] = y[j][i];
      });
    }
    static_for<0, N>([&](auto jj) {
      constexpr int j = decltype(jj)::value;
      static_for<0, j + 1>([&](auto ii) {
        constexpr int i2 = decltype(ii)::value;
        constexpr int e = j * (j + 1) / 2 + i2;
#pragma unroll
        for (int i = 0; i < kGP; ++i) acc[e] = fma(w[i2][i], w[j][i], acc[e]);
      });
    });
  }

  // CTA reduction: lanes by xor-shuffle, warps in ascending order
#pragma unroll
  for (int e = 0; e < TRI; ++e) {
    double s = acc[e];
    for (int o = 16; o > 0; o >>= 1) s += shfl_xor_f64(s, o);
    if (lane == 0) red[warp][e] = s;
  }
  __syncthreads();
  double* dst = prm.partial + blk * static_cast<long long>(N) * N;
  for (int idx = tid; idx < N * N; idx += kGT) {
    const int i = idx % N, j = idx / N;
    double s = 0.0;
    if (i <= j)
      for (int wv = 0; wv < NW; ++wv) s += red[wv][j * (j + 1) / 2 + i];
    dst[idx] = s;
  }
}

template <int OP>
cudaError_t launch_op(const GramParams& prm, long long nb, cudaStream_t st) {
  switch (prm.n) {
    case 1: gram_thread_kernel<1, OP><<<static_cast<unsigned>(nb), kGT, 0, st>>>(prm); break;
    case 2: gram_thread_kernel<2, OP><<<static_cast<unsigned>(nb), kGT, 0, st>>>(prm); break;
    case 3: gram_thread_kernel<3, OP><<<static_cast<unsigned>(nb), kGT, 0, st>>>(prm); break;
    case 4: gram_thread_kernel<4, OP><<<static_cast<unsigned>(nb), kGT, 0, st>>>(prm); break;
    case 5: gram_thread_kernel<5, OP><<<static_cast<unsigned>(nb), kGT, 0, st>>>(prm); break;
    case 6: gram_thread_kernel<6, OP><<<static_cast<unsigned>(nb), kGT, 0, st>>>(prm); break;
    case 7: gram_thread_kernel<7, OP><<<static_cast<unsigned>(nb), kGT, 0, st>>>(prm); break;
    case 8: gram_thread_kernel<8, OP><<<static_cast<unsigned>(nb), kGT, 0, st>>>(prm); break;
    case 9: gram_thread_kernel<9, OP><<<static_cast<unsigned>(nb), kGT, 0, st>>>(prm); break;
    case 10: gram_thread_kernel<10, OP><<<static_cast<unsigned>(nb), kGT, 0, st>>>(prm); break;
    case 11: gram_thread_kernel<11, OP><<<static_cast<unsigned>(nb), kGT, 0, st>>>(prm); break;
    case 12: gram_thread_kernel<12, OP><<<static_cast<unsigned>(nb), kGT, 0, st>>>(prm); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_gram_thread(const GramParams& prm, int op, long long num_blocks,
                               cudaStream_t stream) {
  switch (op) {
    case OP_PLAIN: return launch_op<OP_PLAIN>(prm, num_blocks, stream);
    case OP_SOLVE: return launch_op<OP_SOLVE>(prm, num_blocks, stream);
    case OP_MULTIPLY: return launch_op<OP_MULTIPLY>(prm, num_blocks, stream);
    default: return cudaErrorInvalidValue;
  }
}

int gram_thread_chunk_rows(int n, int op) {
  return ((n >= 7 && op != OP_MULTIPLY) || n >= 9) ? 64 : 128;  // GtCfg<N, OP>::kChunk
}
int gram_thread_warps() { return kGT / 32; }
int gram_thread_ctas_per_sm(int n, int op) { return ((op == OP_MULTIPLY && n >= 5) || n >= 9) ? 1 : 2; }

}  // namespace sqb
