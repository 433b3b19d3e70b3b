// Synthetic inputs generated in place on the device (harness side of the hot path).
//
//   fill_gaussian   counter-based Box-Muller over the reference's SplitMix64 stream
//                   (reference src/matgen.cpp:8-17 provides mix64 / uniform01 only - it has no
//                   Gaussian generator; element e = j*m_total + i draws positions 2e and 2e+1)
//   generate        X = U diag(sigma) V^T with prescribed 2-norm condition number
//                   (reference generate, src/matgen.cpp:77-109; random_reflectors :32-59)
#include "kernels.h"

namespace sqb {

namespace {

__host__ __device__ __forceinline__ unsigned long long mix64(unsigned long long seed,
                                                             unsigned long long index) {
  unsigned long long z = seed + (index + 1ull) * 0x9E3779B97F4A7C15ull;  // matgen.cpp:8-13
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

__host__ __device__ __forceinline__ double uniform01(unsigned long long seed,
                                                     unsigned long long index) {
  return static_cast<double>(mix64(seed, index) >> 11) * 0x1.0p-53;  // matgen.cpp:15-17
}

__global__ void fill_gaussian_kernel(double* __restrict__ x, long long m, int n, long long ld,
                                     unsigned long long seed, long long row_offset,
                                     long long m_total) {
  const long long total = m * n;
  for (long long t = threadIdx.x + static_cast<long long>(blockIdx.x) * blockDim.x; t < total;
       t += static_cast<long long>(blockDim.x) * gridDim.x) {
    const long long j = t / m, i = t - j * m;
    const unsigned long long e =
        static_cast<unsigned long long>(j) * static_cast<unsigned long long>(m_total) +
        static_cast<unsigned long long>(i + row_offset);
    const double u1 = fmax(uniform01(seed, 2ull * e), 0x1.0p-53);
    const double u2 = uniform01(seed, 2ull * e + 1ull);
    x[i + j * ld] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
  }
}

// ---- controlled-spectrum generator ---------------------------------------------------------
constexpr int kGenMaxN = 64;
constexpr int kGenThreads = 256;
constexpr int kGenBlocks = 148 * 4;

__global__ void gen_identity_kernel(double* __restrict__ u, long long m, int n, long long ld) {
  const long long total = m * n;
  for (long long t = threadIdx.x + static_cast<long long>(blockIdx.x) * blockDim.x; t < total;
       t += static_cast<long long>(blockDim.x) * gridDim.x) {
    const long long j = t / m, i = t - j * m;
    u[i + j * ld] = i == j ? 1.0 : 0.0;
  }
}

// partial[block][0] = sum v_i^2, partial[block][1+j] = sum v_i u(i,j); v_i from the stream at
// base + jr*len + i mapped to (-1,1)  (matgen.cpp:38-47)
__global__ void __launch_bounds__(kGenThreads)
    gen_dots_kernel(const double* __restrict__ u, long long m, int n, long long ld,
                    unsigned long long seed, unsigned long long base, long long jr,
                    double* __restrict__ partial) {
  double acc[kGenMaxN + 1];
#pragma unroll
  for (int j = 0; j <= kGenMaxN; ++j) acc[j] = 0.0;
  for (long long i = threadIdx.x + static_cast<long long>(blockIdx.x) * blockDim.x; i < m;
       i += static_cast<long long>(blockDim.x) * gridDim.x) {
    const double v = 2.0 * uniform01(seed, base + static_cast<unsigned long long>(jr * m + i)) - 1.0;
    acc[0] = fma(v, v, acc[0]);
#pragma unroll
    for (int j = 0; j < kGenMaxN; ++j)
      if (j < n) acc[1 + j] = fma(v, u[i + j * ld], acc[1 + j]);
  }
  __shared__ double red[kGenThreads / 32][kGenMaxN + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j <= kGenMaxN; ++j) {
    if (j <= n) {
      double s = acc[j];
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) red[warp][j] = s;
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j <= n; j += kGenThreads) {
    double s = 0.0;
    for (int w = 0; w < kGenThreads / 32; ++w) s += red[w][j];
    partial[static_cast<long long>(blockIdx.x) * (kGenMaxN + 1) + j] = s;
  }
}

// coef[j] = (2 / vv) * s_j   (0 when vv == 0: reflector skipped, matgen.cpp:48)
__global__ void gen_coef_kernel(const double* __restrict__ partial, int blocks, int n,
                                double* __restrict__ coef) {
  __shared__ double vv_s;
  if (threadIdx.x == 0) {
    double vv = 0.0;
    for (int b = 0; b < blocks; ++b) vv += partial[static_cast<long long>(b) * (kGenMaxN + 1)];
    vv_s = vv;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < blocks; ++b) s += partial[static_cast<long long>(b) * (kGenMaxN + 1) + 1 + j];
    coef[j] = vv_s == 0.0 ? 0.0 : (2.0 / vv_s) * s;
  }
}

__global__ void gen_update_kernel(double* __restrict__ u, long long m, int n, long long ld,
                                  unsigned long long seed, unsigned long long base, long long jr,
                                  const double* __restrict__ coef) {
  __shared__ double cf[kGenMaxN];
  for (int j = threadIdx.x; j < n; j += blockDim.x) cf[j] = coef[j];
  __syncthreads();
  for (long long i = threadIdx.x + static_cast<long long>(blockIdx.x) * blockDim.x; i < m;
       i += static_cast<long long>(blockDim.x) * gridDim.x) {
    const double v = 2.0 * uniform01(seed, base + static_cast<unsigned long long>(jr * m + i)) - 1.0;
    for (int j = 0; j < n; ++j) u[i + j * ld] = fma(-v, cf[j], u[i + j * ld]);
  }
}

// vs(j,k) = V(j,k) * sigma_k on one CTA: V = H_0...H_{n-1} I with the stream based at 2^63
// (matgen.cpp:21-23), sigma geometric or linear (matgen.cpp:62-75).
__global__ void gen_v_kernel(int n, double kappa, int linear_decay, unsigned long long seed,
                             double* __restrict__ vs) {
  __shared__ double v[kGenMaxN * kGenMaxN];
  __shared__ double w[kGenMaxN];
  __shared__ double cf[kGenMaxN];
  __shared__ double vv_s;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < n * n; idx += blockDim.x) v[idx] = (idx % n == idx / n) ? 1.0 : 0.0;
  __syncthreads();
  for (int jr = n - 1; jr >= 0; --jr) {
    for (int i = tid; i < n; i += blockDim.x)
      w[i] = 2.0 * uniform01(seed, (1ull << 63) + static_cast<unsigned long long>(jr * n + i)) - 1.0;
    __syncthreads();
    if (tid == 0) {
      double vv = 0.0;
      for (int i = 0; i < n; ++i) vv += w[i] * w[i];
      vv_s = vv;
    }
    __syncthreads();
    for (int j = tid; j < n; j += blockDim.x) {
      double s = 0.0;
      for (int i = 0; i < n; ++i) s += w[i] * v[i + j * n];
      cf[j] = vv_s == 0.0 ? 0.0 : (2.0 / vv_s) * s;
    }
    __syncthreads();
    for (int idx = tid; idx < n * n; idx += blockDim.x) v[idx] -= w[idx % n] * cf[idx / n];
    __syncthreads();
  }
  for (int idx = tid; idx < n * n; idx += blockDim.x) {
    const int k = idx / n;
    double sigma;
    if (n == 1) sigma = 1.0;
    else if (!linear_decay) sigma = pow(kappa, -static_cast<double>(k) / static_cast<double>(n - 1));
    else sigma = 1.0 + (static_cast<double>(k) / static_cast<double>(n - 1)) * (1.0 / kappa - 1.0);
    vs[idx] = v[idx] * sigma;
  }
}

// X(i,j) = sum_k (V(j,k) sigma_k) U(i,k), k ascending (matgen.cpp:100-107)
__global__ void gen_product_kernel(const double* __restrict__ u, long long m, int n, long long ldu,
                                   const double* __restrict__ vs, double* __restrict__ x,
                                   long long ld) {
  __shared__ double v[kGenMaxN * kGenMaxN];
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) v[idx] = vs[idx];
  __syncthreads();
  for (long long i = threadIdx.x + static_cast<long long>(blockIdx.x) * blockDim.x; i < m;
       i += static_cast<long long>(blockDim.x) * gridDim.x) {
    double row[kGenMaxN];
#pragma unroll
    for (int k = 0; k < kGenMaxN; ++k) row[k] = k < n ? u[i + k * ldu] : 0.0;
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < kGenMaxN; ++k)
        if (k < n) s = fma(v[j + k * n], row[k], s);
      x[i + j * ld] = s;
    }
  }
}

}  // namespace

cudaError_t launch_fill_gaussian(double* x, long long m, int n, long long ld, unsigned long long seed,
                                 long long row_offset, long long m_total, cudaStream_t stream) {
  fill_gaussian_kernel<<<148 * 8, 256, 0, stream>>>(x, m, n, ld, seed, row_offset, m_total);
  return cudaGetLastError();
}

size_t generate_scratch_doubles(long long m, int n) {
  return static_cast<size_t>(m) * n + static_cast<size_t>(kGenBlocks) * (kGenMaxN + 1) + 2 * kGenMaxN +
         static_cast<size_t>(kGenMaxN) * kGenMaxN;
}

cudaError_t launch_generate(double* x, long long m, int n, long long ld, double kappa,
                            int linear_decay, unsigned long long seed, double* scratch,
                            cudaStream_t stream) {
  if (n < 1 || n > kGenMaxN || m < n) return cudaErrorInvalidValue;
  double* u = scratch;
  double* partial = u + static_cast<size_t>(m) * n;
  double* coef = partial + static_cast<size_t>(kGenBlocks) * (kGenMaxN + 1);
  double* vs = coef + 2 * kGenMaxN;
  gen_identity_kernel<<<kGenBlocks, kGenThreads, 0, stream>>>(u, m, n, m);
  for (long long jr = n - 1; jr >= 0; --jr) {
    gen_dots_kernel<<<kGenBlocks, kGenThreads, 0, stream>>>(u, m, n, m, seed, 0ull, jr, partial);
    gen_coef_kernel<<<1, 64, 0, stream>>>(partial, kGenBlocks, n, coef);
    gen_update_kernel<<<kGenBlocks, kGenThreads, 0, stream>>>(u, m, n, m, seed, 0ull, jr, coef);
  }
  gen_v_kernel<<<1, 256, 0, stream>>>(n, kappa, linear_decay, seed, vs);
  gen_product_kernel<<<kGenBlocks, 128, 0, stream>>>(u, m, n, m, vs, x, ld);
  return cudaGetLastError();
}

}  // namespace sqb
