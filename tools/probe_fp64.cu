// FP64 issue model probe: DFMA throughput vs warps/SM and independent chains per warp (ILP),
// dependent-issue latency, and DFMA mixed with LDS / SHFL / register-bank pressure.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA error %s at %d\n",cudaGetErrorString(e),__LINE__); exit(1);} }while(0)
template <int ILP>
__global__ void k_ilp(double* out, int iters, long long* clk) {
  double a[ILP];
#pragma unroll
  for (int j = 0; j < ILP; ++j) a[j] = threadIdx.x + j;
  double b = 1.0000001, c = 0.5;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int j = 0; j < ILP; ++j) a[j] = fma(a[j], b, c);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int j = 0; j < ILP; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) clk[0] = t1 - t0;
}
// distinct multiplicands per chain (3 different source registers, like the real kernel)
template <int ILP>
__global__ void k_ilp3(double* out, int iters, long long* clk, const double* in) {
  double a[ILP], v[8], w[ILP];
#pragma unroll
  for (int j = 0; j < ILP; ++j) { a[j] = threadIdx.x + j; w[j] = in[j]; }
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = in[8 + j];
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int j = 0; j < ILP; ++j) a[j] = fma(v[r], w[j], a[j]);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int j = 0; j < ILP; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) clk[0] = t1 - t0;
}
template <class F> float timeit(F f, int reps = 3) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); f(); CK(cudaDeviceSynchronize()); float best = 1e30f;
  for (int r = 0; r < reps; r++) { cudaEventRecord(a); f(); cudaEventRecord(b); CK(cudaEventSynchronize(b)); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms; }
  return best;
}
template <int ILP> void run(int sms, double* out, long long* clk, const double* in) {
  int iters = 4000;
  for (int wps : {1, 4, 6, 8, 12, 16}) {
    int thr = wps * 32;
    float ms = timeit([&] { k_ilp<ILP><<<sms, thr>>>(out, iters, clk); });
    long long c; CK(cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost));
    float ms3 = timeit([&] { k_ilp3<ILP><<<sms, thr>>>(out, iters, clk, in); });
    long long c3; CK(cudaMemcpy(&c3, clk, 8, cudaMemcpyDeviceToHost));
    printf("ILP %2d warps/SM %2d: %6.2f TF  %.2f clk/DFMA/warp | 3-src: %6.2f TF %.2f clk/DFMA/warp\n", ILP, wps,
           2.0 * 8 * ILP * iters * (double)sms * thr / ms / 1e9, (double)c / (8.0 * ILP * iters),
           2.0 * 8 * ILP * iters * (double)sms * thr / ms3 / 1e9, (double)c3 / (8.0 * ILP * iters));
  }
}
int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, sizeof(double) * sms * 1024)); long long* clk; CK(cudaMalloc(&clk, 64));
  double* in; CK(cudaMalloc(&in, 64 * 8)); double h[64]; for (int i = 0; i < 64; ++i) h[i] = 1.0 + i * 1e-9; CK(cudaMemcpy(in, h, 512, cudaMemcpyHostToDevice));
  run<1>(sms, out, clk, in); run<2>(sms, out, clk, in); run<3>(sms, out, clk, in); run<4>(sms, out, clk, in); run<6>(sms, out, clk, in); run<8>(sms, out, clk, in); run<16>(sms, out, clk, in);
  return 0;
}
