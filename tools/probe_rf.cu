// Register-file operand bandwidth for DFMA: all-distinct sources vs shared multiplicand.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA error %s at %d\n",cudaGetErrorString(e),__LINE__); exit(1);} }while(0)
template <int KIND>
__global__ void k(double* out, int iters, const double* in) {
  double a[8], x[8], y[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) { a[j] = threadIdx.x + j; x[j] = in[j] + threadIdx.x * 1e-9; y[j] = in[8 + j] + threadIdx.x * 1e-9; }
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (KIND == 0) a[j] = fma(x[j], y[j], a[j]);              // 3 distinct
        if (KIND == 1) a[j] = fma(x[j], y[0], a[j]);              // shared multiplicand
        if (KIND == 2) a[j] = fma(x[j], y[(j + r) & 7], a[j]);    // 3 distinct, varying pairs
        if (KIND == 3) a[j] = fma(x[j], x[j], a[j]);              // square
        if (KIND == 4) a[j] = fma(a[j], y[0], x[0]);              // 1 distinct
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <class F> float timeit(F f, int reps = 3) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); f(); CK(cudaDeviceSynchronize()); float best = 1e30f;
  for (int r = 0; r < reps; r++) { cudaEventRecord(a); f(); cudaEventRecord(b); CK(cudaEventSynchronize(b)); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms; }
  return best;
}
template <int KIND> void run(int sms, double* out, const double* in) {
  int iters = 4000;
  for (int wps : {4, 8, 16}) {
    float ms = timeit([&] { k<KIND><<<sms, wps * 32>>>(out, iters, in); });
    printf("kind %d warps/SM %2d: %.2f TF\n", KIND, wps, 2.0 * 8 * 4 * iters * (double)sms * wps * 32 / ms / 1e9);
  }
}
int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0)); int sms = p.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, sizeof(double) * sms * 1024)); double* in; CK(cudaMalloc(&in, 128));
  double h[16]; for (int i = 0; i < 16; ++i) h[i] = 1.0 + 1e-9 * i; CK(cudaMemcpy(in, h, 128, cudaMemcpyHostToDevice));
  run<0>(sms, out, in); run<1>(sms, out, in); run<2>(sms, out, in); run<3>(sms, out, in); run<4>(sms, out, in);
  return 0;
}
