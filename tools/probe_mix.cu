// Does a DFMA (2 issue cycles on the 16-lane FP64 pipe) block the issue port for other pipes?
// Body: 8 independent DFMAs + M independent ALU (integer) or FP32 or LDS instructions.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA error %s at %d\n",cudaGetErrorString(e),__LINE__); exit(1);} }while(0)
template <int M, int KIND>
__global__ void k_mix(double* out, int iters, const double* in) {
  __shared__ double sh[1024];
  double a[8];
  unsigned x[8]; float f[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) { a[j] = threadIdx.x + j; x[j] = threadIdx.x * 7 + j; f[j] = x[j]; }
  sh[threadIdx.x] = threadIdx.x; __syncthreads();
  double b = in[0], c = in[1];
  double acc = 0;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        a[j] = fma(a[j], b, c);
        if (j < M) {
          if (KIND == 0) x[j] = x[j] * 3u + 1u;               // IMAD
          if (KIND == 1) f[j] = fmaf(f[j], 1.0001f, 0.5f);    // FFMA
          if (KIND == 2) x[j] = (x[j] ^ (x[j] >> 3)) + 1u;     // LOP/SHF/IADD (3 ALU ops)
          if (KIND == 3) acc += sh[(threadIdx.x + j * 32 + i) & 1023];  // LDS + DADD
          if (KIND == 4) sh[(threadIdx.x + j * 32) & 1023] = a[j];     // STS
        }
      }
    }
  }
  double s = acc;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j] + x[j] + f[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <class F> float timeit(F f, int reps = 3) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); f(); CK(cudaDeviceSynchronize()); float best = 1e30f;
  for (int r = 0; r < reps; r++) { cudaEventRecord(a); f(); cudaEventRecord(b); CK(cudaEventSynchronize(b)); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms; }
  return best;
}
template <int M, int KIND> void run(int sms, double* out, const double* in, int khz) {
  int iters = 4000;
  for (int wps : {4, 8}) {
    float ms = timeit([&] { k_mix<M, KIND><<<sms, wps * 32>>>(out, iters, in); });
    double clk = ms * 1e-3 * khz * 1e3;
    printf("kind %d M %d warps/SM %d: %.2f clk per (8 DFMA + %d other) per warp/SMSP -> %.2f TF\n", KIND, M, wps,
           clk / (4.0 * iters) / (wps / 4), M, 2.0 * 8 * 4 * iters * (double)sms * wps * 32 / ms / 1e9);
  }
}
int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0)); int sms = p.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, sizeof(double) * sms * 1024)); double* in; CK(cudaMalloc(&in, 64));
  double h[2] = {1.0000001, 0.5}; CK(cudaMemcpy(in, h, 16, cudaMemcpyHostToDevice));
  int khz = p.clockRate;
  run<0, 0>(sms, out, in, khz); run<4, 0>(sms, out, in, khz); run<8, 0>(sms, out, in, khz);
  run<4, 1>(sms, out, in, khz); run<8, 1>(sms, out, in, khz);
  run<4, 2>(sms, out, in, khz); run<8, 2>(sms, out, in, khz);
  run<2, 3>(sms, out, in, khz); run<4, 3>(sms, out, in, khz);
  run<2, 4>(sms, out, in, khz); run<4, 4>(sms, out, in, khz); run<8, 4>(sms, out, in, khz);
  return 0;
}
