// Hardware probe for design decisions (not part of the product): FP64 FMA vs DMMA issue rates,
// shuffle rate, read-only HBM bandwidth (LDG.128 and cp.async.bulk), H2D bandwidth.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA error %s at %d\n",cudaGetErrorString(e),__LINE__); exit(1);} }while(0)

__global__ void k_dfma(double* out, int iters) {
  double a0=threadIdx.x, a1=a0+1, a2=a0+2, a3=a0+3, a4=a0+4, a5=a0+5, a6=a0+6, a7=a0+7;
  double b=1.0000001, c=0.5;
  for (int i=0;i<iters;i++){
    a0=fma(a0,b,c); a1=fma(a1,b,c); a2=fma(a2,b,c); a3=fma(a3,b,c);
    a4=fma(a4,b,c); a5=fma(a5,b,c); a6=fma(a6,b,c); a7=fma(a7,b,c);
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=a0+a1+a2+a3+a4+a5+a6+a7;
}
__device__ __forceinline__ void dmma884(double& d0,double& d1,double a,double b){
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n":"+d"(d0),"+d"(d1):"d"(a),"d"(b));
}
__global__ void k_dmma(double* out, int iters) {
  double a=threadIdx.x*1e-3, b=1.0+threadIdx.x*1e-6;
  double c[8][2];
  for(int j=0;j<8;j++){c[j][0]=j;c[j][1]=-j;}
  for (int i=0;i<iters;i++){
    #pragma unroll
    for(int j=0;j<8;j++) dmma884(c[j][0],c[j][1],a,b);
  }
  double s=0; for(int j=0;j<8;j++) s+=c[j][0]+c[j][1];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__device__ __forceinline__ void dmma1688(double (&d)[4],const double (&a)[4],const double (&b)[2]){
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
   :"+d"(d[0]),"+d"(d[1]),"+d"(d[2]),"+d"(d[3]):"d"(a[0]),"d"(a[1]),"d"(a[2]),"d"(a[3]),"d"(b[0]),"d"(b[1]));
}
__global__ void k_dmma1688(double* out, int iters) {
  double a[4]={threadIdx.x*1e-3,1e-3,2e-3,3e-3}, b[2]={1.0+threadIdx.x*1e-6,0.5};
  double c[4][4];
  for(int j=0;j<4;j++) for(int t=0;t<4;t++) c[j][t]=j+t;
  for (int i=0;i<iters;i++){
    #pragma unroll
    for(int j=0;j<4;j++) dmma1688(c[j],a,b);
  }
  double s=0; for(int j=0;j<4;j++) for(int t=0;t<4;t++) s+=c[j][t];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
// mixed: DFMA and DMMA interleaved 1:1 (in FMA-equivalents 8 dfma-warp-instr per dmma) to see if pipes are shared
__global__ void k_mixed(double* out, int iters) {
  double a=threadIdx.x*1e-3, b=1.0+threadIdx.x*1e-6;
  double c[4][2]; for(int j=0;j<4;j++){c[j][0]=j;c[j][1]=-j;}
  double f[8]; for(int j=0;j<8;j++) f[j]=j+threadIdx.x;
  for (int i=0;i<iters;i++){
    #pragma unroll
    for(int j=0;j<4;j++){ dmma884(c[j][0],c[j][1],a,b);
      #pragma unroll
      for(int t=0;t<8;t++) f[t]=fma(f[t],b,a);
    }
  }
  double s=0; for(int j=0;j<4;j++) s+=c[j][0]+c[j][1]; for(int t=0;t<8;t++) s+=f[t];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void k_shfl(double* out, int iters) {
  double a0=threadIdx.x, a1=a0+1, a2=a0+2, a3=a0+3;
  for (int i=0;i<iters;i++){
    a0=__shfl_xor_sync(0xffffffffu,a0,1); a1=__shfl_xor_sync(0xffffffffu,a1,2);
    a2=__shfl_xor_sync(0xffffffffu,a2,4); a3=__shfl_xor_sync(0xffffffffu,a3,8);
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=a0+a1+a2+a3;
}
__global__ void k_dsqrt(double* out, int iters) {
  double a0=threadIdx.x+2.0, a1=a0+1, a2=a0+2, a3=a0+3;
  for (int i=0;i<iters;i++){ a0=sqrt(a0)+2.0; a1=sqrt(a1)+2.0; a2=sqrt(a2)+2.0; a3=sqrt(a3)+2.0; }
  out[blockIdx.x*blockDim.x+threadIdx.x]=a0+a1+a2+a3;
}
__global__ void k_drcp(double* out, int iters) {
  double a0=threadIdx.x+2.0, a1=a0+1, a2=a0+2, a3=a0+3;
  for (int i=0;i<iters;i++){ a0=1.0/a0+2.0; a1=1.0/a1+2.0; a2=1.0/a2+2.0; a3=1.0/a3+2.0; }
  out[blockIdx.x*blockDim.x+threadIdx.x]=a0+a1+a2+a3;
}
__global__ void k_drsqrt(double* out, int iters) {
  double a0=threadIdx.x+2.0, a1=a0+1, a2=a0+2, a3=a0+3;
  for (int i=0;i<iters;i++){ a0=rsqrt(a0)+2.0; a1=rsqrt(a1)+2.0; a2=rsqrt(a2)+2.0; a3=rsqrt(a3)+2.0; }
  out[blockIdx.x*blockDim.x+threadIdx.x]=a0+a1+a2+a3;
}
__global__ void k_read(const double2* __restrict__ x, size_t n2, double* out) {
  double s0=0,s1=0,s2=0,s3=0;
  size_t stride=(size_t)gridDim.x*blockDim.x;
  size_t i=(size_t)blockIdx.x*blockDim.x+threadIdx.x;
  for (; i+3*stride<n2; i+=4*stride){
    double2 a=x[i], b=x[i+stride], c=x[i+2*stride], d=x[i+3*stride];
    s0+=a.x+a.y; s1+=b.x+b.y; s2+=c.x+c.y; s3+=d.x+d.y;
  }
  for (; i<n2; i+=stride){ double2 a=x[i]; s0+=a.x+a.y; }
  double s=s0+s1+s2+s3;
  if (s==123.456) out[0]=s;
}
// bulk-copy streaming read: each warp owns one 16 KB stage, lane 0 issues, all lanes touch the data lightly
__device__ __forceinline__ uint32_t smem_u32(const void* p){ return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k_bulk(const double* __restrict__ x, size_t nchunks, int chunk_bytes, int warps, double* out){
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bars[16];
  int warp=threadIdx.x>>5, lane=threadIdx.x&31;
  unsigned char* stage=smem+(size_t)warp*chunk_bytes;
  uint32_t bar=smem_u32(&bars[warp]);
  if(lane==0){ asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;"::"r"(bar)); }
  asm volatile("fence.mbarrier_init.release.cluster;":::"memory");
  __syncthreads();
  size_t gw=(size_t)blockIdx.x*warps+warp, tw=(size_t)gridDim.x*warps;
  uint32_t phase=0; double s=0;
  size_t c=gw;
  if(c<nchunks && lane==0){
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"::"r"(bar),"r"(chunk_bytes):"memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(stage)),"l"((const char*)x+c*(size_t)chunk_bytes),"r"(chunk_bytes),"r"(bar):"memory");
  }
  for(; c<nchunks; c+=tw){
    uint32_t done=0;
    while(!done){ asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}":"=r"(done):"r"(bar),"r"(phase):"memory"); }
    phase^=1;
    const double2* sp=(const double2*)stage;
    for(int i=lane;i<chunk_bytes/16;i+=32){ double2 v=sp[i]; s+=v.x+v.y; }
    __syncwarp();
    size_t nx=c+tw;
    if(nx<nchunks && lane==0){
      asm volatile("fence.proxy.async.shared::cta;":::"memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"::"r"(bar),"r"(chunk_bytes):"memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(stage)),"l"((const char*)x+nx*(size_t)chunk_bytes),"r"(chunk_bytes),"r"(bar):"memory");
    }
  }
  if(s==123.456) out[0]=s;
}
template<class F> float timeit(F f,int reps=5){ cudaEvent_t a,b; cudaEventCreate(&a);cudaEventCreate(&b); f(); CK(cudaDeviceSynchronize()); float best=1e30f;
  for(int r=0;r<reps;r++){ cudaEventRecord(a); f(); cudaEventRecord(b); CK(cudaEventSynchronize(b)); float ms; cudaEventElapsedTime(&ms,a,b); if(ms<best)best=ms;} return best; }
int main(){
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,0));
  printf("device %s SMs %d smem/block optin %zu clock %d kHz mem %zu MB L2 %d\n",p.name,p.multiProcessorCount,p.sharedMemPerBlockOptin,p.clockRate,p.totalGlobalMem>>20,p.l2CacheSize);
  int sms=p.multiProcessorCount; double* out; CK(cudaMalloc(&out,sizeof(double)*sms*1024*4));
  int iters=20000;
  for(int wps: {4,8,16,32}){
    int thr=wps*32;
    float ms=timeit([&]{k_dfma<<<sms,thr>>>(out,iters);});
    printf("DFMA   warps/SM %2d: %.2f TFLOP/s\n",wps, 2.0*8*iters*(double)sms*thr/ms/1e9);
    ms=timeit([&]{k_dmma<<<sms,thr>>>(out,iters);});
    printf("DMMA884 warps/SM %2d: %.2f TFLOP/s\n",wps, 2.0*256*8*iters*(double)sms*wps/ms/1e9);
    ms=timeit([&]{k_dmma1688<<<sms,thr>>>(out,iters);});
    printf("DMMA1688 warps/SM %2d: %.2f TFLOP/s\n",wps, 2.0*1024*4*iters*(double)sms*wps/ms/1e9);
    ms=timeit([&]{k_mixed<<<sms,thr>>>(out,iters);});
    printf("MIXED  warps/SM %2d: %.2f TFLOP/s (dmma+dfma equal flops)\n",wps, 2.0*(256*4+32*8*4)*iters*(double)sms*wps/ms/1e9);
    ms=timeit([&]{k_shfl<<<sms,thr>>>(out,iters);});
    printf("SHFL64 warps/SM %2d: %.2f warp-shfl64/clk/SM (at %d kHz)\n",wps, 4.0*iters*wps/(ms*1e-3*p.clockRate*1e3), p.clockRate);
    ms=timeit([&]{k_dsqrt<<<sms,thr>>>(out,iters/10);});
    printf("DSQRT  warps/SM %2d: %.1f clk per warp-sqrt per SM\n",wps, (ms*1e-3*p.clockRate*1e3)/(4.0*iters/10*wps));
    ms=timeit([&]{k_drcp<<<sms,thr>>>(out,iters/10);});
    printf("DRCP   warps/SM %2d: %.1f clk per warp-div per SM\n",wps, (ms*1e-3*p.clockRate*1e3)/(4.0*iters/10*wps));
    ms=timeit([&]{k_drsqrt<<<sms,thr>>>(out,iters/10);});
    printf("DRSQRT warps/SM %2d: %.1f clk per warp-rsqrt per SM\n",wps, (ms*1e-3*p.clockRate*1e3)/(4.0*iters/10*wps));
  }
  size_t bytes=(size_t)8<<30; double* x; CK(cudaMalloc(&x,bytes)); CK(cudaMemset(x,0,bytes));
  for(int mult: {2,4,8}) for(int thr: {256,512,1024}){
    float ms=timeit([&]{k_read<<<sms*mult,thr>>>((const double2*)x,bytes/16,out);});
    printf("READ LDG.128 grid %dxSM thr %4d: %.1f GB/s\n",mult,thr,bytes/ms/1e6);
  }
  for(int chunk: {8192,16384,32768}) for(int warps: {4,6,8,12}){
    size_t sm=(size_t)chunk*warps; if(sm>220*1024) continue;
    CK(cudaFuncSetAttribute(k_bulk,cudaFuncAttributeMaxDynamicSharedMemorySize,(int)sm));
    for(int cps: {1,2}){
      if(sm*cps>220*1024) continue;
      float ms=timeit([&]{k_bulk<<<sms*cps,warps*32,sm>>>(x,bytes/chunk,chunk,warps,out);});
      printf("READ BULK chunk %5d warps %2d ctas/SM %d: %.1f GB/s\n",chunk,warps,cps,bytes/ms/1e6);
    }
  }
  // copy bw for reference
  { float ms=timeit([&]{cudaMemcpyAsync(x,(char*)x+(bytes/2),bytes/2,cudaMemcpyDeviceToDevice);}); printf("D2D memcpy: %.1f GB/s (read+write)\n",bytes/ms/1e6); }
  // H2D pinned
  { size_t hb=(size_t)1<<30; void* h; CK(cudaMallocHost(&h,hb)); float ms=timeit([&]{cudaMemcpyAsync(x,h,hb,cudaMemcpyHostToDevice);},3); printf("H2D pinned: %.1f GB/s\n",hb/ms/1e6);
    ms=timeit([&]{cudaMemcpyAsync(h,x,hb,cudaMemcpyDeviceToHost);},3); printf("D2H pinned: %.1f GB/s\n",hb/ms/1e6); cudaFreeHost(h);}
  CK(cudaDeviceSynchronize());
  return 0;
}
