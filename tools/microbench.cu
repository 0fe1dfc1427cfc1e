// Primitive-throughput probes used to pick the GEE kernel design (not product code).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s line %d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

__device__ __forceinline__ uint32_t mix(uint32_t x){ x^=x>>16; x*=0x7feb352dU; x^=x>>15; x*=0x846ca68bU; x^=x>>16; return x; }

template<int MODE>
__global__ void smem_atomic(int iters, unsigned long long* sink){
  extern __shared__ unsigned char sm[];
  uint32_t* s32=(uint32_t*)sm; unsigned long long* s64=(unsigned long long*)sm; float* sf=(float*)sm;
  for(int i=threadIdx.x;i<16384;i+=blockDim.x) s32[i]=0;
  __syncthreads();
  uint32_t h=mix(threadIdx.x+blockIdx.x*977);
  for(int i=0;i<iters;i++){
    h=h*1664525u+1013904223u;
    uint32_t a=h>>18; // 14 bits
    if(MODE==0) atomicAdd(&s32[a],1u);
    else if(MODE==1) atomicAdd(&s64[a>>1],(unsigned long long)h);
    else if(MODE==2) atomicAdd(&sf[a],1.0f);
    else if(MODE==3) { s32[a]+=1u; }
    else if(MODE==4) { atomicAdd(&s32[a],h&15u);} // general u32 add
  }
  __syncthreads();
  if(threadIdx.x==0) atomicAdd(sink,(unsigned long long)s32[5]);
}

__global__ void gather_u8(const uint8_t* __restrict__ lab, uint64_t n, int iters, unsigned long long* sink){
  uint32_t h=mix(threadIdx.x+blockIdx.x*blockDim.x);
  uint32_t acc=0;
  #pragma unroll 8
  for(int i=0;i<iters;i++){ h=mix(h+i); uint64_t idx=((uint64_t)h* n)>>32; acc+=__ldg(lab+idx);}
  if(acc==0x12345) atomicAdd(sink,1ull);
}
__global__ void gather_i32(const int* __restrict__ lab, uint64_t n, int iters, unsigned long long* sink){
  uint32_t h=mix(threadIdx.x+blockIdx.x*blockDim.x);
  uint32_t acc=0;
  #pragma unroll 8
  for(int i=0;i<iters;i++){ h=mix(h+i); uint64_t idx=((uint64_t)h* n)>>32; acc+=__ldg(lab+idx);}
  if(acc==0x12345) atomicAdd(sink,1ull);
}
__global__ void red_f32(float* z, uint64_t n, int iters){
  uint32_t h=mix(threadIdx.x+blockIdx.x*blockDim.x);
  #pragma unroll 4
  for(int i=0;i<iters;i++){ h=mix(h+i); uint64_t a=((uint64_t)h*(uint64_t)(n>>6))>>32; uint64_t idx=(a<<6)|(mix(h)&63); atomicAdd(z+idx,0.5f);}
}
__global__ void stream_read(const int4* __restrict__ p, uint64_t n4, unsigned long long* sink){
  int4 acc=make_int4(0,0,0,0);
  for(uint64_t i=blockIdx.x*(uint64_t)blockDim.x+threadIdx.x;i<n4;i+=(uint64_t)gridDim.x*blockDim.x){int4 v=__ldg(p+i); acc.x^=v.x;acc.y^=v.y;acc.z^=v.z;acc.w^=v.w;}
  if((acc.x^acc.y^acc.z^acc.w)==0x1234567) atomicAdd(sink,1ull);
}
__global__ void stream_write(int4* p, uint64_t n4){
  for(uint64_t i=blockIdx.x*(uint64_t)blockDim.x+threadIdx.x;i<n4;i+=(uint64_t)gridDim.x*blockDim.x) p[i]=make_int4(1,2,3,4);
}
__global__ void match_any_k(int iters, unsigned long long* sink){
  uint32_t h=mix(threadIdx.x+blockIdx.x*blockDim.x); uint32_t acc=0;
  for(int i=0;i<iters;i++){ h=h*1664525u+1013904223u; acc+=__match_any_sync(0xffffffffu,h>>26);} 
  if(acc==0x12345) atomicAdd(sink,1ull);
}

int main(){
  int sms; cudaDeviceGetAttribute(&sms,cudaDevAttrMultiProcessorCount,0);
  int l2; cudaDeviceGetAttribute(&l2,cudaDevAttrL2CacheSize,0);
  int clk; cudaDeviceGetAttribute(&clk,cudaDevAttrClockRate,0);
  printf("SMs %d L2 %d B clock %d kHz\n",sms,l2,clk);
  unsigned long long* sink; CK(cudaMalloc(&sink,8));
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  const char* names[]={"smem atomicAdd u32","smem atomicAdd u64","smem atomicAdd f32","smem plain RMW u32","smem atomicAdd u32 general value"};
  for(int mode=0;mode<5;mode++){
    for(int cps: {2,4}){
      int iters=4096; int blocks=sms*cps; size_t sh=65536;
      void* k = mode==0?(void*)smem_atomic<0>:mode==1?(void*)smem_atomic<1>:mode==2?(void*)smem_atomic<2>:mode==3?(void*)smem_atomic<3>:(void*)smem_atomic<4>;
      CK(cudaFuncSetAttribute(k,cudaFuncAttributeMaxDynamicSharedMemorySize,(int)sh));
      for(int rep=0;rep<2;rep++){
      cudaEventRecord(a);
      if(mode==0) smem_atomic<0><<<blocks,256,sh>>>(iters,sink);
      if(mode==1) smem_atomic<1><<<blocks,256,sh>>>(iters,sink);
      if(mode==2) smem_atomic<2><<<blocks,256,sh>>>(iters,sink);
      if(mode==3) smem_atomic<3><<<blocks,256,sh>>>(iters,sink);
      if(mode==4) smem_atomic<4><<<blocks,256,sh>>>(iters,sink);
      cudaEventRecord(b); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms,a,b);}
      double ops=(double)blocks*256*iters;
      printf("%s (%d CTA/SM): %.1f Gop/s = %.2f op/clk/SM\n",names[mode],cps,ops/ms/1e6, ops/(ms*1e-3)/sms/(clk*1e3));
    }
  }
  // gathers
  uint64_t big=(uint64_t)1<<30; uint8_t* buf; CK(cudaMalloc(&buf,big*4)); CK(cudaMemset(buf,1,big*4));
  for(uint64_t n: {(uint64_t)16<<20,(uint64_t)64<<20,(uint64_t)100<<20,(uint64_t)134217728,(uint64_t)512<<20}){
    int iters=256; int blocks=sms*8;
    for(int rep=0;rep<2;rep++){cudaEventRecord(a); gather_u8<<<blocks,256>>>(buf,n,iters,sink); cudaEventRecord(b); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms,a,b);}
    double ops=(double)blocks*256*iters;
    printf("gather u8 over %llu MB: %.1f G/s\n",(unsigned long long)(n>>20),ops/ms/1e6);
  }
  for(uint64_t n: {(uint64_t)4<<20,(uint64_t)16<<20,(uint64_t)134217728}){
    int iters=256; int blocks=sms*8;
    for(int rep=0;rep<2;rep++){cudaEventRecord(a); gather_i32<<<blocks,256>>>((int*)buf,n,iters,sink); cudaEventRecord(b); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms,a,b);}
    double ops=(double)blocks*256*iters;
    printf("gather i32 over %llu MB: %.1f G/s\n",(unsigned long long)(n*4>>20),ops/ms/1e6);
  }
  // stream
  uint64_t n4=(big*4)/16;
  for(int rep=0;rep<3;rep++){cudaEventRecord(a); stream_read<<<sms*8,512>>>((int4*)buf,n4,sink); cudaEventRecord(b); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms,a,b);}
  printf("stream read 4GB: %.1f GB/s\n",big*4/ms/1e6);
  for(int rep=0;rep<3;rep++){cudaEventRecord(a); stream_write<<<sms*8,512>>>((int4*)buf,n4); cudaEventRecord(b); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms,a,b);}
  printf("stream write 4GB: %.1f GB/s\n",big*4/ms/1e6);
  for(int rep=0;rep<3;rep++){cudaEventRecord(a); cudaMemsetAsync(buf,0,big*4); cudaEventRecord(b); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms,a,b);}
  printf("memset 4GB: %.1f GB/s\n",big*4/ms/1e6);
  CK(cudaFree(buf));
  // red.global
  for(uint64_t bytes: {(uint64_t)64<<20,(uint64_t)200<<20,(uint64_t)4<<30,(uint64_t)26<<30}){
    float* z; CK(cudaMalloc(&z,bytes)); CK(cudaMemset(z,0,bytes)); uint64_t n=bytes/4; int iters=64; int blocks=sms*8;
    for(int rep=0;rep<2;rep++){cudaEventRecord(a); red_f32<<<blocks,256>>>(z,n,iters); cudaEventRecord(b); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms,a,b);}
    double ops=(double)blocks*256*iters;
    printf("red.f32 random over %llu MB: %.1f G/s\n",(unsigned long long)(bytes>>20),ops/ms/1e6);
    CK(cudaFree(z));
  }
  for(int rep=0;rep<2;rep++){cudaEventRecord(a); match_any_k<<<sms*8,256>>>(4096,sink); cudaEventRecord(b); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms,a,b);}
  printf("match_any: %.1f G warp-ops/s\n",(double)sms*8*8*4096/ms/1e6);
  CK(cudaDeviceSynchronize());
  printf("done\n");
  return 0;
}
