// Design probe 2 (not product code): shared-memory 128-bit CAS and 64-bit CAS throughput
// vs bank-conflict pattern, with 4 independent updates in flight per thread.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hsh(uint32_t x){ x^=x>>16; x*=0x7feb352dU; x^=x>>15; x*=0x846ca68bU; x^=x>>16; return x; }
__device__ __forceinline__ bool cas128(uint32_t addr, unsigned long long cl, unsigned long long ch, unsigned long long nl, unsigned long long nh, unsigned long long &ol, unsigned long long &oh){
  asm volatile("{\n .reg .b128 c, n, o;\n mov.b128 c, {%2,%3};\n mov.b128 n, {%4,%5};\n atom.shared.cas.b128 o, [%6], c, n;\n mov.b128 {%0,%1}, o;\n}" : "=l"(ol), "=l"(oh) : "l"(cl), "l"(ch), "l"(nl), "l"(nh), "r"(addr) : "memory");
  return ol==cl && oh==ch;
}
__device__ __forceinline__ void add2(double2* cell, double w){
  uint32_t a=(uint32_t)__cvta_generic_to_shared(cell); double2 cur=*cell;
  while(true){ unsigned long long ol,oh; if(cas128(a,__double_as_longlong(cur.x),__double_as_longlong(cur.y),__double_as_longlong(cur.x+w),__double_as_longlong(cur.y+w*w),ol,oh)) break; cur=make_double2(__longlong_as_double(ol),__longlong_as_double(oh)); }
}
// mode 0 random bins, 1 conflict-free (lane-distinct 16B bank groups within each 8-lane phase), 2 same bin per warp
template<int MODE>
__global__ void k_cas128(double* out, int nbins, int iters){
  extern __shared__ double2 s2[];
  for(int i=threadIdx.x;i<nbins;i+=blockDim.x) s2[i]=make_double2(0,0);
  __syncthreads();
  uint32_t st = hsh(blockIdx.x*blockDim.x+threadIdx.x);
  int lane=threadIdx.x&31;
  for(int it=0; it<iters; ++it){
    uint32_t b[4];
    #pragma unroll
    for(int u=0;u<4;++u){ st = st*1664525u+1013904223u;
      if(MODE==0) b[u]=__umulhi(st,nbins);
      else if(MODE==1) b[u]=((__umulhi(st,nbins/8))*8 + (lane&7)) % nbins;
      else b[u]=__shfl_sync(0xffffffff, __umulhi(st,nbins), 0); }
    #pragma unroll
    for(int u=0;u<4;++u) add2(&s2[b[u]], 1.0+(st&255)*(1.0/256));
  }
  __syncthreads();
  double acc=0; for(int i=threadIdx.x;i<nbins;i+=blockDim.x) acc+=s2[i].x+s2[i].y;
  atomicAdd(out, acc);
}
template<int MODE>
__global__ void k_cas64(double* out, int nbins, int iters){
  extern __shared__ double sd[];
  for(int i=threadIdx.x;i<2*nbins;i+=blockDim.x) sd[i]=0;
  __syncthreads();
  uint32_t st = hsh(blockIdx.x*blockDim.x+threadIdx.x);
  int lane=threadIdx.x&31;
  for(int it=0; it<iters; ++it){
    uint32_t b[4];
    #pragma unroll
    for(int u=0;u<4;++u){ st = st*1664525u+1013904223u;
      if(MODE==0) b[u]=__umulhi(st,nbins);
      else if(MODE==1) b[u]=((__umulhi(st,nbins/16))*16 + (lane&15)) % nbins;
      else b[u]=__shfl_sync(0xffffffff, __umulhi(st,nbins), 0); }
    #pragma unroll
    for(int u=0;u<4;++u){ double w=1.0+(st&255)*(1.0/256); atomicAdd(&sd[2*b[u]], w); atomicAdd(&sd[2*b[u]+1], w*w);} 
  }
  __syncthreads();
  double acc=0; for(int i=threadIdx.x;i<2*nbins;i+=blockDim.x) acc+=sd[i];
  atomicAdd(out, acc);
}
// plain LDS.128 + STS.128 (non-atomic RMW), for comparison
template<int MODE>
__global__ void k_rmw128(double* out, int nbins, int iters){
  extern __shared__ double2 s2[];
  for(int i=threadIdx.x;i<nbins;i+=blockDim.x) s2[i]=make_double2(0,0);
  __syncthreads();
  uint32_t st = hsh(blockIdx.x*blockDim.x+threadIdx.x);
  int lane=threadIdx.x&31;
  for(int it=0; it<iters; ++it){
    uint32_t b[4];
    #pragma unroll
    for(int u=0;u<4;++u){ st = st*1664525u+1013904223u;
      if(MODE==0) b[u]=__umulhi(st,nbins);
      else b[u]=((__umulhi(st,nbins/8))*8 + (lane&7)) % nbins; }
    #pragma unroll
    for(int u=0;u<4;++u){ double w=1.0+(st&255)*(1.0/256); double2 v=s2[b[u]]; v.x+=w; v.y+=w*w; s2[b[u]]=v; }
  }
  __syncthreads();
  double acc=0; for(int i=threadIdx.x;i<nbins;i+=blockDim.x) acc+=s2[i].x+s2[i].y;
  atomicAdd(out, acc);
}
__global__ void k_atoms_u32x4(unsigned long long* out, int nbins, int iters){
  extern __shared__ uint32_t s[];
  for(int i=threadIdx.x;i<nbins;i+=blockDim.x) s[i]=0;
  __syncthreads();
  uint32_t st = hsh(blockIdx.x*blockDim.x+threadIdx.x);
  for(int it=0; it<iters; ++it){ 
    #pragma unroll
    for(int u=0;u<4;++u){ st = st*1664525u+1013904223u; atomicAdd(&s[__umulhi(st,nbins)], st>>20); } }
  __syncthreads();
  unsigned long long acc=0; for(int i=threadIdx.x;i<nbins;i+=blockDim.x) acc+=s[i];
  atomicAdd(out, acc);
}
int main(){
  int nsm=148; void* dout; cudaMalloc(&dout, 1<<20);
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  auto T=[&](const char* nm, double ops, auto L){ L(); cudaDeviceSynchronize(); cudaEventRecord(a); L(); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
    printf("%-44s %8.3f ms %8.2f Gop/s %.3f op/clk/SM %s\n", nm, ms, ops/ms/1e6, ops/(ms*1e-3)/nsm/1.965e9, cudaGetErrorString(cudaGetLastError())); };
  int nb=10002, it=512; 
  cudaFuncSetAttribute(k_cas128<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200*1024);
  cudaFuncSetAttribute(k_cas128<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200*1024);
  cudaFuncSetAttribute(k_cas128<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200*1024);
  cudaFuncSetAttribute(k_cas64<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200*1024);
  cudaFuncSetAttribute(k_cas64<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200*1024);
  cudaFuncSetAttribute(k_rmw128<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200*1024);
  cudaFuncSetAttribute(k_rmw128<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200*1024);
  for(int thr: {512,1024}){ double ops=(double)nsm*thr*it*4; char nm[64];
    snprintf(nm,64,"cas128 random thr%d",thr); T(nm,ops,[&]{k_cas128<0><<<nsm,thr,nb*16>>>((double*)dout,nb,it);});
    snprintf(nm,64,"cas128 conflict-free thr%d",thr); T(nm,ops,[&]{k_cas128<1><<<nsm,thr,nb*16>>>((double*)dout,nb,it);});
    snprintf(nm,64,"cas128 same-bin-per-warp thr%d",thr); T(nm,ops/8,[&]{k_cas128<2><<<nsm,thr,nb*16>>>((double*)dout,nb,it/8);});
    snprintf(nm,64,"cas64x2 random thr%d",thr); T(nm,ops,[&]{k_cas64<0><<<nsm,thr,nb*16>>>((double*)dout,nb,it);});
    snprintf(nm,64,"cas64x2 conflict-free thr%d",thr); T(nm,ops,[&]{k_cas64<1><<<nsm,thr,nb*16>>>((double*)dout,nb,it);});
    snprintf(nm,64,"rmw128 (non-atomic) random thr%d",thr); T(nm,ops,[&]{k_rmw128<0><<<nsm,thr,nb*16>>>((double*)dout,nb,it);});
    snprintf(nm,64,"rmw128 (non-atomic) conflict-free thr%d",thr); T(nm,ops,[&]{k_rmw128<1><<<nsm,thr,nb*16>>>((double*)dout,nb,it);});
    snprintf(nm,64,"atoms u32 x4 random thr%d",thr); T(nm,ops,[&]{k_atoms_u32x4<<<nsm,thr,nb*16>>>((unsigned long long*)dout,nb*4,it);});
  }
}
