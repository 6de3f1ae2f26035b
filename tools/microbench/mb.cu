// Design-probe microbenchmarks (not product code): smem/global atomic rates and
// read-only HBM streaming on B200. Results feed DESIGN.md kernel choices.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__device__ __forceinline__ uint32_t hsh(uint32_t x){ x^=x>>16; x*=0x7feb352dU; x^=x>>15; x*=0x846ca68bU; x^=x>>16; return x; }

template<int REPL>
__global__ void k_atoms_u32(unsigned long long* out, int nbins, int iters){
  extern __shared__ uint32_t s[];
  int tot = nbins*REPL;
  for(int i=threadIdx.x;i<tot;i+=blockDim.x) s[i]=0;
  __syncthreads();
  uint32_t st = hsh(blockIdx.x*blockDim.x+threadIdx.x);
  int rep = (REPL==1)?0:((threadIdx.x>>5)%REPL);
  uint32_t* my = s + rep*nbins;
  for(int it=0; it<iters; ++it){ st = st*1664525u+1013904223u; uint32_t b = __umulhi(st, nbins); atomicAdd(&my[b], 1u); }
  __syncthreads();
  unsigned long long acc=0; for(int i=threadIdx.x;i<tot;i+=blockDim.x) acc+=s[i];
  atomicAdd(out, acc);
}
__global__ void k_cas64x2(double* out, int nbins, int iters){
  extern __shared__ double sd[];
  for(int i=threadIdx.x;i<2*nbins;i+=blockDim.x) sd[i]=0;
  __syncthreads();
  uint32_t st = hsh(blockIdx.x*blockDim.x+threadIdx.x);
  for(int it=0; it<iters; ++it){ st = st*1664525u+1013904223u; uint32_t b = __umulhi(st, nbins); double w = 1.0+(st&255)*(1.0/256);
    atomicAdd(&sd[b], w); atomicAdd(&sd[nbins+b], w*w); }
  __syncthreads();
  double acc=0; for(int i=threadIdx.x;i<2*nbins;i+=blockDim.x) acc+=sd[i];
  atomicAdd(out, acc);
}
__device__ __forceinline__ bool cas128(unsigned addr, unsigned long long cl, unsigned long long ch, unsigned long long nl, unsigned long long nh, unsigned long long &ol, unsigned long long &oh){
  asm volatile("{\n .reg .b128 c, n, o;\n mov.b128 c, {%2,%3};\n mov.b128 n, {%4,%5};\n atom.shared.cas.b128 o, [%6], c, n;\n mov.b128 {%0,%1}, o;\n}" : "=l"(ol), "=l"(oh) : "l"(cl), "l"(ch), "l"(nl), "l"(nh), "r"(addr) : "memory");
  return ol==cl && oh==ch;
}
__global__ void k_cas128(double* out, int nbins, int iters){
  extern __shared__ double2 s2[];
  for(int i=threadIdx.x;i<nbins;i+=blockDim.x) s2[i]=make_double2(0,0);
  __syncthreads();
  uint32_t st = hsh(blockIdx.x*blockDim.x+threadIdx.x);
  for(int it=0; it<iters; ++it){ st = st*1664525u+1013904223u; uint32_t b = __umulhi(st, nbins); double w = 1.0+(st&255)*(1.0/256);
    unsigned a = (unsigned)__cvta_generic_to_shared(&s2[b]);
    double2 cur = s2[b];
    while(true){ unsigned long long ol,oh; double nx=cur.x+w, ny=cur.y+w*w;
      if(cas128(a,__double_as_longlong(cur.x),__double_as_longlong(cur.y),__double_as_longlong(nx),__double_as_longlong(ny),ol,oh)) break;
      cur=make_double2(__longlong_as_double(ol),__longlong_as_double(oh)); }
  }
  __syncthreads();
  double acc=0; for(int i=threadIdx.x;i<nbins;i+=blockDim.x) acc+=s2[i].x+s2[i].y;
  atomicAdd(out, acc);
}
// per-thread private u32 columns [bin][thread] (no atomics)
__global__ void k_private(unsigned long long* out, int nbins, int iters){
  extern __shared__ uint32_t s[];
  for(int i=threadIdx.x;i<nbins*blockDim.x;i+=blockDim.x) s[i]=0;
  __syncthreads();
  uint32_t st = hsh(blockIdx.x*blockDim.x+threadIdx.x);
  for(int it=0; it<iters; ++it){ st = st*1664525u+1013904223u; uint32_t b = __umulhi(st, nbins); s[b*blockDim.x+threadIdx.x]++; }
  __syncthreads();
  unsigned long long acc=0; for(int i=threadIdx.x;i<nbins*blockDim.x;i+=blockDim.x) acc+=s[i];
  atomicAdd(out, acc);
}
__global__ void k_red_f64(double* h, int nbins, int iters){
  uint32_t st = hsh(blockIdx.x*blockDim.x+threadIdx.x);
  for(int it=0; it<iters; ++it){ st = st*1664525u+1013904223u; uint32_t b = __umulhi(st, nbins); double w = 1.0+(st&255)*(1.0/256);
    atomicAdd(&h[b], w); atomicAdd(&h[nbins+b], w*w); }
}
__global__ void k_red_u64(unsigned long long* h, int nbins, int iters){
  uint32_t st = hsh(blockIdx.x*blockDim.x+threadIdx.x);
  for(int it=0; it<iters; ++it){ st = st*1664525u+1013904223u; uint32_t b = __umulhi(st, nbins); atomicAdd(&h[b], 1ull); }
}
__global__ void k_red_u32(unsigned* h, int nbins, int iters){
  uint32_t st = hsh(blockIdx.x*blockDim.x+threadIdx.x);
  for(int it=0; it<iters; ++it){ st = st*1664525u+1013904223u; uint32_t b = __umulhi(st, nbins); atomicAdd(&h[b], 1u); }
}
__global__ void k_stream(const double2* __restrict__ x, size_t n2, double* out){
  double acc=0; size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x, stride=(size_t)gridDim.x*blockDim.x;
  #pragma unroll 4
  for(; i<n2; i+=stride){ double2 v = __ldcs(&x[i]); acc += v.x+v.y; }
  if(acc==12345.678) out[0]=acc;
}
__global__ void k_stream_u4(const double2* __restrict__ x, size_t n2, double* out){
  // each thread 4 independent double2 per iteration
  double acc=0; size_t stride=(size_t)gridDim.x*blockDim.x;
  size_t i = blockIdx.x*(size_t)blockDim.x+threadIdx.x;
  for(; i+3*stride<n2; i+=4*stride){ double2 a=__ldcs(&x[i]),b=__ldcs(&x[i+stride]),c=__ldcs(&x[i+2*stride]),d=__ldcs(&x[i+3*stride]); acc+=a.x+b.x+c.x+d.x+a.y+b.y+c.y+d.y; }
  for(; i<n2; i+=stride){ double2 v=__ldcs(&x[i]); acc+=v.x+v.y; }
  if(acc==12345.678) out[0]=acc;
}

int main(){
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,0));
  printf("dev %s SMs %d L2 %d MB smemOptin %zu clock %d\n", p.name, p.multiProcessorCount, p.l2CacheSize>>20, p.sharedMemPerBlockOptin, p.clockRate);
  int nsm = p.multiProcessorCount;
  void* dout; CK(cudaMalloc(&dout, 1<<20));
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  auto T = [&](const char* name, double ops, auto launch){ launch(); cudaDeviceSynchronize(); cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
     cudaError_t e = cudaGetLastError(); printf("%-40s %8.3f ms  %8.2f Gop/s  (%.3f op/clk/SM @1.9GHz) %s\n", name, ms, ops/ms/1e6, ops/(ms*1e-3)/nsm/1.9e9, e==cudaSuccess?"":cudaGetErrorString(e)); };
  int iters=2048;
  for (int thr : {256, 512, 1024}) {
    int blocks = nsm * (2048/thr);
    double ops = (double)blocks*thr*iters;
    char nm[64];
    snprintf(nm,64,"atoms_u32 102 bins R1 thr%d",thr); T(nm, ops, [&]{ k_atoms_u32<1><<<blocks,thr,102*4>>>((unsigned long long*)dout,102,iters); });
    snprintf(nm,64,"atoms_u32 102 bins R8 thr%d",thr); T(nm, ops, [&]{ k_atoms_u32<8><<<blocks,thr,102*4*8>>>((unsigned long long*)dout,102,iters); });
    snprintf(nm,64,"atoms_u32 10002 bins R1 thr%d",thr); T(nm, ops, [&]{ k_atoms_u32<1><<<blocks,thr,10002*4>>>((unsigned long long*)dout,10002,iters); });
  }
  cudaFuncSetAttribute(k_cas64x2, cudaFuncAttributeMaxDynamicSharedMemorySize, 200*1024);
  cudaFuncSetAttribute(k_cas128, cudaFuncAttributeMaxDynamicSharedMemorySize, 200*1024);
  cudaFuncSetAttribute(k_private, cudaFuncAttributeMaxDynamicSharedMemorySize, 200*1024);
  for (int thr : {512, 1024}) {
    int blocks = nsm; double ops=(double)blocks*thr*iters; char nm[64];
    snprintf(nm,64,"cas64x2 10002 bins thr%d (events)",thr); T(nm, ops, [&]{ k_cas64x2<<<blocks,thr,10002*16>>>((double*)dout,10002,iters); });
    snprintf(nm,64,"cas128 10002 bins thr%d (events)",thr); T(nm, ops, [&]{ k_cas128<<<blocks,thr,10002*16>>>((double*)dout,10002,iters); });
    snprintf(nm,64,"cas128 102 bins thr%d (events)",thr); T(nm, ops, [&]{ k_cas128<<<blocks,thr,102*16>>>((double*)dout,102,iters); });
  }
  { int thr=256; int blocks=nsm*1; double ops=(double)blocks*thr*iters; T("private u32 102 bins thr256 1cta/sm", ops, [&]{ k_private<<<blocks,thr,102*256*4>>>((unsigned long long*)dout,102,iters); });
    blocks=nsm*2; ops=(double)blocks*thr*iters; T("private u32 102 bins thr256 2cta/sm", ops, [&]{ k_private<<<blocks,thr,102*256*4>>>((unsigned long long*)dout,102,iters); }); }
  void* dh; CK(cudaMalloc(&dh, 64<<20)); cudaMemset(dh,0,64<<20);
  { int thr=512, blocks=nsm*4; double ops=(double)blocks*thr*iters;
    T("red_f64x2 10002 bins (events)", ops, [&]{ k_red_f64<<<blocks,thr>>>((double*)dh,10002,iters); });
    T("red_u64 1004004 bins", ops, [&]{ k_red_u64<<<blocks,thr>>>((unsigned long long*)dh,1004004,iters); });
    T("red_u32 1004004 bins", ops, [&]{ k_red_u32<<<blocks,thr>>>((unsigned*)dh,1004004,iters); });
    T("red_u64 8 bins (hot)", ops/16, [&]{ k_red_u64<<<blocks,thr>>>((unsigned long long*)dh,8,iters/16); });
    T("red_u64 1061208 bins", ops, [&]{ k_red_u64<<<blocks,thr>>>((unsigned long long*)dh,1061208,iters); });
  }
  size_t nbytes = (size_t)8<<30; void* dx; CK(cudaMalloc(&dx, nbytes)); cudaMemset(dx,0,nbytes);
  for (int thr : {256, 512, 1024}) for (int per : {1,2,4,8}) {
    int blocks = nsm*per*(1024/thr); char nm[64];
    snprintf(nm,64,"stream LDG128 thr%d blocks%d (GB/s=Gop*16)",thr,blocks);
    T(nm, nbytes/16.0, [&]{ k_stream<<<blocks,thr>>>((const double2*)dx, nbytes/16, (double*)dout); });
    snprintf(nm,64,"stream_u4 thr%d blocks%d",thr,blocks);
    T(nm, nbytes/16.0, [&]{ k_stream_u4<<<blocks,thr>>>((const double2*)dx, nbytes/16, (double*)dout); });
  }
  return 0;
}
