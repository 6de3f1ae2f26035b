// Design probe 3 (not product code): global RED.64 throughput on a 1M-bin (8 MB) array,
// alone and interleaved with a streaming read (the C3 fill pattern).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hsh(uint32_t x){ x^=x>>16; x*=0x7feb352dU; x^=x>>15; x*=0x846ca68bU; x^=x>>16; return x; }
template<int K>
__global__ void k_red(unsigned long long* h, int nbins, int iters){
  uint32_t st = hsh(blockIdx.x*blockDim.x+threadIdx.x);
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int k=0;k<K;++k){ st = st*1664525u+1013904223u; atomicAdd(&h[__umulhi(st, nbins)], 1ull); }
  }
}
// stream x (double2) and do one RED per element with bin from x
__global__ void k_stream_red(const double2* __restrict__ x, long n2, unsigned long long* h, int nbins){
  long stride=(long)gridDim.x*blockDim.x;
  for(long i=blockIdx.x*(long)blockDim.x+threadIdx.x; i<n2; i+=stride){
    double2 v=__ldcs(&x[i]);
    atomicAdd(&h[(int)(v.x*nbins)], 1ull);
    atomicAdd(&h[(int)(v.y*nbins)], 1ull);
  }
}
__global__ void k_stream_red2(const double2* __restrict__ x, long n2, unsigned long long* h, int nbins){
  long stride=(long)gridDim.x*blockDim.x;
  long i=blockIdx.x*(long)blockDim.x+threadIdx.x;
  for(; i+3*stride<n2; i+=4*stride){
    double2 a=__ldcs(&x[i]), b=__ldcs(&x[i+stride]), c=__ldcs(&x[i+2*stride]), d=__ldcs(&x[i+3*stride]);
    atomicAdd(&h[(int)(a.x*nbins)], 1ull); atomicAdd(&h[(int)(a.y*nbins)], 1ull);
    atomicAdd(&h[(int)(b.x*nbins)], 1ull); atomicAdd(&h[(int)(b.y*nbins)], 1ull);
    atomicAdd(&h[(int)(c.x*nbins)], 1ull); atomicAdd(&h[(int)(c.y*nbins)], 1ull);
    atomicAdd(&h[(int)(d.x*nbins)], 1ull); atomicAdd(&h[(int)(d.y*nbins)], 1ull);
  }
  for(; i<n2; i+=stride){ double2 v=__ldcs(&x[i]); atomicAdd(&h[(int)(v.x*nbins)], 1ull); atomicAdd(&h[(int)(v.y*nbins)], 1ull); }
}
__global__ void k_fill_uniform(double* x, long n){ long i=blockIdx.x*(long)blockDim.x+threadIdx.x; if(i<n) x[i]=(hsh((uint32_t)i)^hsh((uint32_t)(i>>32)+7))*(1.0/4294967296.0); }
int main(){
  int nsm=148; unsigned long long* h; cudaMalloc(&h, 64<<20); cudaMemset(h,0,64<<20);
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  auto T=[&](const char* nm, double ops, auto L){ L(); cudaDeviceSynchronize(); cudaEventRecord(a); L(); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
    printf("%-52s %8.3f ms %8.2f Gop/s %s\n", nm, ms, ops/ms/1e6, cudaGetErrorString(cudaGetLastError())); };
  int nb=1004004;
  for(int thr: {256,512,1024}) for(int per: {1,2,4,8}) { int blocks=nsm*per*(1024/thr)/ (thr==1024?1:1); char nm[80];
    if ((long)blocks*thr > 148*2048*2) continue;
    snprintf(nm,80,"red u64 K=4 thr%d blocks%d",thr,blocks); double ops=(double)blocks*thr*256*4; T(nm,ops,[&]{k_red<4><<<blocks,thr>>>(h,nb,256);}); }
  long n=(long)1<<28; double* x; cudaMalloc(&x, n*8); k_fill_uniform<<<(n+255)/256,256>>>(x,n); cudaDeviceSynchronize();
  for(int thr: {256,512,1024}) for(int per: {1,2,4}) { int blocks=nsm*per*(1024/thr); if ((long)blocks*thr > 148*2048*4) continue; char nm[80];
    snprintf(nm,80,"stream+red thr%d blocks%d (events/s)",thr,blocks); T(nm,(double)n,[&]{k_stream_red<<<blocks,thr>>>((const double2*)x,n/2,h,1000000);});
    snprintf(nm,80,"stream+red unroll4 thr%d blocks%d (events/s)",thr,blocks); T(nm,(double)n,[&]{k_stream_red2<<<blocks,thr>>>((const double2*)x,n/2,h,1000000);}); }
}
