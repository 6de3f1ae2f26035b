// Design probe 4 (not product code): ways to accumulate (w, w^2) into 10,002 float64 pairs in
// shared memory from random bins, one update per thread per iteration (like k_fill's sink):
//   cas   : LDS.128 of the cell, then ATOMS.CAS.128 retry loop (round-1 PRIV weighted sink)
//   exch  : take-and-return with ATOMS.EXCH.128 (take the cell's pair, leave (0,0); return the
//           sum; if the return brought back a deposit made meanwhile, take again and repeat)
//   rmw   : non-atomic LDS.128 + STS.128 (wrong under races; the pipe's floor)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb4 mb4.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hsh(uint32_t x){ x^=x>>16; x*=0x7feb352dU; x^=x>>15; x*=0x846ca68bU; x^=x>>16; return x; }
__device__ __forceinline__ void exch128(uint32_t a, unsigned long long il, unsigned long long ih,
                                        unsigned long long &ol, unsigned long long &oh){
  asm volatile("{ .reg .b128 d, z; mov.b128 z, {%2,%3}; atom.shared.exch.b128 d, [%4], z; mov.b128 {%0,%1}, d; }"
               : "=l"(ol), "=l"(oh) : "l"(il), "l"(ih), "r"(a) : "memory");
}
__device__ __forceinline__ bool cas128(uint32_t addr, unsigned long long cl, unsigned long long ch, unsigned long long nl,
                                       unsigned long long nh, unsigned long long &ol, unsigned long long &oh){
  asm volatile("{ .reg .b128 c, n, o; mov.b128 c, {%2,%3}; mov.b128 n, {%4,%5}; atom.shared.cas.b128 o, [%6], c, n;"
               " mov.b128 {%0,%1}, o; }" : "=l"(ol), "=l"(oh) : "l"(cl), "l"(ch), "l"(nl), "l"(nh), "r"(addr) : "memory");
  return ol==cl && oh==ch;
}
template<int MODE>
__device__ __forceinline__ void add(double2* cell, double w){
  uint32_t a=(uint32_t)__cvta_generic_to_shared(cell);
  if (MODE == 0) {
    double2 cur=*cell;
    while(true){ unsigned long long ol,oh;
      if(cas128(a,__double_as_longlong(cur.x),__double_as_longlong(cur.y),__double_as_longlong(cur.x+w),__double_as_longlong(cur.y+w*w),ol,oh)) break;
      cur=make_double2(__longlong_as_double(ol),__longlong_as_double(oh)); }
  } else if (MODE == 1) {
    unsigned long long l, h;
    exch128(a, 0ull, 0ull, l, h);
    double sx = __longlong_as_double(l) + w, sy = __longlong_as_double(h) + w*w;
    while (true) {
      exch128(a, __double_as_longlong(sx), __double_as_longlong(sy), l, h);
      if ((l | h) == 0) break;
      unsigned long long l2, h2;
      exch128(a, 0ull, 0ull, l2, h2);
      sx = __longlong_as_double(l) + __longlong_as_double(l2); sy = __longlong_as_double(h) + __longlong_as_double(h2);
    }
  } else {
    double2 v=*cell; v.x+=w; v.y+=w*w; *cell=v;
  }
}
template<int MODE>
__global__ void __launch_bounds__(1024, 1) k_sink(double* out, int nbins, int iters, int hot){
  extern __shared__ double2 s2[];
  for(int i=threadIdx.x;i<nbins;i+=blockDim.x) s2[i]=make_double2(0,0);
  __syncthreads();
  uint32_t st = hsh(blockIdx.x*blockDim.x+threadIdx.x);
  for(int it=0; it<iters; ++it){
    st = st*1664525u+1013904223u;
    uint32_t b = __umulhi(st, nbins);
    if (hot && (st & 0xff) < (uint32_t)hot) b = 17;       // hot/256 of the events in one bin
    add<MODE>(&s2[b], 1.0+(st>>24)*(1.0/256));
  }
  __syncthreads();
  double acc=0; for(int i=threadIdx.x;i<nbins;i+=blockDim.x) acc+=s2[i].x+s2[i].y;
  atomicAdd(out, acc);
}
int main(){
  int nsm=148; double* dout; cudaMalloc(&dout, 8);
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  int nb=10002, it=2048, thr=1024;
  cudaFuncSetAttribute(k_sink<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200*1024);
  cudaFuncSetAttribute(k_sink<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200*1024);
  cudaFuncSetAttribute(k_sink<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200*1024);
  const char* names[3] = {"cas (LDS.128 + CAS.128)", "exch (2x EXCH.128)", "rmw (non-atomic)"};
  for (int hot : {0, 8, 64}) for (int m = 0; m < 3; ++m) {
    double ops=(double)nsm*thr*it; double exact = 0;
    auto L = [&]{ cudaMemset(dout, 0, 8);
      if (m==0) k_sink<0><<<nsm,thr,nb*16>>>(dout,nb,it,hot);
      else if (m==1) k_sink<1><<<nsm,thr,nb*16>>>(dout,nb,it,hot);
      else k_sink<2><<<nsm,thr,nb*16>>>(dout,nb,it,hot); };
    L(); cudaDeviceSynchronize(); cudaEventRecord(a); L(); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);
    double r; cudaMemcpy(&r, dout, 8, cudaMemcpyDeviceToHost);
    if (m==0) exact = r;
    printf("hot %3d/256  %-26s %8.3f ms %8.2f Gupd/s %.3f upd/clk/SM  checksum %.17g %s\n", hot, names[m], ms, ops/ms/1e6,
           ops/(ms*1e-3)/nsm/1.965e9, r, cudaGetErrorString(cudaGetLastError()));
  }
}
