// Microbenchmark (not product code): Blackwell/Hopper asynchronous shared-memory
// reductions. red.async...add.u64 (SASS REDAS.ADD.64, native 64-bit integer add,
// completion tracked by an mbarrier transaction count) vs the 2 x u32 ATOMS.ADD
// carry scheme, random slots in a 16 KB shared array.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// shared::cluster address of this CTA's own shared variable
__device__ __forceinline__ uint32_t sc(const void* p) {
  uint32_t r;
  asm volatile("{\n .reg .u32 rk;\n mov.u32 rk, %%cluster_ctarank;\n mapa.shared::cluster.u32 %0, %1, rk;\n}\n"
               : "=r"(r) : "r"(sa(p)));
  return r;
}

__global__ void k(unsigned long long* out, int iters, int mode) {
  __shared__ unsigned long long s[2048];
  __shared__ __align__(8) unsigned long long bar;
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = 0;
  if (threadIdx.x == 0)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&bar)), "r"(blockDim.x) : "memory");
  __syncthreads();
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  if (mode == 0) {
    for (int it = 0; it < iters; ++it) {
      // the mbarrier transaction count is bounded (2^20 - 1): announce per batch
      if ((it & 15) == 0)
        asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(sa(&bar)), "r"(8 * 16) : "memory");
      const uint32_t h = hash32(tid * 2654435761u + it);
      asm volatile("red.async.relaxed.cluster.shared::cluster.mbarrier::complete_tx::bytes.add.u64 [%0], %1, [%2];"
                   ::"r"(sc(s + (h & 2047))), "l"((unsigned long long)(h >> 8)), "r"(sc(&bar)) : "memory");
    }
  } else {
    for (int it = 0; it < iters; ++it) {
      const uint32_t h = hash32(tid * 2654435761u + it);
      const unsigned long long q = h >> 8;
      uint32_t* p = reinterpret_cast<uint32_t*>(s + (h & 2047));
      const uint32_t lo = (uint32_t)q, hi = (uint32_t)(q >> 32);
      const uint32_t old = atomicAdd(p, lo);
      atomicAdd(p + 1, hi + ((old + lo < old) ? 1u : 0u));
    }
  }
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&bar)) : "memory");
  uint32_t ok = 0;
  while (!ok) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(sa(&bar)) : "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[0];
}

int main() {
  unsigned long long* o;
  cudaMalloc(&o, 1 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = 148 * 4, threads = 512, iters = 1024;  // iters % 16 == 0
  const char* nm[2] = {"red.async add.u64 (REDAS)", "2 x u32 ATOMS.ADD + carry"};
  for (int m = 0; m < 2; ++m) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = blocks;
    cfg.blockDim = threads;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, o, iters, m);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, k, o, iters, m);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double ops = (double)blocks * threads * iters;
    printf("%-28s %.3f ms  %.1f G u64-adds/s (%.2f /clk/SM)\n", nm[m], ms, ops / ms / 1e6, ops / ms / 1e6 / 148 / 1.965);
  }
  return 0;
}
