// Microbenchmark (not product code): exact 64-bit fixed-point shared-memory adds,
// plain (each lane: ATOMS lo with return + carry into hi) vs warp-aggregated
// (__match_any_sync on the pixel, __reduce_add_sync of three 22-bit chunks per
// peer group, one fixed-point add per distinct pixel). Lanes draw pixels from a
// window of A pixels of a 32x16 tile (row stride 40 words): A = 80 ~ the random
// pixels of one 8x8 sort tile (time order), A = 10 ~ spatially ordered events.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
constexpr int kRowW = 40, kPlane = 16 * kRowW;

__device__ __forceinline__ void fx_add(uint32_t* lo, uint32_t* hi, unsigned long long q) {
  const uint32_t l = (uint32_t)q;
  const uint32_t old = atomicAdd(lo, l);
  atomicAdd(hi, (uint32_t)(q >> 32) + ((old + l) < old ? 1u : 0u));
}

template <int MODE>
__global__ void k(unsigned long long* out, int iters, int A) {
  __shared__ uint32_t acc[2 * kPlane];
  for (int i = threadIdx.x; i < 2 * kPlane; i += blockDim.x) acc[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int it = 0; it < iters; ++it) {
    const uint32_t h = hash32(warp * 7919u + it * 104729u);
    const uint32_t g = hash32(h ^ (lane * 2654435761u));
    const int base = h % (kPlane / kRowW * 32 - 128);
    int px = (base + (int)(g % A)) % (16 * 32);
    const int o = (px / 32) * kRowW + px % 32;
    const unsigned long long q = ((unsigned long long)(g & 0x3ffff) << 32) | hash32(g);  // < 2^50
    if (MODE == 0) {
      fx_add(acc + o, acc + kPlane + o, q);
    } else {
      const unsigned peers = __match_any_sync(0xffffffffu, o);
      const uint32_t c0 = __reduce_add_sync(peers, (uint32_t)(q & 0x3fffff));
      const uint32_t c1 = __reduce_add_sync(peers, (uint32_t)((q >> 22) & 0x3fffff));
      const uint32_t c2 = __reduce_add_sync(peers, (uint32_t)(q >> 44));
      if (lane == __ffs(peers) - 1)
        fx_add(acc + o, acc + kPlane + o,
               (unsigned long long)c0 + ((unsigned long long)c1 << 22) + ((unsigned long long)c2 << 44));
    }
  }
  __syncthreads();
  unsigned long long s = 0;
  for (int i = threadIdx.x; i < kPlane; i += blockDim.x)
    s += ((unsigned long long)acc[kPlane + i] << 32) + acc[i];
  atomicAdd(out, s);
}

int main() {
  unsigned long long* o;
  cudaMalloc(&o, 16);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int blocks = 148 * 4, threads = 512, iters = 4096;
  for (int A : {80, 30, 10}) {
    unsigned long long sums[2];
    for (int m = 0; m < 2; ++m) {
      float ms = 0;
      for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(o, 0, 8);
        cudaEventRecord(a);
        if (m == 0) k<0><<<blocks, threads>>>(o, iters, A); else k<1><<<blocks, threads>>>(o, iters, A);
        cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
      }
      cudaMemcpy(&sums[m], o, 8, cudaMemcpyDeviceToHost);
      const double adds = (double)blocks * threads * iters;
      printf("A=%3d %-11s %.3f ms  %.1f G lane-adds/s\n", A, m ? "aggregated" : "plain", ms, adds / (ms * 1e-3) / 1e9);
    }
    printf("A=%3d sums %s\n", A, sums[0] == sums[1] ? "equal" : "DIFFER");
  }
  return 0;
}
