// Microbenchmark (not product code): native shared-memory 32-bit integer
// atomics (ATOMS.ADD / RED on shared) vs fp64 CAS loops on B200, to size a
// fixed-point (3 x 18-bit chunk) IWE accumulation.
//   mode 0: u32 atomicAdd, result unused (RED-style), random slots in 16 KB
//   mode 1: u32 atomicAdd with the return value used
//   mode 2: fp64 atomicAdd (CAS loop), random slots in 16 KB
//   mode 3: u32 atomicAdd, 4 consecutive words per lane (one 2x2 corner set)
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

__global__ void k(uint32_t* out, int iters, int mode) {
  __shared__ uint32_t s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = 0;
  __syncthreads();
  uint32_t acc = 0;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    const uint32_t h = hash32(tid * 2654435761u + it);
    const uint32_t slot = h & 4095;
    if (mode == 0) atomicAdd(s + slot, h >> 20);
    else if (mode == 1) acc += atomicAdd(s + slot, h >> 20);
    else if (mode == 2) atomicAdd(reinterpret_cast<double*>(s) + (slot >> 1), 1.0);
    else {
      const uint32_t b = slot & ~3u;
      atomicAdd(s + b, h >> 20); atomicAdd(s + b + 1, h >> 21);
      atomicAdd(s + b + 2, h >> 22); atomicAdd(s + b + 3, h >> 23);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[0] + acc;
}

int main() {
  uint32_t* o;
  cudaMalloc(&o, 1 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = 148 * 4, threads = 512, iters = 2048;
  const char* nm[4] = {"u32 add (no return)", "u32 add (return used)", "f64 add (CAS loop)", "u32 add x4 adjacent"};
  for (int m = 0; m < 4; ++m) {
    k<<<blocks, threads>>>(o, iters, m);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    k<<<blocks, threads>>>(o, iters, m);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double ops = (double)blocks * threads * iters * (m == 3 ? 4 : 1);
    printf("%-24s %.3f ms  %.1f G lane-ops/s  (%.2f lane-ops/clk/SM @1.965GHz)\n", nm[m], ms, ops / ms / 1e6,
           ops / ms / 1e6 / 148 / 1.965);
  }
  return 0;
}
