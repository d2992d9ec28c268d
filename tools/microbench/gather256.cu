// Microbenchmark (not product code): scattered 128-bit vs 256-bit gathers on B200.
// Each warp's 32 lanes read cells at random positions inside a 10x10-pixel window
// of a 640-wide double2 plane (the corner-gather pattern of k_bwd_event /
// k_traj_records). mode 0: 4 x LDG.128 (the 4 corners of a bilinear cell);
// mode 1: 2 x LDG.256 from an x-pair layout (v(p), v(p+1)) per pixel (32 B).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
constexpr int W = 640, H = 480;

__global__ void k128(const double2* __restrict__ f, double* out, int iters) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    const uint32_t h = hash32(warp * 7919u + it * 104729u);
    const int bx = h % (W - 12), by = (h >> 12) % (H - 12);
    const uint32_t g = hash32(h ^ (lane * 2654435761u));
    const int x = bx + g % 10, y = by + (g >> 8) % 10;
    const double2* p = f + (size_t)(it & 7) * W * H + y * W + x;
    const double2 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + W), d = __ldg(p + W + 1);
    acc += a.x + b.y + c.x + d.y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k256(const double4* __restrict__ f, double* out, int iters) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    const uint32_t h = hash32(warp * 7919u + it * 104729u);
    const int bx = h % (W - 12), by = (h >> 12) % (H - 12);
    const uint32_t g = hash32(h ^ (lane * 2654435761u));
    const int x = bx + g % 10, y = by + (g >> 8) % 10;
    const double* p = reinterpret_cast<const double*>(f + (size_t)(it & 7) * W * H + y * W + x);
    double a0, a1, a2, a3, c0, c1, c2, c3;
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a0), "=d"(a1), "=d"(a2), "=d"(a3) : "l"(p));
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(c0), "=d"(c1), "=d"(c2), "=d"(c3) : "l"(p + 4 * W));
    acc += a0 + a3 + c0 + c3;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  double2* f; double4* f4; double* o;
  cudaMalloc(&f, sizeof(double2) * 8 * W * H + 4096);
  cudaMalloc(&f4, sizeof(double4) * 8 * W * H + 4096);
  cudaMalloc(&o, 1 << 24);
  cudaMemset(f, 0, sizeof(double2) * 8 * W * H);
  cudaMemset(f4, 0, sizeof(double4) * 8 * W * H);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int blocks = 148 * 16, threads = 128, iters = 2000;
  for (int m = 0; m < 2; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (m == 0) k128<<<blocks, threads>>>(f, o, iters); else k256<<<blocks, threads>>>(f4, o, iters);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double cells = (double)blocks * threads * iters;
      if (rep) printf("%s: %.3f ms, %.2f G cells/s (4 corners each)\n", m ? "2 x LDG.256 (x-pair layout)" : "4 x LDG.128",
                      ms, cells / (ms * 1e-3) / 1e9);
    }
  }
  return 0;
}
