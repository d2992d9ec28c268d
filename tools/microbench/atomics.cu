// Microbenchmark: atomic / fp64 throughput on B200, to size the splat and
// backward scatter design. Standalone; not product code.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// mode 0: random float2 vector red; 1: random double red; 2: random float red (2 scalars)
// 3: clustered float2 (warp lanes within a 32x32 px tile of a 640-wide image)
__global__ void k_global(float2* f2, double* d, float* f, uint32_t n_slots, uint32_t iters, int mode) {
  uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t warp = tid >> 5, lane = tid & 31;
  for (uint32_t it = 0; it < iters; ++it) {
    uint32_t h = hash32(tid * 2654435761u + it * 97u);
    uint32_t slot;
    if (mode == 3) {
      uint32_t tile = hash32(warp * 131u + it) % (n_slots / 1024);
      uint32_t tx = (tile % 20) * 32, ty = (tile / 20) * 32;
      slot = ((ty + (h >> 5) % 32) * 640 + tx + (h % 32)) % n_slots;
    } else {
      slot = h % n_slots;
    }
    if (mode == 0 || mode == 3) {
      atomicAdd(&f2[slot], make_float2(1.0f, 0.5f));
    } else if (mode == 1) {
      atomicAdd(&d[slot], 1.0);
    } else {
      atomicAdd(&f[2 * slot], 1.0f);
      atomicAdd(&f[2 * slot + 1], 0.5f);
    }
  }
}

// smem: mode 0 float atomic, 1 double atomic, 2 float2 plain RMW (racy, timing only), 3 int64 atomic
__global__ void k_smem(float* out, uint32_t iters, int mode) {
  extern __shared__ double sm[];
  const uint32_t n = 4096;  // 32 KB of doubles
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) sm[i] = 0.0;
  __syncthreads();
  uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  for (uint32_t it = 0; it < iters; ++it) {
    uint32_t slot = hash32(tid * 2654435761u + it) % n;
    if (mode == 0) atomicAdd(reinterpret_cast<float*>(sm) + slot, 1.0f);
    else if (mode == 1) atomicAdd(sm + slot, 1.0);
    else if (mode == 2) { float2* p = reinterpret_cast<float2*>(sm) + (slot >> 1); float2 v = *p; v.x += 1.f; v.y += .5f; *p = v; }
    else atomicAdd(reinterpret_cast<unsigned long long*>(sm) + slot, 3ull);
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = (float)sm[0];
}

__global__ void k_dfma(double* out, uint32_t iters) {
  double a = threadIdx.x * 1e-3, b = 1.0000001, c = 1e-9, e = 0.5, f = 0.25, g = 0.125, h = 0.0625;
  for (uint32_t i = 0; i < iters; ++i) {
    a = fma(a, b, c); e = fma(e, b, c); f = fma(f, b, c); g = fma(g, b, c); h = fma(h, b, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + e + f + g + h;
}

int main() {
  const uint32_t n_slots = 44u * 307200u;  // (B+1)*2*2 planes of 640x480 as float2 -> 108 MB
  float2* f2; double* d; float* f; float* o; double* od;
  CK(cudaMalloc(&f2, sizeof(float2) * n_slots));
  CK(cudaMalloc(&d, sizeof(double) * n_slots));
  CK(cudaMalloc(&f, sizeof(float) * 2 * n_slots));
  CK(cudaMalloc(&o, 1 << 20));
  CK(cudaMalloc(&od, 148 * 1024 * 8 * 8));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int blocks = 148 * 8, threads = 256; const uint32_t iters = 128;
  const double ops = double(blocks) * threads * iters;
  const char* gname[4] = {"red.v2.f32 random", "red.f64 random", "red.f32 x2 random", "red.v2.f32 clustered"};
  uint32_t sl[2] = {n_slots / 4, n_slots};  // 27 MB and 108 MB footprints
  for (int s = 0; s < 2; ++s)
    for (int m = 0; m < 4; ++m) {
      k_global<<<blocks, threads>>>(f2, d, f, sl[s], iters, m);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(a);
      k_global<<<blocks, threads>>>(f2, d, f, sl[s], iters, m);
      cudaEventRecord(b); CK(cudaEventSynchronize(b));
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("global %-22s slots=%u: %.3f ms  %.1f Gop/s\n", gname[m], sl[s], ms, ops / ms / 1e6);
    }
  const char* sname[4] = {"atom.f32", "atom.f64", "rmw.v2.f32", "atom.u64"};
  for (int m = 0; m < 4; ++m) {
    k_smem<<<blocks, threads, 32768>>>(o, iters * 4, m);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    k_smem<<<blocks, threads, 32768>>>(o, iters * 4, m);
    cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("smem %-12s: %.3f ms  %.1f Gop/s\n", sname[m], ms, ops * 4 / ms / 1e6);
  }
  k_dfma<<<148 * 8, 256>>>(od, 4096); CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  k_dfma<<<148 * 8, 256>>>(od, 4096);
  cudaEventRecord(b); CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("dfma: %.3f ms  %.2f TFLOP/s fp64\n", ms, 148.0 * 8 * 256 * 4096 * 5 * 2 / ms / 1e9);
  return 0;
}
