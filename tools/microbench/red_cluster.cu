// Microbenchmark (not product code): throughput of native L2 fp64 reductions
// (RED.E.ADD.F64) on B200 by address pattern, to choose between a shared-memory
// owner design and a sorted-event global-reduction design for the IWE splat.
//
// Every thread plays one "event": 4 bilinear corners x {count, tsum} fp64 adds
// into a double2 (C, S) plane of W x H pixels, for `refs` references.
//   mode 0: events uniformly random over the plane (time-ordered events)
//   mode 1: the 32 events of a warp lie in one 8x8 px tile (tile-sorted events)
//   mode 2: like 1, but the warp first merges lanes hitting the same pixel
//           (__match_any_sync) and only the leader issues the reduction
//   mode 3: like 1 with fp32x2 vector reductions (red.global.add.v2.f32)
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

__global__ void k_splat(double* plane, float* planef, int W, int H, int refs, uint32_t n, int mode) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= n) return;
  const uint32_t warp = tid >> 5;
  const int ntx = W / 8, nty = H / 8;
  for (int r = 0; r < refs; ++r) {
    int x, y;
    const uint32_t h = hash32(tid * 2654435761u + r * 977u);
    if (mode == 0) {
      x = h % (W - 1);
      y = (h >> 12) % (H - 1);
    } else {
      const uint32_t t = hash32(warp * 131u) % (ntx * nty);  // the warp's tile, shifted per ref
      const int tx = (int)(t % ntx) * 8 + r, ty = (int)(t / ntx) * 8 + r;
      x = min(tx + (int)(h & 7), W - 2);
      y = min(ty + (int)((h >> 3) & 7), H - 2);
    }
    const double wx = (h & 0xffff) * (1.0 / 65536.0), wy = (h >> 16) * (1.0 / 65536.0);
    const double tb = 0.3;
    double* pl = plane + (size_t)r * 2 * W * H;
    const int i00 = y * W + x;
    const int idx[4] = {i00, i00 + 1, i00 + W, i00 + W + 1};
    const double wq[4] = {(1 - wx) * (1 - wy), wx * (1 - wy), (1 - wx) * wy, wx * wy};
    if (mode == 3) {
      float* pf = planef + (size_t)r * 2 * W * H;
      for (int q = 0; q < 4; ++q) {
        float2* p = reinterpret_cast<float2*>(pf) + idx[q];
        atomicAdd(p, make_float2((float)wq[q], (float)(wq[q] * tb)));
      }
    } else if (mode == 2) {
      for (int q = 0; q < 4; ++q) {
        const unsigned peers = __match_any_sync(__activemask(), idx[q]);
        double c = wq[q], s = wq[q] * tb;
        // leader sums the peers' values (lane order)
        const int leader = __ffs(peers) - 1;
        double cs = c, ss = s;
        for (int o = 0; o < 32; ++o) {
          if (!((peers >> o) & 1u)) continue;
          const double a = __shfl_sync(peers, c, o), b = __shfl_sync(peers, s, o);
          if (o != (threadIdx.x & 31)) { cs += a; ss += b; }
        }
        if ((threadIdx.x & 31) == leader) {
          atomicAdd(pl + 2 * idx[q], cs);
          atomicAdd(pl + 2 * idx[q] + 1, ss);
        }
      }
    } else {
      for (int q = 0; q < 4; ++q) {
        atomicAdd(pl + 2 * idx[q], wq[q]);
        atomicAdd(pl + 2 * idx[q] + 1, wq[q] * tb);
      }
    }
  }
}

int main() {
  const int cfgW[2] = {346, 640}, cfgH[2] = {260, 480};
  const uint32_t cfgN[2] = {800000, 4000000};
  const int refs = 11;
  for (int c = 0; c < 2; ++c) {
    const int W = cfgW[c], H = cfgH[c];
    const uint32_t n = cfgN[c];
    double* plane;
    float* planef;
    CK(cudaMalloc(&plane, sizeof(double) * 2 * W * H * refs));
    CK(cudaMalloc(&planef, sizeof(float) * 2 * W * H * refs));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char* names[4] = {"random f64", "tile f64", "tile f64 warp-merged", "tile f32x2"};
    for (int mode = 0; mode < 4; ++mode) {
      k_splat<<<(n + 255) / 256, 256>>>(plane, planef, W, H, refs, n, mode);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(a);
      for (int it = 0; it < 5; ++it) k_splat<<<(n + 255) / 256, 256>>>(plane, planef, W, H, refs, n, mode);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      ms /= 5;
      const double reds = (double)n * refs * 8;  // scalar f64 adds
      printf("%dx%d n=%u refs=%d %-22s %.3f ms  %.1f G scalar adds/s\n", W, H, n, refs, names[mode], ms,
             reds / ms / 1e6);
    }
    cudaFree(plane);
    cudaFree(planef);
  }
  return 0;
}
