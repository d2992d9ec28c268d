// Owner-computes CMax pipeline (sm_100a): no global atomics on the IWE stack or
// the flow gradients and no memsets of them; the focus loss and the per-pixel
// loss coefficients are fused into the stack accumulation, and the flows
// backward is fused into the gradient gather. See DESIGN.md §Kernels.
//
//   k_stage_pack    validate (EventSlice::validate) + pack events to 8 B
//   k_key_hist      approximate position of every event at the middle reference
//                   -> 8x8 px sort-tile key + per-(chunk, tile) histogram
//   k_sort_colscan  per tile: prefix over chunks; k_sort_tilescan: tile offsets
//   k_sort_scatter  stable counting sort of the events by key
//   k_bin_ptr       per sort tile: first event of every time bin
//   k_traj_records  full trajectory -> per (event, ref) splat record {cell, pol,
//                   dt, compressed bilinear fractions} + per (sort tile, slot)
//                   boxes of the cells (slots 0..B: references, B+1..2B: source
//                   pixel of the events of bin j)
//   k_build_lists   per (slot, owner tile): the sort tiles whose box touches it
//   k_bwd_event     per event: splat_position_grad at every ref + adjoint sweep
//                   (engine.hpp:475-504) -> one (gx, gy) per sink
// The owner-tile accumulation kernels (IWE stack + loss coefficients; flow
// gradient tiles + fused flows backward) are in cmax_cells.cu.
//
// Sorting by the position at the middle reference keeps every sort tile compact
// at every reference (a tile of source pixels would smear along the motion by
// |flow| x window), so each record is read by ~2 owner tiles.
//
// Determinism: stable sort; owners visit sort tiles in index order and events
// in sorted order; lanes resolve shared-pixel conflicts in lane order; per-warp
// shared copies are merged in warp order; every partial sum is reduced in a
// fixed order -> results are bit-stable run to run.
#include <algorithm>
#include <cstdint>

#include "cmax_device.cuh"
#include "cmax_kernels.h"
#include "cmax_owner.h"
#include "cmax_owner_dev.cuh"

namespace evcm_b200 {

void count_launch();  // cmax_kernels.cu

using namespace owner_dev;

// ---------------------------------------------------------------------------
// staging and sort

__global__ void __launch_bounds__(kSortThreads) k_stage_pack(
    const evcm_event* __restrict__ ev, const uint64_t* __restrict__ ev_off, WinParams P,
    uint2* __restrict__ packed, unsigned long long* __restrict__ err) {
  const int w = blockIdx.y;
  const uint64_t base = ev_off[w];
  const uint64_t n = ev_off[w + 1] - base;
  const uint64_t t0 = P.t0 + (uint64_t)w * P.stride_us, t_end = P.t_end + (uint64_t)w * P.stride_us;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const evcm_event e = ev[base + k];
    unsigned code = 0;  // EventSlice::validate order (types.hpp:143-155)
    if (e.x >= P.W || e.y >= P.H) code = 3;
    else if (e.p != 1 && e.p != -1) code = 4;
    else if (k > 0 && e.t_us < ev[base + k - 1].t_us) code = 5;
    else if (e.t_us < t0 || e.t_us >= t_end) code = 6;
    if (code) {
      atomicMin(err + w, ((unsigned long long)k << 4) | code);
      packed[base + k] = make_uint2(kDead, kDead);
      continue;
    }
    const uint32_t dt = (uint32_t)(e.t_us - t0);
    packed[base + k] = make_uint2(dt | (e.p > 0 ? 0u : 0x80000000u),
                                  (uint32_t)e.x | ((uint32_t)e.y << 16));
  }
}

// Coarse flow map for the sort key: the flow of every bin sampled at the
// centre pixel of every 8x8 sort tile, [w][B][nT] (768 KB per 640x480 window:
// L2-resident, unlike per-event gathers from the full flow planes).
__global__ void k_coarse_flow(const double2* __restrict__ flows, WinParams P, TileParams TP,
                              double2* __restrict__ coarse, uint4* __restrict__ bbox, size_t n_bbox,
                              uint32_t* __restrict__ lcount, size_t n_lcount){
  const size_t total = (size_t)P.n_windows * P.B * TP.nT;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int S = (int)(i % TP.nT);
    const size_t wb = i / TP.nT;  // w * B + b
    const int cx = min((S % TP.ntx) * kSortTile + kSortTile / 2, P.W - 1);
    const int cy = min((S / TP.ntx) * kSortTile + kSortTile / 2, P.H - 1);
    coarse[i] = flows[wb * P.HW + (size_t)cy * P.W + cx];
  }
  // the empty cell boxes and list counts of k_traj_records / k_build_lists
  // (folded in here instead of two memset nodes)
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_bbox;
       i += (size_t)gridDim.x * blockDim.x)
    bbox[i] = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_lcount;
       i += (size_t)gridDim.x * blockDim.x)
    lcount[i] = 0u;
}

// Sort key: 8x8 tile of the event's approximate position at the middle
// reference rm = (B+1)/2, extrapolated with the coarse flow of its own bin at
// its own tile: x0 + u_j(tile(x0)) * (e_rm - t). Any deterministic key is valid;
// this one keeps every tile compact at every reference.
// counts layout: [w][chunk][tile] (coalesced writes and column scans).
__global__ void __launch_bounds__(kSortThreads) k_key_hist(
    const uint2* __restrict__ packed, const uint64_t* __restrict__ ev_off, WinParams P,
    TileParams TP, const double2* __restrict__ coarse, uint32_t* __restrict__ keys,
    uint32_t* __restrict__ counts) {
  extern __shared__ uint32_t hist[];
  __shared__ double es[kMaxRefs];
  __shared__ uint32_t erel[kMaxRefs];
  for (int i = threadIdx.x; i < TP.nT; i += blockDim.x) hist[i] = 0;
  for (int i = threadIdx.x; i <= P.B; i += blockDim.x) {
    es[i] = P.es[i];
    erel[i] = P.erel[i];
  }
  __syncthreads();
  const int w = blockIdx.y, B = P.B;
  const double em = es[(B + 1) / 2];
  const uint64_t base = ev_off[w];
  const uint64_t n = ev_off[w + 1] - base;
  const uint64_t c0 = (uint64_t)blockIdx.x * TP.chunk;
  const uint64_t c1 = c0 + TP.chunk < n ? c0 + TP.chunk : n;
  const double2* cf = coarse + (size_t)w * B * TP.nT;
  for (uint64_t k = c0 + threadIdx.x; k < c1; k += blockDim.x) {
    const uint2 e = packed[base + k];
    if (e.y == kDead) {
      keys[base + k] = kDead;
      continue;
    }
    const uint32_t dtu = ev_dt(e);
    const int j = bin_of(dtu, erel, B);
    const int x0 = ev_x(e), y0 = ev_y(e);
    const double2 u = __ldg(cf + (size_t)j * TP.nT + (y0 / kSortTile) * TP.ntx + x0 / kSortTile);
    const double dt = em - (double)dtu * 1e-6;
    const uint32_t key = (uint32_t)sort_tile_of(x0 + u.x * dt, y0 + u.y * dt, P, TP);
    keys[base + k] = key;
    atomicAdd(&hist[key], 1u);
  }
  __syncthreads();
  uint32_t* cw = counts + ((size_t)w * TP.nchunks + blockIdx.x) * TP.nT;
  for (int t = threadIdx.x; t < TP.nT; t += blockDim.x) cw[t] = hist[t];
}

// Per tile: exclusive prefix over chunks (in place, counts -> offsets inside the
// tile) and the tile total. A CTA covers 32 tiles x kColSeg chunk segments: each
// thread sums its segment (independent, coalesced loads across the 32 tiles),
// the segment sums are scanned in shared memory, then each thread writes its
// segment's running offsets -- two load round trips instead of nchunks / 8.
constexpr int kColSeg = 8;
__global__ void __launch_bounds__(32 * kColSeg) k_sort_colscan(uint32_t* __restrict__ counts,
                                                               TileParams TP,
                                                               uint32_t* __restrict__ totals) {
  __shared__ uint32_t seg_sum[kColSeg][32];
  const int w = blockIdx.y, lane = threadIdx.x & 31, sg = threadIdx.x >> 5;
  const int t = blockIdx.x * 32 + lane;
  const int per = (TP.nchunks + kColSeg - 1) / kColSeg;
  const int c0 = sg * per, c1 = min(TP.nchunks, c0 + per);
  uint32_t* c = counts + (size_t)w * TP.nchunks * TP.nT + t;
  uint32_t sum = 0;
  if (t < TP.nT) {
#pragma unroll 8
    for (int ch = c0; ch < c1; ++ch) sum += c[(size_t)ch * TP.nT];
  }
  seg_sum[sg][lane] = sum;
  __syncthreads();
  uint32_t run = 0;
  for (int q = 0; q < sg; ++q) run += seg_sum[q][lane];
  if (t < TP.nT) {
    for (int ch = c0; ch < c1; ++ch) {
      const uint32_t v = c[(size_t)ch * TP.nT];
      c[(size_t)ch * TP.nT] = run;
      run += v;
    }
    if (sg == kColSeg - 1) totals[(size_t)w * TP.nT + t] = run;
  }
}

// Exclusive scan of the tile totals: tile_ptr[w][t] = first sorted slot of tile
// t, tile_ptr[w][nT] = valid events of the window. One CTA per window.
__global__ void __launch_bounds__(1024) k_sort_tilescan(const uint32_t* __restrict__ totals,
                                                        TileParams TP,
                                                        uint32_t* __restrict__ tile_ptr) {
  __shared__ uint32_t warp_tot[32];
  __shared__ uint32_t s_carry;
  const int w = blockIdx.x, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t* tot = totals + (size_t)w * TP.nT;
  uint32_t* tp = tile_ptr + (size_t)w * (TP.nT + 1);
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int b = 0; b < TP.nT; b += blockDim.x) {
    const int t = b + threadIdx.x;
    const uint32_t v = t < TP.nT ? tot[t] : 0u;
    uint32_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      uint32_t q = warp_tot[lane];
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, q, o);
        if (lane >= o) q += y;
      }
      warp_tot[lane] = q;
    }
    __syncthreads();
    const uint32_t excl = s_carry + x - v + (wid > 0 ? warp_tot[wid - 1] : 0u);
    if (t < TP.nT) tp[t] = excl;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) s_carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) tp[TP.nT] = s_carry;
}

// Stable scatter: warp `wid` of chunk c owns events [c*chunk + wid*chunk/nW, ...);
// per-warp tile counts (u16) give each warp its base inside the chunk's run of
// the tile, so the output keeps the input (time) order inside every tile.
// (__maxnreg__: ptxas picked 32 registers for the 128-thread form and spilled;
// 48 leaves no spill and does not limit occupancy, which shared memory sets)
template <int NW>
__global__ void __maxnreg__(48) k_sort_scatter(
    const uint2* __restrict__ packed, const uint32_t* __restrict__ keys,
    const uint64_t* __restrict__ ev_off, TileParams TP, const uint32_t* __restrict__ offsets,
    const uint32_t* __restrict__ tile_ptr, uint2* __restrict__ sorted, uint32_t* __restrict__ perm,
    uint32_t* __restrict__ sorted_keys) {
  extern __shared__ __align__(16) uint16_t whist[];  // [nW warps][ws]
  constexpr int nW = NW;  // 8 warps, or 4 for many tiles (launch_sort)
  const int per = TP.chunk / nW;
  const int ws = (TP.nT + 7) & ~7;  // row stride: 8 tiles per 16 B word
  for (int i = threadIdx.x; i < nW * ws / 8; i += blockDim.x)
    reinterpret_cast<uint4*>(whist)[i] = make_uint4(0u, 0u, 0u, 0u);
  __syncthreads();
  const int w = blockIdx.y, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t base = ev_off[w];
  const uint64_t n = ev_off[w + 1] - base;
  const uint64_t k0 = (uint64_t)blockIdx.x * TP.chunk + (uint64_t)wid * per;
  uint16_t* mine = whist + wid * ws;
  // pass 1: per-warp counts. Many-tile chunks (NW = 4, e.g. 640x480) pipeline
  // the key loads by hand (see pass 3); the 8-warp form measured faster as is.
  if constexpr (NW <= 4) {
    int tn = -1;  // the next step's key in flight
    {
      const uint64_t k = k0 + lane;
      if (per > 0 && k < n) {
        const uint32_t key = keys[base + k];
        if (key != kDead) tn = (int)key;
      }
    }
    for (int b = 0; b < per; b += 32) {
      const int t = tn;
      tn = -1;
      {
        const uint64_t k = k0 + b + 32 + lane;
        if (b + 32 < per && k < n) {
          const uint32_t key = keys[base + k];
          if (key != kDead) tn = (int)key;
        }
      }
      const unsigned act = __ballot_sync(kFull, t >= 0);
      if (t >= 0) {
        const unsigned peers = __match_any_sync(act, t);
        if (lane == __ffs(peers) - 1) mine[t] = (uint16_t)(mine[t] + __popc(peers));
      }
      __syncwarp();
    }
  } else {
    for (int b = 0; b < per; b += 32) {  // pass 1: per-warp counts
      const uint64_t k = k0 + b + lane;
      int t = -1;
      if (k < n) {
        const uint32_t key = keys[base + k];
        if (key != kDead) t = (int)key;
      }
      const unsigned act = __ballot_sync(kFull, t >= 0);
      if (t >= 0) {
        const unsigned peers = __match_any_sync(act, t);
        if (lane == __ffs(peers) - 1) mine[t] = (uint16_t)(mine[t] + __popc(peers));
      }
      __syncwarp();
    }
  }
  __syncthreads();
  const uint32_t* off = offsets + ((size_t)w * TP.nchunks + blockIdx.x) * TP.nT;
  const uint32_t* tp = tile_ptr + (size_t)w * (TP.nT + 1);
  // pass 2: prefix over warps, 8 tiles per thread as u16 pairs in u32 words
  // (every partial sum is <= chunk < 2^16: no carry between the halves)
  for (int i = threadIdx.x; i < ws / 8; i += blockDim.x) {
    uint4 run = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
    for (int q = 0; q < nW; ++q) {
      uint4* p = reinterpret_cast<uint4*>(whist + q * ws) + i;
      const uint4 v = *p;
      *p = run;
      run.x += v.x;
      run.y += v.y;
      run.z += v.z;
      run.w += v.w;
    }
  }
  __syncthreads();
  if constexpr (NW <= 4) {
    // pass 3: place in order. Software-pipelined by hand (the warp syncs keep the
    // compiler from hoisting loads): the key of step i + 2 and the event and tile
    // base (tile_ptr + chunk offset) of step i + 1 are in flight while step i places.
    auto key_at = [&](int b) -> int {
      const uint64_t k = k0 + b + lane;
      if (b >= per || k >= n) return -1;
      const uint32_t key = keys[base + k];
      return key != kDead ? (int)key : -1;
    };
    auto ev_at = [&](int b) -> uint2 {
      const uint64_t k = k0 + b + lane;
      return (b < per && k < n) ? packed[base + k] : make_uint2(0u, 0u);
    };
    auto base_of = [&](int t) -> uint32_t { return t >= 0 ? tp[t] + off[t] : 0u; };
    int t1 = key_at(0), t2 = key_at(32);
    uint32_t g1 = base_of(t1);
    uint2 e1 = ev_at(0);
    for (int b = 0; b < per; b += 32) {
      const int t = t1;
      const uint32_t gb = g1;
      const uint2 ev = e1;
      t1 = t2;
      g1 = base_of(t2);
      e1 = ev_at(b + 32);
      t2 = key_at(b + 64);
      const uint64_t k = k0 + b + lane;
      const unsigned act = __ballot_sync(kFull, t >= 0);
      if (t >= 0) {
        const unsigned peers = __match_any_sync(act, t);
        const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
        const uint32_t dst = gb + mine[t] + rank;
        sorted[base + dst] = ev;
        sorted_keys[base + dst] = (uint32_t)t;
        if (perm) perm[base + dst] = (uint32_t)k;
        __syncwarp(peers);
        if (lane == __ffs(peers) - 1) mine[t] = (uint16_t)(mine[t] + __popc(peers));
      }
      __syncwarp();
    }
  } else {
    for (int b = 0; b < per; b += 32) {  // pass 3: place in order
      const uint64_t k = k0 + b + lane;
      int t = -1;
      if (k < n) {
        const uint32_t key = keys[base + k];
        if (key != kDead) t = (int)key;
      }
      const unsigned act = __ballot_sync(kFull, t >= 0);
      if (t >= 0) {
        const unsigned peers = __match_any_sync(act, t);
        const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
        const uint32_t dst = tp[t] + off[t] + mine[t] + rank;
        sorted[base + dst] = packed[base + k];
        sorted_keys[base + dst] = (uint32_t)t;
        if (perm) perm[base + dst] = (uint32_t)k;
        __syncwarp(peers);
        if (lane == __ffs(peers) - 1) mine[t] = (uint16_t)(mine[t] + __popc(peers));
      }
      __syncwarp();
    }
  }
}

// bin_ptr[w][S][b] = first sorted slot of tile S whose event bin is >= b
// (the stable sort keeps events time-ordered inside a tile, so bins are
// non-decreasing along the tile's run): one warp per tile, lane b runs the
// binary search for the first slot with dt >= erel[b] -- the B-1 searches of a
// tile proceed in parallel instead of one after another.
__global__ void k_bin_ptr(const uint2* __restrict__ sorted, const uint64_t* __restrict__ ev_off,
                          WinParams P, TileParams TP, const uint32_t* __restrict__ tile_ptr,
                          uint32_t* __restrict__ bin_ptr) {
  const int w = blockIdx.y, lane = threadIdx.x & 31;
  const int S = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (S >= TP.nT) return;
  const int B = P.B;
  const uint64_t base = ev_off[w];
  const uint32_t* tp = tile_ptr + (size_t)w * (TP.nT + 1);
  const uint32_t lo = tp[S], hi = tp[S + 1];
  uint32_t* out = bin_ptr + ((size_t)w * TP.nT + S) * (B + 1);
  if (lane == 0) {
    out[0] = lo;
    out[B] = hi;
  } else if (lane < B) {
    const uint32_t th = P.erel[lane];
    uint32_t a = lo, z = hi;  // first slot with dt >= erel[lane]
    while (a < z) {
      const uint32_t m = (a + z) >> 1;
      if ((__ldg(&sorted[base + m].x) & 0x7fffffffu) >= th) z = m; else a = m + 1;
    }
    out[lane] = a;
  }
}

constexpr int kSrcBaseThreads = 512;

// Source-sink layout (bin, tile, time): srcbase[w][b][S] = window-relative
// position of the first source sink of sort tile S's events of bin b, so that
// the events of bin b of consecutive sort tiles are contiguous and the backward
// owner's source ranges merge like its record ranges (k_ranges). One CTA per
// (bin, window): the bin's offset is the number of the window's events in
// earlier bins (bin_ptr is cumulative per tile: sum over S of bp[S][b] - bp[S][0]),
// then an exclusive scan over the tiles of the per-(tile, bin) counts.
__global__ void __launch_bounds__(kSrcBaseThreads) k_src_base(const uint32_t* __restrict__ bin_ptr,
                                                              WinParams P, TileParams TP,
                                                              uint32_t* __restrict__ srcbase) {
  __shared__ uint32_t warp_tot[kSrcBaseThreads / 32];
  __shared__ uint32_t s_carry;
  const int b = blockIdx.x, w = blockIdx.y, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int B = P.B, nw = kSrcBaseThreads / 32;
  const uint32_t* bp = bin_ptr + (size_t)w * TP.nT * (B + 1);
  uint32_t before = 0;
  for (int S = threadIdx.x; S < TP.nT; S += kSrcBaseThreads)
    before += bp[(size_t)S * (B + 1) + b] - bp[(size_t)S * (B + 1)];
  before = __reduce_add_sync(kFull, before);
  if (lane == 0) warp_tot[wid] = before;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t c = 0;
    for (int i = 0; i < nw; ++i) c += warp_tot[i];
    s_carry = c;
  }
  __syncthreads();
  uint32_t* out = srcbase + ((size_t)w * B + b) * TP.nT;
  for (int c = 0; c < TP.nT; c += kSrcBaseThreads) {
    const int S = c + threadIdx.x;
    const uint32_t v = S < TP.nT ? bp[(size_t)S * (B + 1) + b + 1] - bp[(size_t)S * (B + 1) + b] : 0u;
    uint32_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      uint32_t q = lane < nw ? warp_tot[lane] : 0u;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, q, o);
        if (lane >= o) q += y;
      }
      if (lane < nw) warp_tot[lane] = q;
    }
    __syncthreads();
    const uint32_t excl = s_carry + x - v + (wid > 0 ? warp_tot[wid - 1] : 0u);
    if (S < TP.nT) out[S] = excl;
    __syncthreads();
    if (threadIdx.x == kSrcBaseThreads - 1) s_carry = excl + v;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// trajectories -> splat records + per-(sort tile, slot) cell boxes

__device__ __forceinline__ uint4 make_rec(const Cell& c, uint32_t dt, int pol) {
  return make_uint4((uint32_t)c.x0 | ((uint32_t)c.y0 << 16) | ((uint32_t)pol << 31), dt,
                    __float_as_uint(compress_frac(c.wx)), __float_as_uint(compress_frac(c.wy)));
}

// trajectory (cmax_device.cuh, build_trajectory warp.hpp:257-281) emitting the
// splat record of every reference instead of its position: the bilinear cells
// of the interior references 1..B-1 are the ones the flow sampling of the next
// step computes anyway, so only references 0 and B need their own bilin_cell.
// rec[r * stride] receives the record of reference r. Returns alive.
// Records go straight to global memory (plane r of `grec`, stride n_total; a
// warp's lanes mostly share j, so the stores of a step mostly share a plane) and
// the cell of every reference to shared memory (scell[r * stride], for the box
// reduction that needs all lanes at the same reference).
__device__ __forceinline__ bool trajectory_records(double x0, double y0, double t, int j,
                                                   const double2* __restrict__ flows,
                                                   const WinParams& P, const double* es,
                                                   uint4* grec, uint64_t gstride, uint32_t* scell,
                                                   int stride, uint32_t dtu, int pol) {
  const int W = P.W, H = P.H, B = P.B, HW = P.HW;
  const Cell c0 = bilin_cell(x0, y0, W, H);
  const double2 u0 = sample_flow(flows + (size_t)j * HW, c0);
  const double db = ds(es[j], t), df = ds(es[j + 1], t);
  double2 pb = make_double2(da(x0, dm(db, u0.x)), da(y0, dm(db, u0.y)));
  double2 pf = make_double2(da(x0, dm(df, u0.x)), da(y0, dm(df, u0.y)));
  bool ok = in_bounds(pb.x, pb.y, W, H) && in_bounds(pf.x, pf.y, W, H);
  for (int s = 0; s < B - 1; ++s) {
    const bool back = s < j;
    // backward leg: bin i = j-1-s sampled at pos[i+1] (reference i+1), writes pos[i]
    // forward leg:  bin i = s+1     sampled at pos[i]   (reference i),   writes pos[i+1]
    const int i = back ? j - 1 - s : s + 1;
    const double2 p = back ? pb : pf;
    const double dt = back ? ds(es[i], es[i + 1]) : ds(es[i + 1], es[i]);
    const Cell c = bilin_cell(p.x, p.y, W, H);
    const int rr = back ? i + 1 : i;
    const uint4 rv = make_rec(c, dtu, pol);
    grec[rr * gstride] = rv;
    scell[rr * stride] = rv.x;
    const double2 u = sample_flow(flows + (size_t)i * HW, c);
    const double2 q = make_double2(da(p.x, dm(dt, u.x)), da(p.y, dm(dt, u.y)));
    ok = ok && in_bounds(q.x, q.y, W, H);
    if (back) pb = q; else pf = q;
  }
  const uint4 r0 = make_rec(bilin_cell(pb.x, pb.y, W, H), dtu, pol);  // pb = pos[0]
  const uint4 rB = make_rec(bilin_cell(pf.x, pf.y, W, H), dtu, pol);  // pf = pos[B]
  grec[0] = r0;
  scell[0] = r0.x;
  grec[B * gstride] = rB;
  scell[B * stride] = rB.x;
  return ok;
}

__global__ void __launch_bounds__(kEvBlock) k_traj_records(
    const uint2* __restrict__ sorted, const uint64_t* __restrict__ ev_off, WinParams P,
    TileParams TP, const uint32_t* __restrict__ tile_ptr, const uint32_t* __restrict__ sorted_keys,
    const double2* __restrict__ flows, uint64_t n_total, FwdRec* __restrict__ recs,
    uint4* __restrict__ bbox) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* es = reinterpret_cast<double*>(smem);
  uint32_t* erel = reinterpret_cast<uint32_t*>(es + kMaxRefs);
  uint32_t* scell = reinterpret_cast<uint32_t*>(smem + kEvSmemHeader) + threadIdx.x;  // [r][thread]
  for (int i = threadIdx.x; i <= P.B; i += blockDim.x) {
    es[i] = P.es[i];
    erel[i] = P.erel[i];
  }
  __syncthreads();
  const int w = blockIdx.y, R = P.B + 1, NS = R + P.B;
  const uint64_t base = ev_off[w];
  const uint32_t* tp = tile_ptr + (size_t)w * (TP.nT + 1);
  const uint64_t n = tp[TP.nT];  // valid (sorted) events
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = k < n;
  bool alive = false;
  uint2 e = make_uint2(0, 0);
  int j = 0;
  int S = -1;
  if (valid) {
    e = sorted[base + k];
    const uint32_t dt = ev_dt(e);
    const double t = dm((double)dt, 1e-6);
    j = bin_of(dt, erel, P.B);
    alive = trajectory_records((double)ev_x(e), (double)ev_y(e), t, j,
                               flows + (size_t)w * P.B * P.HW, P, es,
                               reinterpret_cast<uint4*>(recs) + base + k, n_total, scell,
                               blockDim.x, dt, ev_pol(e));
    S = (int)sorted_keys[base + k];  // sort tile of this slot
  }
  const unsigned amask = __ballot_sync(kFull, alive);
  const unsigned peers = alive ? __match_any_sync(amask, S) : 0u;
  const bool leader = alive && (threadIdx.x & 31) == __ffs(peers) - 1;
  uint4* bb = bbox + (size_t)w * NS * TP.nT;
  auto box_update = [&](unsigned grp, bool lead, int slot, uint32_t x0, uint32_t y0) {
    const uint32_t mnx = __reduce_min_sync(grp, x0), mny = __reduce_min_sync(grp, y0);
    const uint32_t cmx = __reduce_min_sync(grp, 0xffffu - x0);
    const uint32_t cmy = __reduce_min_sync(grp, 0xffffu - y0);
    if (lead) {
      uint4* b = bb + (size_t)slot * TP.nT + S;
      atomicMin(&b->x, mnx);
      atomicMin(&b->y, mny);
      atomicMin(&b->z, cmx);
      atomicMin(&b->w, cmy);
    }
  };
  // a dead (left the sensor) event's records are rewritten dead
  const uint4 dead = make_uint4(kDead, 0u, 0u, 0u);
  for (int r = 0; r < R; ++r) {
    if (valid && !alive) reinterpret_cast<uint4*>(recs)[(size_t)r * n_total + base + k] = dead;
    if (alive) {
      const uint32_t cell = scell[r * blockDim.x];
      box_update(peers, leader, r, cell & 0xffffu, (cell >> 16) & 0x7fffu);
    }
  }
  // source-pixel boxes per bin (the partial steps of the backward sink at x0)
  if (alive) {
    const unsigned g2 = __match_any_sync(amask, S * kMaxRefs + j);
    const bool l2 = (threadIdx.x & 31) == __ffs(g2) - 1;
    box_update(g2, l2, R + j, (uint32_t)ev_x(e), (uint32_t)ev_y(e));
  }
}

// ---------------------------------------------------------------------------
// owner source lists

// For every (window, slot, sort tile) with alive events: append S to the list of
// every owner tile its cell box can touch (cells touch [x0, x0+1] x [y0, y0+1]).
// Lists are unordered here; owners sort them, so the visit order is fixed.
__global__ void k_build_lists(const uint4* __restrict__ bbox, WinParams P, TileParams TP,
                              uint32_t* __restrict__ lcount, uint16_t* __restrict__ lists) {
  const int S = blockIdx.x * blockDim.x + threadIdx.x, slot = blockIdx.y, w = blockIdx.z;
  if (S >= TP.nT) return;
  const int NS = 2 * P.B + 1;
  const size_t ws = (size_t)w * NS + slot;
  const uint4 b = bbox[ws * TP.nT + S];
  if (b.x == 0xffffffffu) return;
  const int mnx = (int)b.x, mny = (int)b.y, mxx = 0xffff - (int)b.z, mxy = 0xffff - (int)b.w;
  const int tx0 = mnx / kOwnW, tx1 = min((mxx + 1) / kOwnW, TP.otx - 1);
  const int ty0 = mny / kOwnH, ty1 = min((mxy + 1) / kOwnH, TP.oty - 1);
  for (int ty = ty0; ty <= ty1; ++ty)
    for (int tx = tx0; tx <= tx1; ++tx) {
      const size_t T = ws * TP.oT + (size_t)ty * TP.otx + tx;
      const uint32_t c = atomicAdd(lcount + T, 1u);
      if (c < (uint32_t)kListCapO) lists[T * kListCapO + c] = (uint16_t)S;
    }
}

// ---------------------------------------------------------------------------
// backward, per event: d[r] at every reference + adjoint sweep -> (gx, gy) per bin

// cp: the event's polarity in a polarity-interleaved plane (pixel stride 2)
__device__ __forceinline__ double2 pos_grad_w(const double2* __restrict__ cp, int W, int ox, int oy,
                                              const CellW& c, double tb, double scale) {
  const int i00 = 2 * (c.y0 * W + c.x0);
  const double2 k00 = __ldg(cp + i00), k10 = __ldg(cp + i00 + 2 * ox);
  const double2 k01 = __ldg(cp + i00 + 2 * oy * W), k11 = __ldg(cp + i00 + 2 * (oy * W + ox));
  const double g00 = scale * k00.y * (tb - k00.x);
  const double g10 = scale * k10.y * (tb - k10.x);
  const double g01 = scale * k01.y * (tb - k01.x);
  const double g11 = scale * k11.y * (tb - k11.x);
  return make_double2(-c.ay * g00 + c.ay * g10 - c.wy * g01 + c.wy * g11,
                      -c.ax * g00 - c.wx * g10 + c.ax * g01 + c.wx * g11);
}

__global__ void __launch_bounds__(kEvBlock, 8) k_bwd_event(
    const uint2* __restrict__ sorted, const uint64_t* __restrict__ ev_off, WinParams P,
    TileParams TP, const uint32_t* __restrict__ tile_ptr, const float2* __restrict__ flows32,
    const FwdRec* __restrict__ recs, uint64_t n_total, const double2* __restrict__ coef,
    const double* __restrict__ scale_tab, const int* __restrict__ no_surv,
    const uint32_t* __restrict__ sorted_keys, const uint32_t* __restrict__ bin_ptr,
    const uint32_t* __restrict__ srcbase, uint4* __restrict__ srcrec, float2* __restrict__ bwd,
    uint32_t* __restrict__ gmax) {
  __shared__ double es[kMaxRefs];
  __shared__ uint32_t erel[kMaxRefs];
  for (int i = threadIdx.x; i <= P.B; i += blockDim.x) {
    es[i] = P.es[i];
    erel[i] = P.erel[i];
  }
  __syncthreads();
  const int w = blockIdx.y;
  if (no_surv[w]) return;
  const uint64_t base = ev_off[w];
  const uint64_t n = tile_ptr[(size_t)w * (TP.nT + 1) + TP.nT];
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const FwdRec* rk = recs + base + k;  // + r * n_total
  // sink values: bwd[(r - 1) * n_total + slot] for the sink at reference r in
  // 1..B-1 (each is the sink of exactly one bin: r - 1 if r <= j, else r); the
  // source-pixel sink of bin j goes with the packed event to srcrec at its
  // (bin, tile, time) position (k_src_base)
  const int B = P.B, R = B + 1, W = P.W, H = P.H, HW = P.HW;
  const uint2 e = sorted[base + k];
  const uint32_t dt_us = ev_dt(e);
  const int j = bin_of(dt_us, erel, B);
  uint4* src_out;
  {
    const uint32_t S = sorted_keys[base + k];
    const uint32_t b0 = bin_ptr[((size_t)w * TP.nT + S) * (B + 1) + j];
    src_out = srcrec + base + srcbase[((size_t)w * B + j) * TP.nT + S] + ((uint32_t)k - b0);
  }
  if (rk[0].cell == kDead) {  // masked event: contributes nothing (engine.hpp:564)
    *src_out = make_uint4(e.x, e.y, 0u, 0u);
    return;
  }
  const int ox = W >= 2 ? 1 : 0, oy = H >= 2 ? 1 : 0;
  const double t = dm((double)dt_us, 1e-6);
  const int pol = ev_pol(e);
  const double2* cpw = coef + (size_t)w * R * 2 * HW + pol;  // + r*2*HW, [px][pol]
  const double* sc = scale_tab + (size_t)w * R;
  const float2* fl = flows32 + (size_t)w * B * HW;
  float2* bo = bwd + base + k;  // + i * n_total
  const double iwin = P.inv_window;  // same tb formula as k_fwd_owner
  auto tb_of = [&](int r) { return fabs(t - es[r]) * iwin; };

  float gm = 0.f;  // max |value| written by this event
  double2 gb, gf;
  {
    const CellW c = decode(rk[0]);
    gb = pos_grad_w(cpw, W, ox, oy, c, tb_of(0), sc[0]);
  }
  {
    const CellW c = decode(rk[(size_t)B * n_total]);
    gf = pos_grad_w(cpw + (size_t)B * 2 * HW, W, ox, oy, c, tb_of(B), sc[B]);
  }
  // the records stream from HBM and each step starts by decoding its record:
  // pull the next step's record into L2 one step ahead (no registers held)
  auto ref_at = [&](int s) { return s < j ? s + 1 : B - 1 - (s - j); };
  if (B > 1) asm volatile("prefetch.global.L2 [%0];" ::"l"(rk + (size_t)ref_at(0) * n_total));
  for (int s = 0; s < B - 1; ++s) {
    if (s + 1 < B - 1)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(rk + (size_t)ref_at(s + 1) * n_total));
    const bool back = s < j;
    const int i = back ? s : B - 1 - (s - j);
    const int r = back ? i + 1 : i;
    const double dt = back ? es[i] - es[i + 1] : es[i + 1] - es[i];
    const CellW c = decode(rk[(size_t)r * n_total]);
    const double2 g = back ? gb : gf;
    const float2 o = make_float2((float)(dt * g.x), (float)(dt * g.y));
    bo[(size_t)(r - 1) * n_total] = o;
    gm = fmaxf(gm, fmaxf(fabsf(o.x), fabsf(o.y)));
    // (I + dt J_i)^T g + d[r]   (warp.hpp:91-94, engine.hpp:490-491); the flow
    // Jacobian from the fp32 copy of the flows: dt J enters next to the identity,
    // so its 2^-24 relative error stays ~1e-7 of the adjoint, within the
    // gradient tolerance, and the 8 B pixel halves the gathers' sectors
    const int i00 = c.y0 * W + c.x0;
    const float2* f = fl + (size_t)i * HW;
    const float2 a = __ldg(f + i00), b = __ldg(f + i00 + ox);
    const float2 d0 = __ldg(f + i00 + oy * W), d1 = __ldg(f + i00 + oy * W + ox);
    const double dux = c.ay * ((double)b.x - a.x) + c.wy * ((double)d1.x - d0.x);
    const double duy = c.ax * ((double)d0.x - a.x) + c.wx * ((double)d1.x - b.x);
    const double dvx = c.ay * ((double)b.y - a.y) + c.wy * ((double)d1.y - d0.y);
    const double dvy = c.ax * ((double)d0.y - a.y) + c.wx * ((double)d1.y - b.y);
    const double2 d = pos_grad_w(cpw + (size_t)r * 2 * HW, W, ox, oy, c, tb_of(r), sc[r]);
    const double nx = g.x * (1.0 + dt * dux) + g.y * dt * dvx + d.x;
    const double ny = g.y * (1.0 + dt * dvy) + g.x * dt * duy + d.y;
    if (back) gb = make_double2(nx, ny); else gf = make_double2(nx, ny);
  }
  const double cb = es[j] - t, cf = es[j + 1] - t;
  const float2 o = make_float2((float)(cb * gb.x + cf * gf.x), (float)(cb * gb.y + cf * gf.y));
  *src_out = make_uint4(e.x, e.y, __float_as_uint(o.x), __float_as_uint(o.y));
  gm = fmaxf(gm, fmaxf(fabsf(o.x), fabsf(o.y)));
  // window max |value|: the fixed-point scale of the backward owner (cmax_cells.cu)
  const unsigned am = __activemask();
  const uint32_t mb = __reduce_max_sync(am, __float_as_uint(gm));
  if ((threadIdx.x & 31) == __ffs(am) - 1) atomicMax(gmax + w, mb);
  (void)H;
}

// ---------------------------------------------------------------------------
// launchers

TileParams make_tiles(const WinParams& P, uint64_t max_n) {
  TileParams TP;
  TP.ntx = (P.W + kSortTile - 1) / kSortTile;
  TP.nty = (P.H + kSortTile - 1) / kSortTile;
  TP.nT = TP.ntx * TP.nty;
  TP.otx = (P.W + kOwnW - 1) / kOwnW;
  TP.oty = (P.H + kOwnH - 1) / kOwnH;
  TP.oT = TP.otx * TP.oty;
  // chunk size: the largest power of two <= kChunk that still gives the sort
  // kernels >= 4 CTAs per SM over the batch (small batches, e.g. config B)
  int chunk = kChunk;
  while (chunk > 1024 &&
         (double)((max_n + chunk - 1) / chunk) * P.n_windows < 4.0 * 148.0)
    chunk /= 2;
  TP.chunk = chunk;
  TP.nchunks = (int)std::max<uint64_t>(1, (max_n + chunk - 1) / chunk);
  return TP;
}

static void set_smem(const void* fn, size_t bytes, size_t* have) {
  if (bytes > 48 * 1024 && bytes > *have) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    *have = bytes;
  }
}

void launch_stage_pack(cudaStream_t s, const evcm_event* ev, const uint64_t* ev_off,
                       const WinParams& P, uint64_t max_n, uint2* packed, unsigned long long* err) {
  const int blocks = (int)std::min<uint64_t>((max_n + kSortThreads - 1) / kSortThreads, 148 * 8);
  if (blocks == 0) return;
  count_launch();
  k_stage_pack<<<dim3(blocks, P.n_windows), kSortThreads, 0, s>>>(ev, ev_off, P, packed, err);
}

void launch_sort(cudaStream_t s, const uint2* packed, const uint64_t* ev_off, const WinParams& P,
                 const TileParams& TP, const double2* flows, uint64_t n_total, uint32_t* keys,
                 uint32_t* counts, uint32_t* tile_ptr, uint2* sorted, uint32_t* perm,
                 uint32_t* bin_ptr, uint32_t* srcbase, uint4* bbox, size_t n_bbox,
                 uint32_t* lcount, size_t n_lcount) {
  static size_t a1 = 0, a2 = 0;
  // many sort tiles: 4 warps per CTA, so the per-warp tile counts (2 B per tile)
  // leave room for more resident CTAs (measured: -9 % sort at 640x480)
  const int sc_threads = TP.nT > 2048 ? kScatterThreads / 2 : kScatterThreads;
  const size_t sc_smem = (size_t)(sc_threads / 32) * ((TP.nT + 7) & ~7) * 2;
  set_smem(reinterpret_cast<const void*>(k_key_hist), TP.nT * sizeof(uint32_t), &a1);
  static size_t a3 = 0;
  if (sc_threads == kScatterThreads)
    set_smem(reinterpret_cast<const void*>(k_sort_scatter<kScatterThreads / 32>), sc_smem, &a2);
  else
    set_smem(reinterpret_cast<const void*>(k_sort_scatter<kScatterThreads / 64>), sc_smem, &a3);
  const dim3 grid(TP.nchunks, P.n_windows);
  uint32_t* totals = keys + 2 * n_total;  // nw * nT scratch after the two key arrays
  double2* coarse = reinterpret_cast<double2*>(totals + (((size_t)P.n_windows * TP.nT + 3) & ~(size_t)3));
  count_launch();
  k_coarse_flow<<<148 * 4, 256, 0, s>>>(flows, P, TP, coarse, bbox, n_bbox, lcount, n_lcount);
  count_launch();
  k_key_hist<<<grid, kSortThreads, TP.nT * sizeof(uint32_t), s>>>(packed, ev_off, P, TP, coarse,
                                                                  keys, counts);
  count_launch();
  k_sort_colscan<<<dim3((TP.nT + 31) / 32, P.n_windows), 32 * kColSeg, 0, s>>>(counts, TP, totals);
  count_launch();
  k_sort_tilescan<<<P.n_windows, 1024, 0, s>>>(totals, TP, tile_ptr);
  count_launch();
if (sc_threads == kScatterThreads)
    k_sort_scatter<kScatterThreads / 32><<<grid, sc_threads, sc_smem, s>>>(packed, keys, ev_off, TP, counts, tile_ptr,
                                                        sorted, perm, keys + n_total);
  else
    k_sort_scatter<kScatterThreads / 64><<<grid, sc_threads, sc_smem, s>>>(packed, keys, ev_off, TP, counts, tile_ptr,
                                                        sorted, perm, keys + n_total);
  count_launch();
  k_bin_ptr<<<dim3((TP.nT + 7) / 8, P.n_windows), 256, 0, s>>>(sorted, ev_off, P, TP,
                                                                    tile_ptr, bin_ptr);
  if (srcbase) {
    count_launch();
    k_src_base<<<dim3(P.B, P.n_windows), kSrcBaseThreads, 0, s>>>(bin_ptr, P, TP, srcbase);
  }
}

void launch_traj_records(cudaStream_t s, const uint2* sorted, const uint64_t* ev_off,
                         const WinParams& P, const TileParams& TP, const uint32_t* tile_ptr,
                         const uint32_t* sorted_keys, uint64_t max_n, const double2* flows,
                         uint64_t n_total, FwdRec* recs, uint4* bbox, uint32_t* lcount,
                         uint16_t* lists) {
  static size_t a = 0;
  const size_t smem = kEvSmemHeader + sizeof(uint32_t) * (size_t)(P.B + 1) * kEvBlock;
  set_smem(reinterpret_cast<const void*>(k_traj_records), smem, &a);
  // shared-memory carveout: just what the register-limited 9 resident CTAs need
  // (+1 KB reserved each), the rest of the 256 KB stays L1 for the flow gathers
  // (the driver's default carveout measured 2 % slower)
  static size_t carved = 0;
  if (smem != carved) {
    const int pct = (int)std::min<size_t>(100, (9 * (smem + 1024) * 100 + 228 * 1024 - 1) / (228 * 1024));
    cudaFuncSetAttribute(reinterpret_cast<const void*>(k_traj_records),
                         cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    carved = smem;
  }
  if (max_n > 0) {
    count_launch();
    k_traj_records<<<dim3((unsigned)((max_n + kEvBlock - 1) / kEvBlock), P.n_windows), kEvBlock,
                     smem, s>>>(sorted, ev_off, P, TP, tile_ptr, sorted_keys, flows, n_total, recs,
                                bbox);
  }
  count_launch();
  k_build_lists<<<dim3((TP.nT + 127) / 128, 2 * P.B + 1, P.n_windows), 128, 0, s>>>(bbox, P, TP,
                                                                                    lcount, lists);
}

void launch_bwd_event(cudaStream_t s, const uint2* sorted, const uint64_t* ev_off,
                      const WinParams& P, const TileParams& TP, const uint32_t* tile_ptr,
                      uint64_t max_n, const float2* flows32, const FwdRec* recs, uint64_t n_total,
                      const double2* coef, const double* scale, const int* no_surv,
                      const uint32_t* sorted_keys, const uint32_t* bin_ptr, const uint32_t* srcbase,
                      uint4* srcrec, float2* bwd, uint32_t* gmax) {
  cudaMemsetAsync(gmax, 0, (size_t)P.n_windows * sizeof(uint32_t), s);
  if (max_n == 0) return;
  count_launch();
  k_bwd_event<<<dim3((unsigned)((max_n + kEvBlock - 1) / kEvBlock), P.n_windows), kEvBlock, 0, s>>>(
      sorted, ev_off, P, TP, tile_ptr, flows32, recs, n_total, coef, scale, no_surv, sorted_keys,
      bin_ptr, srcbase, srcrec, bwd, gmax);
}

}  // namespace evcm_b200
