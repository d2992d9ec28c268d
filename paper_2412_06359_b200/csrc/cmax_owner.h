// Owner-computes pipeline launchers (cmax_owner.cu).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/evcm_cuda.h"
#include "cmax_device.cuh"

namespace evcm_b200 {

constexpr int kSortTile = 8;       // sort tiles: 8x8 px of the position at the middle reference
constexpr int kOwnW = 32;          // owner tiles: 32x16 px of the IWE stack / gradient planes
constexpr int kOwnH = 16;
constexpr int kChunk = 8192;       // max events per sort chunk (one CTA); TileParams.chunk adapts
constexpr int kSortThreads = 512;  // key/histogram CTA size
constexpr int kScatterThreads = 256;  // 8 warps x 1024 events per scatter chunk
// sort tiles per window: the scatter keeps nW x nT u16 counters in shared memory
// (nW = 4 warps above 2048 tiles: 4 x 28000 x 2 B = 219 KB of the 227 KB), the
// owner lists store u16 tile ids. 28000 tiles: up to 1280 x 1024 (or 1600 x 1120)
constexpr int kMaxTiles = 28000;
constexpr int kListCapO = 128;     // source-list capacity per (window, slot, owner tile)

struct TileParams {
  int ntx, nty, nT;  // sort tiles
  int otx, oty, oT;  // owner tiles
  int nchunks;       // sort chunks per window (max over the batch)
  int chunk;         // events per sort chunk: 1024..kChunk, enough CTAs for the batch
};

// Per (event, reference) splat record, 16 B. cell = x0 | y0 << 16 | negative
// polarity << 31 (0xffffffff: masked event); dt = t_us - t0; fx, fy = the
// compressed bilinear fractions (cmax_owner.cu: compress_frac).
struct __align__(16) FwdRec {
  uint32_t cell;
  uint32_t dt;
  float fx, fy;
};

TileParams make_tiles(const WinParams& P, uint64_t max_n);
void launch_stage_pack(cudaStream_t s, const evcm_event* ev, const uint64_t* ev_off,
                       const WinParams& P, uint64_t max_n, uint2* packed, unsigned long long* err);
// keys: 2 * n_total + n_windows * nT entries (unsorted keys, keys in sorted
// order, per-tile totals)
void launch_sort(cudaStream_t s, const uint2* packed, const uint64_t* ev_off, const WinParams& P,
                 const TileParams& TP, const double2* flows, uint64_t n_total, uint32_t* keys,
                 uint32_t* counts, uint32_t* tile_ptr, uint2* sorted, uint32_t* perm,
                 uint32_t* bin_ptr, uint32_t* srcbase = nullptr, uint4* bbox = nullptr,
                 size_t n_bbox = 0, uint32_t* lcount = nullptr, size_t n_lcount = 0);
void launch_traj_records(cudaStream_t s, const uint2* sorted, const uint64_t* ev_off,
                         const WinParams& P, const TileParams& TP, const uint32_t* tile_ptr,
                         const uint32_t* sorted_keys, uint64_t max_n, const double2* flows,
                         uint64_t n_total, FwdRec* recs, uint4* bbox, uint32_t* lcount,
                         uint16_t* lists);
void launch_bwd_event(cudaStream_t s, const uint2* sorted, const uint64_t* ev_off,
                      const WinParams& P, const TileParams& TP, const uint32_t* tile_ptr,
                      uint64_t max_n, const float2* flows32, const FwdRec* recs, uint64_t n_total,
                      const double2* coef, const double* scale, const int* no_surv,
                      const uint32_t* sorted_keys, const uint32_t* bin_ptr, const uint32_t* srcbase,
                      uint4* srcrec, float2* bwd, uint32_t* gmax);
// Owner kernels with exact fixed-point shared-memory accumulation (cmax_cells.cu).
void launch_fwd_cells(cudaStream_t s, const uint64_t* ev_off, const WinParams& P,
                      const TileParams& TP, const uint32_t* tile_ptr, const FwdRec* recs,
                      uint64_t n_total, const uint4* bbox, const uint32_t* lcount,
                      const uint16_t* lists, const uint2* ranges, double2* coef, double2* stack_out,
                      double* part_acc, unsigned long long* part_act, int groups);
// CTA groups of the owner kernels: split the references (forward) / bins
// (backward) over `groups` CTAs per (tile, window) when tiles x windows alone
// fill fewer than ~4 waves of 2 CTAs per SM (EVCM_FWD_GROUPS / EVCM_BWD_GROUPS
// override, for measurements)
int owner_groups(const TileParams& TP, const WinParams& P, bool backward);
void launch_bwd_cells(cudaStream_t s, const uint2* sorted, const uint64_t* ev_off,
                      const WinParams& P, const TileParams& TP, const uint32_t* tile_ptr,
                      const uint32_t* bin_ptr, const FwdRec* recs, const float2* bwd,
                      uint64_t n_total, const uint32_t* gmax, const uint4* bbox,
                      const uint32_t* lcount, const uint16_t* lists, const uint2* ranges,
                      const uint32_t* srcbase, const uint4* srcrec, const int* no_surv,
                      const double* depth, const uint8_t* mask, const double* pose_tab,
                      const double* K, double* d_depth, double* pose_part, double* grad_out,
                      int groups, double* dbin);
// Per (window, slot, owner tile) list: precomputed candidate ranges (kListCapO + 2
// uint2 entries; see cmax_cells.cu)
void launch_ranges(cudaStream_t s, const uint32_t* lcount, const uint16_t* lists,
                   const uint32_t* tile_ptr, const uint32_t* bin_ptr, const uint32_t* srcbase,
                   const WinParams& P, const TileParams& TP, uint2* ranges);

}  // namespace evcm_b200
