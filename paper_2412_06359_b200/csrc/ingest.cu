// Event ingestion on the device: the EVT1 wire format
// (io.hpp:106-172) carries 16 B records byte-identical to evcm::Event, so a
// file's payload is copied to the device untouched; these kernels validate it
// and cut it into the windows of the batched chain.
//
//   k_validate_events   the per-record checks of read_events (io.hpp:134-144) and
//                       EventSlice::validate (types.hpp:137-161): the first violating
//                       record, and for it the first failed check in the reference's
//                       order -- coordinate, polarity, timestamp order, [window]
//   k_window_offsets    offsets[w] = lower_bound(t, t0 + w * window_us) over the
//                       time-sorted events (one binary search per boundary)
#include <cstdint>

#include "cmax_kernels.h"

namespace evcm_b200 {

namespace {

__global__ void k_validate_events(const evcm_event* __restrict__ ev, uint64_t n, int W, int H,
                                  int check_window, uint64_t t_lo, uint64_t t_hi,
                                  unsigned long long* __restrict__ first) {
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const evcm_event e = ev[k];
    unsigned code = 0;
    if (e.x >= W || e.y >= H) code = 3;                            // CoordinateRangeError
    else if (e.p != 1 && e.p != -1) code = 4;                      // InvalidPolarityError
    else if (k > 0 && e.t_us < ev[k - 1].t_us) code = 5;           // UnsortedEventsError
    else if (check_window && (e.t_us < t_lo || e.t_us >= t_hi)) code = 6;  // TimeRangeError
    if (code) atomicMin(first, ((unsigned long long)k << 4) | code);
  }
}

__global__ void k_window_offsets(const evcm_event* __restrict__ ev, uint64_t n, uint64_t t0,
                                 uint64_t window_us, int n_windows, uint64_t* __restrict__ offsets) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w > n_windows) return;
  const uint64_t t = t0 + (uint64_t)w * window_us;
  uint64_t lo = 0, hi = n;  // first k with ev[k].t_us >= t
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (ev[mid].t_us < t) lo = mid + 1; else hi = mid;
  }
  offsets[w] = lo;
}

}  // namespace

void launch_validate_events(cudaStream_t s, const evcm_event* ev, uint64_t n, int W, int H,
                            int check_window, uint64_t t_lo, uint64_t t_hi,
                            unsigned long long* first) {
  if (n == 0) return;
  count_launch();
  const unsigned blocks = (unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 8);
  k_validate_events<<<blocks, 256, 0, s>>>(ev, n, W, H, check_window, t_lo, t_hi, first);
}

void launch_window_offsets(cudaStream_t s, const evcm_event* ev, uint64_t n, uint64_t t0,
                           uint64_t window_us, int n_windows, uint64_t* offsets) {
  count_launch();
  k_window_offsets<<<(n_windows + 1 + 127) / 128, 128, 0, s>>>(ev, n, t0, window_us, n_windows,
                                                              offsets);
}

}  // namespace evcm_b200
