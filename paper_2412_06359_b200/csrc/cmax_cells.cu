// Fast owner kernels (sm_100a): the forward (IWE stack tile + focus-loss
// partials + coefficient planes) and backward (flow-gradient tile + fused
// depth_pose_to_flows_backward) of the owner-computes pipeline.
//
// Accumulation is exact 64-bit FIXED POINT in shared memory, built from native
// 32-bit integer atomics. sm_100 has no native fp64 (or f32 / u64) shared atomic
// add -- the compiler emits ATOMS.CAST.SPIN compare-and-swap loops (0.41 T adds/s
// measured) -- while 32-bit ATOMS.ADD runs at 2.1 T lane-ops/s
// (tools/microbench/atoms_u32.cu); native L2 fp64 reductions top out near
// 250 G adds/s (tools/microbench/red_cluster.cu). A value v is added as
// q = round(v * 2^k) (u64 or two's-complement s64): the low word with
// atomicAdd (its return value gives the carry) and the high word plus the carry
// with a second atomicAdd. Integer addition is associative, so the sums are
// BIT-IDENTICAL whatever the order of the atomics: the fast mode is
// deterministic.
//
// Precision: the IWE weights w and w*tb lie in [0, 1] and use k = 50 fraction
// bits (2^-51 absolute rounding per term) whenever the reference's candidate
// count T of the owner tile is below 2^13 (T bounds every pixel's weight sum);
// denser tiles get k = 63 - bits(T), so the sums can never wrap. The
// reference's sensitive quantity is the splat_position_grad factor
// a*inv*(tb - a), largest where C ~ eps = 1e-9; there a term's relative error
// is ~2^-51 / 1e-9 ~ 4e-7. Gradient terms w*g use k = kbits - e with
// 2^e > max|g| of the window (k_bwd_event) and kbits <= 49 chosen from the
// largest candidate count of the CTA's groups. n_active is exact: a pixel is
// active iff some contribution has w > 0 (weights below the fixed-point
// resolution are flagged).
//
// Candidates: warp 0 stages every record range of the owner tile (a sort tile's
// events at this reference) into shared memory with one cp.async.bulk (TMA bulk
// copy) each, all completing on one mbarrier; every thread then adds its
// candidates' corner contributions.
//
// References (proj/include/evcm): splat_bilinear / IweStack warp.hpp:147-193,
// splat_event_refs engine.hpp:365-374, refresh_active warp.hpp:186-192,
// reference_loss warp.hpp:299-312, splat_position_grad factors warp.hpp:334-358,
// BufferGradSink::add warp.hpp:391-407, depth_pose_to_flows_backward
// geometry.hpp:279-325.
#include <cstdint>
#include <cstdlib>
#include <algorithm>

#include "cmax_device.cuh"
#include "cmax_kernels.h"
#include "cmax_owner.h"
#include "cmax_owner_dev.cuh"

namespace evcm_b200 {

void count_launch();  // cmax_kernels.cu

using namespace owner_dev;

namespace {

constexpr int kThreads = 512;                      // 16 warps
constexpr int kWarps = kThreads / 32;
constexpr int kBatchCap = 3 * kListCapO;           // sort-tile ranges per batch
// accumulator row stride = 8 (mod 32): an 8 x 8 pixel block (the cells of one
// sort tile's events, which share a warp) covers all 32 shared-memory banks
constexpr int kRowW = kOwnW + 8;
constexpr int kPlane = kOwnH * kRowW;              // words per accumulator plane

// ---- mbarrier + TMA bulk copy (cp.async.bulk) --------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// the single arrival of a phase, announcing `bytes` of bulk-copy transactions
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// try_wait with a suspend-time hint: the waiting warp is parked by the hardware
// until the phase completes (or the hint expires), instead of polling -- waiting
// warps leave the issue slots to the CTAs that still compute
__device__ __forceinline__ bool mbar_try_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait_sleep(bar, parity)) {
  }
}
// global -> shared bulk copy (16 B aligned, size a multiple of 16) completing on bar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// order earlier generic-proxy shared accesses before later bulk copies into them
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// barrier among the `count` threads of the consumer warps (id 1; id 0 is __syncthreads)
__device__ __forceinline__ void consumer_sync(int count) {
  asm volatile("bar.sync 1, %0;" ::"r"(count) : "memory");
}
// Warp sums of N components at once by transposition: each halving step trades
// half of the remaining components with the partner lane (N - 1 + log2(32 / N)
// double shuffles instead of 5 N); lane l returns the sum of component
// (l >> (5 - log2 N)) & (N - 1) (lanes with l % (32 / N) == 0 hold distinct
// components). Fixed order: deterministic.
template <int N>
__device__ __forceinline__ double warp_comp_sum(double (&c)[N], int lane) {
#pragma unroll
  for (int h = N / 2, off = 16; h >= 1; h >>= 1, off >>= 1) {
    const bool up = lane & off;
#pragma unroll
    for (int k = 0; k < h; ++k) {
      const double mine = up ? c[h + k] : c[k], other = up ? c[k] : c[h + k];
      c[k] = mine + __shfl_xor_sync(0xffffffffu, other, off);
    }
  }
  double v = c[0];
#pragma unroll
  for (int off = 16 / N; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}
__device__ __forceinline__ uint32_t warp_sum_u32(uint32_t v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// Candidate source ranges of the current batch: list[l] = sort tile, pre[l] =
// virtual index of its first candidate, rng[l] = its first record slot;
// seg_end[s] = virtual end of segment s.
struct Batch {
  uint16_t list[kBatchCap];
  uint32_t pre[kBatchCap + 1];
  uint32_t rng[kBatchCap];
  uint32_t seg_end[3];
  int nl;
  int seg, S;  // slow-path cursor (seg < 0: fast path not tried yet)
  int more;    // another batch follows
};

// Next batch of candidate ranges (warp 0, collective). Fast path: every
// segment's precomputed owner list fits (k_build_lists) -> one batch with all
// segments concatenated. Otherwise each segment's sort-tile boxes are scanned
// in chunks of <= kBatchCap hits, one segment per batch.
// list_at(s): index of (window, slot of segment s, owner tile) in lcount/lists;
// box_at(s): first box of (window, slot of segment s); lohi(s, S): record range.
template <int NSEG, typename ListAt, typename BoxAt, typename Lohi>
__device__ void next_batch(Batch& bt, const uint32_t* __restrict__ lcount,
                           const uint16_t* __restrict__ lists, const uint4* __restrict__ bbox,
                           int nT, int ox0, int oy0, ListAt&& list_at, BoxAt&& box_at,
                           Lohi&& lohi) {
  const int lane = threadIdx.x & 31;
  if (bt.seg < 0) {
    uint32_t cnt[NSEG];
    bool fit = true;
#pragma unroll
    for (int s = 0; s < NSEG; ++s) {
      cnt[s] = lcount[list_at(s)];
      fit = fit && cnt[s] <= (uint32_t)kListCapO;
    }
    if (fit) {
      int n = 0;
      int lend[NSEG];
#pragma unroll
      for (int s = 0; s < NSEG; ++s) {
        const uint16_t* src = lists + (size_t)list_at(s) * kListCapO;
        for (uint32_t e = lane; e < cnt[s]; e += 32) bt.list[n + e] = src[e];
        n += (int)cnt[s];
        lend[s] = n;
      }
      __syncwarp();
      int s_cur = 0;
      warp_ranges(0, n, 0u, bt.pre, bt.rng, [&](int l) {
        int s = 0;
#pragma unroll
        for (int q = 0; q < NSEG - 1; ++q) s += (l >= lend[q]) ? 1 : 0;
        return lohi(s, (int)bt.list[l]);
      });
      (void)s_cur;
      if (lane == 0) {
#pragma unroll
        for (int s = 0; s < NSEG; ++s) bt.seg_end[s] = bt.pre[lend[s]];
        bt.nl = n;
        bt.more = 0;
        bt.seg = NSEG;
      }
      __syncwarp();
      return;
    }
    if (lane == 0) {
      bt.seg = 0;
      bt.S = 0;
    }
    __syncwarp();
  }
  // slow path: scan the boxes of segment bt.seg from sort tile bt.S
  const int lx = ox0 - 1, hx = ox0 + kOwnW - 1, ly = oy0 - 1, hy = oy0 + kOwnH - 1;
  int seg = bt.seg, S0 = bt.S, fill = 0;
  while (seg < NSEG && fill == 0) {
    const uint4* bb = bbox + box_at(seg);
    while (S0 < nT && fill <= kBatchCap - 32) {
      const int S = S0 + lane;
      bool hit = false;
      if (S < nT) {
        const uint4 b = __ldg(bb + S);
        if (b.x != 0xffffffffu) {
          const int mnx = (int)b.x, mny = (int)b.y;
          const int mxx = 0xffff - (int)b.z, mxy = 0xffff - (int)b.w;
          hit = !(mxx < lx || mnx > hx || mxy < ly || mny > hy);
        }
      }
      const unsigned hits = __ballot_sync(kFull, hit);
      if (hit) bt.list[fill + __popc(hits & ((1u << lane) - 1u))] = (uint16_t)S;
      fill += __popc(hits);
      S0 += 32;
    }
    if (fill == 0 || S0 >= nT) {
      if (fill == 0) {
        ++seg;
        S0 = 0;
      }
    }
    if (fill > 0) break;
  }
  __syncwarp();
  const int bseg = seg;
  if (fill > 0 && S0 >= nT) {  // this segment is finished after the batch
    ++seg;
    S0 = 0;
  }
  warp_ranges(0, fill, 0u, bt.pre, bt.rng, [&](int l) { return lohi(bseg, (int)bt.list[l]); });
  if (lane == 0) {
    const uint32_t tot = bt.pre[fill];
#pragma unroll
    for (int s = 0; s < NSEG; ++s) bt.seg_end[s] = (s < bseg) ? 0u : tot;
    bt.nl = fill;
    bt.seg = seg;
    bt.S = S0;
    bt.more = seg < NSEG;
  }
  __syncwarp();
}

// Warp-level stream compaction: the warp scans slots [v0, n) 32 at a time with
// stride kStride, `hit(v)` classifies slot v, and `work(v)` runs only on full
// warps of hits (queued in the warp's 64-entry shared queue), so the heavy
// corner path does not run at the density of the (about 50 %) hits.
template <int kStride, typename Hit, typename Work>
__device__ __forceinline__ void compacted(uint32_t v0, uint32_t n, uint16_t* q, Hit&& hit,
                                          Work&& work) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  int qn = 0;
  for (uint32_t vb = v0; vb < n; vb += kStride) {
    const uint32_t v = vb + lane;
    const bool h = v < n && hit(v);
    const unsigned bal = __ballot_sync(0xffffffffu, h);
    if (h) q[qn + __popc(bal & lt)] = (uint16_t)v;
    qn += __popc(bal);
    __syncwarp();
    if (qn >= 32) {
      work((uint32_t)q[lane]);
      __syncwarp();
      if (lane < qn - 32) q[lane] = q[lane + 32];
      qn -= 32;
      __syncwarp();
    }
  }
  if (lane < qn) work((uint32_t)q[lane]);
  __syncwarp();
}

// Exact fixed-point accumulation into a (lo, hi) pair of 32-bit shared words at
// shared-window addresses a_lo / a_hi: two native ATOMS.ADD, the first one's
// return value giving the carry (add.cc / addc) into the second.
__device__ __forceinline__ void fx_add(uint32_t a_lo, uint32_t a_hi, unsigned long long q) {
  asm volatile(
      "{\n"
      ".reg .u32 lo, hi, old, t;\n"
      "mov.b64 {lo, hi}, %2;\n"
      "atom.shared.add.u32 old, [%0], lo;\n"
      "add.cc.u32 t, old, lo;\n"
      "addc.u32 hi, hi, 0;\n"
      "red.shared.add.u32 [%1], hi;\n"
      "}\n" ::"r"(a_lo),
      "r"(a_hi), "l"(q)
      : "memory");
}
// 1 / x to within 1 ulp (MUFU.RCP64H seed + two Newton steps), for x > 0 normal:
// the epilogues' reciprocals feed the loss, coefficients and gradients, which are
// tolerance-checked (1e-5), so they need not be the correctly rounded 1.0 / x
// (__drcp_rn is a longer sequence with a slow path)
__device__ __forceinline__ double rcp_fast(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
// round-to-nearest-even integer conversions by the 2^52 "magic number": adding
// 2^52 (1.5 * 2^52) to x leaves round(x) in the low mantissa bits -- one DADD and
// an integer subtract instead of the F2I.64 conversion (a quarter-rate pipe).
// Identical to __double2ull_rn / __double2ll_rn on the stated ranges.
__device__ __forceinline__ unsigned long long fx_q(double x) {  // 0 <= x < 2^52
  return (unsigned long long)__double_as_longlong(__dadd_rn(x, 0x1.0p52)) - 0x4330000000000000ull;
}
__device__ __forceinline__ unsigned long long fx_qs(double x) {  // |x| < 2^51, two's complement
  return (unsigned long long)__double_as_longlong(__dadd_rn(x, 0x1.8p52)) - 0x4338000000000000ull;
}
// bits needed to count t: fixed-point sums of t terms bounded by 2^k need k + bits
__device__ __forceinline__ int bits_for(uint32_t t) { return 32 - __clz(t); }

__device__ __forceinline__ unsigned long long fx_read(const uint32_t* plo, const uint32_t* phi) {
  return ((unsigned long long)*phi << 32) | *plo;
}

}  // namespace

// Clip range l of the batch to the round [rb, rb + cap): [lo, hi) virtual.
__device__ __forceinline__ void clip(const Batch& bt, int l, uint32_t rb, uint32_t cap,
                                     uint32_t& lo, uint32_t& hi) {
  lo = max(bt.pre[l], rb);
  hi = min(bt.pre[l + 1], rb + cap);
}

// ---------------------------------------------------------------------------
// Precomputed candidate ranges (k_ranges): per (window, slot, owner tile) list,
// kRgCap uint2 entries: e[0] = {count (kOverflow: the list overflowed), total},
// e[1 + l] = {first record slot, exclusive prefix of the lengths}. The
// producers fetch a whole list with one cp.async.bulk.

constexpr int kRgCap = kListCapO + 2;  // 130 entries = 1040 B (a multiple of 16)
constexpr uint32_t kOverflow = 0xffffffffu;

// Ranges of up to two lists concatenated in virtual candidate space: ranges
// [0, n0) from a (kind 0), then [n0, n0 + n1) from b (kind 1).
struct Cat {
  const uint2* a;
  const uint2* b;
  int n0, n1;
  uint32_t t0, t1;
  __device__ __forceinline__ int nl() const { return n0 + n1; }
  __device__ __forceinline__ uint32_t total() const { return t0 + t1; }
  __device__ __forceinline__ uint32_t pre(int l) const {
    return l < n0 ? a[1 + l].y : (l < n0 + n1 ? t0 + b[1 + l - n0].y : t0 + t1);
  }
  __device__ __forceinline__ uint32_t rng(int l) const { return l < n0 ? a[1 + l].x : b[1 + l - n0].x; }
};
__device__ __forceinline__ Cat make_cat(const uint2* a, const uint2* b) {
  Cat c;
  c.a = a;
  c.b = b;
  c.n0 = a ? (int)a[0].x : 0;
  c.t0 = a ? a[0].y : 0u;
  c.n1 = b ? (int)b[0].x : 0;
  c.t1 = b ? b[0].y : 0u;
  return c;
}
// the next batch of an overflowed list, via next_batch, as a Cat view in fb
__device__ __forceinline__ void batch_to_view(const Batch& bt, uint2* fb) {
  const int lane = threadIdx.x & 31;
  for (int l = lane; l < bt.nl; l += 32) fb[1 + l] = make_uint2(bt.rng[l], bt.pre[l]);
  if (lane == 0) fb[0] = make_uint2((uint32_t)bt.nl, bt.nl > 0 ? bt.pre[bt.nl] : 0u);
  __syncwarp();
}

__global__ void k_ranges(const uint32_t* __restrict__ lcount, const uint16_t* __restrict__ lists,
                         const uint32_t* __restrict__ tile_ptr, const uint32_t* __restrict__ bin_ptr,
                         const uint32_t* __restrict__ srcbase, WinParams P, TileParams TP,
                         uint2* __restrict__ ranges) {
  const int lane = threadIdx.x & 31;
  const size_t gid = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int NS = 2 * P.B + 1, R = P.B + 1;
  if (gid >= (size_t)P.n_windows * NS * TP.oT) return;
  const size_t ws = gid / TP.oT;
  const int slot = (int)(ws % NS), w = (int)(ws / NS);
  const uint32_t cnt = lcount[gid];
  uint2* out = ranges + gid * kRgCap;
  if (cnt > (uint32_t)kListCapO) {
    if (lane == 0) out[0] = make_uint2(kOverflow, 0u);
    return;
  }
  const uint32_t* tp = tile_ptr + (size_t)w * (TP.nT + 1);
  const uint32_t* bp = bin_ptr + (size_t)w * TP.nT * (P.B + 1);
  const int sb = slot - R;  // source slot: bin
  const uint32_t* src_b = srcbase + ((size_t)w * P.B + (sb >= 0 ? sb : 0)) * TP.nT;
  // first position and length of sort tile S's candidates: its records at the
  // reference (tile order), or the source sinks of its events of bin sb in the
  // (bin, tile, time) layout (k_src_base)
  auto lo_of = [&](uint32_t S) { return slot < R ? tp[S] : src_b[S]; };
  auto len_of = [&](uint32_t S) {
    return slot < R ? tp[S + 1] - tp[S]
                    : bp[(size_t)S * (P.B + 1) + sb + 1] - bp[(size_t)S * (P.B + 1) + sb];
  };
  if (cnt <= 32u) {
    // the candidates of consecutive sort tiles are contiguous (tile order in
    // both layouts), so the list is sorted (rank by counting, ids are distinct)
    // and every run S, S+1, ... becomes ONE range -- an owner tile's row of
    // sort tiles is one bulk copy instead of one per tile
    const uint32_t S = lane < (int)cnt ? lists[gid * kListCapO + lane] : 0xffffffffu;
    uint32_t rank = 0;
    for (uint32_t m = 0; m < cnt; ++m) rank += __shfl_sync(kFull, S, (int)m) < S ? 1u : 0u;
    // lane k gets the k-th smallest id: the lane whose rank is k
    uint32_t sk = 0xffffffffu;
    for (uint32_t m = 0; m < cnt; ++m) {
      const uint32_t rm = __shfl_sync(kFull, rank, (int)m), vm = __shfl_sync(kFull, S, (int)m);
      if (rm == (uint32_t)lane) sk = vm;
    }
    const uint32_t prev = __shfl_up_sync(kFull, sk, 1);
    const bool valid = lane < (int)cnt;
    const bool start = valid && (lane == 0 || sk != prev + 1u);
    const unsigned starts = __ballot_sync(kFull, start);
    const int nr = __popc(starts);
    // run of this start lane: [sk, last] with last = the id before the next start
    const int ridx = __popc(starts & ((1u << lane) - 1u));
    const unsigned later = starts & ~((2u << lane) - 1u);  // starts after this lane
    const int next_start = later ? __ffs(later) - 1 : (int)cnt;
    const uint32_t last = __shfl_sync(kFull, sk, max(next_start - 1, 0));
    uint32_t lo = 0, len = 0;
    if (start) {
      lo = lo_of(sk);
      len = lo_of(last) + len_of(last) - lo;
    }
    // prefix of the run lengths in run order (runs are in increasing lane order)
    uint32_t x = len;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (start) out[1 + ridx] = make_uint2(lo, x - len);
    const uint32_t tot = __shfl_sync(kFull, x, 31);
    if (lane == 0) out[0] = make_uint2((uint32_t)nr, tot);
    return;
  }
  uint32_t carry = 0;
  for (uint32_t l0 = 0; l0 < cnt; l0 += 32) {
    const uint32_t l = l0 + lane;
    uint32_t lo = 0, len = 0;
    if (l < cnt) {
      const uint32_t S = lists[gid * kListCapO + l];
      lo = lo_of(S);
      len = len_of(S);
    }
    uint32_t x = len;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (l < cnt) out[1 + l] = make_uint2(lo, carry + x - len);
    carry += __shfl_sync(kFull, x, 31);
  }
  if (lane == 0) out[0] = make_uint2(cnt, carry);
}

// ---------------------------------------------------------------------------
// forward: one CTA per (owner tile, window, reference group), the group's
// references [r0, r1) in order, warp specialised. References are independent
// here, so the groups only add CTAs when the tiles x windows alone leave SMs
// idle (owner_groups); the outputs do not depend on the grouping. Warp 0 (producer) builds each round's candidate ranges and
// stages them with cp.async.bulk into one of two buffers (full/empty mbarrier
// pair per buffer), running up to two rounds ahead; warps 1..16 (consumers, one
// pixel each in the pixel phase) accumulate a round, release its buffer and,
// after the last round of a reference, turn the tile into loss partials and
// coefficient planes.

constexpr int kCons = kThreads;                 // consumer threads (16 warps)
// forward consumers: 12 warps for the 512 pixels of a tile (the epilogue loops
// over them): measured -0.8 % at C and -2 % at B against 16 (8: +3 % at C); the
// consumers are bound by the shared-memory atomic unit, not by warp count
constexpr int kFwdWarps = 12;
constexpr int kFwdCons = 32 * kFwdWarps;
constexpr int kFwdThreads = kFwdCons + 32;      // + producer warp
constexpr int kStageP = 2304;                   // candidates per buffer

struct RoundDesc {
  uint32_t n;  // staged candidates
  int r;       // reference
  int last;    // last round of this reference
  int fb;      // fraction bits of this reference's sums (<= 50, see below)
};

template <bool kGrouped>
__global__ void __launch_bounds__(kFwdThreads, 2) k_fwd_cells(
    const uint64_t* __restrict__ ev_off, WinParams P, TileParams TP,
    const uint32_t* __restrict__ tile_ptr, const FwdRec* __restrict__ recs, uint64_t n_total,
    const uint4* __restrict__ bbox, const uint32_t* __restrict__ lcount,
    const uint16_t* __restrict__ lists, const uint2* __restrict__ ranges,
    double2* __restrict__ coef, double2* __restrict__ stack_out, double* __restrict__ part_acc,
    unsigned long long* __restrict__ part_act) {
  extern __shared__ __align__(16) unsigned char smem[];
  FwdRec* stage = reinterpret_cast<FwdRec*>(smem);                    // [2][kStageP]
  uint32_t* acc = reinterpret_cast<uint32_t*>(stage + 2 * kStageP);   // [pol][C, S][lo, hi][kPlane]
  uint32_t* flag = acc + 8 * kPlane;  // [kPlane] a w > 0 rounded to 0 in fixed point
  __shared__ Batch bt;
  __shared__ RoundDesc desc[2];
  __shared__ __align__(16) uint2 rv[2][kRgCap];    // prefetched ranges
  __shared__ __align__(16) uint2 fb[kBatchCap + 1];  // overflow-path ranges
  __shared__ __align__(8) uint64_t full[2], empty[2], rbar[2];
  __shared__ uint16_t wq[kFwdWarps][64];  // per-warp compaction queues
  __shared__ double s_red[2][kFwdWarps];
  __shared__ unsigned s_act[2][kFwdWarps];

  const int T = blockIdx.x, w = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int R = P.B + 1, NS = 2 * P.B + 1, W = P.W, H = P.H, HW = P.HW;
  const int r0 = kGrouped ? (int)blockIdx.z * R / (int)gridDim.z : 0;
  const int r1 = kGrouped ? ((int)blockIdx.z + 1) * R / (int)gridDim.z : R;
  const int ox0 = (T % TP.otx) * kOwnW, oy0 = (T / TP.otx) * kOwnH;
  const int ox = W >= 2 ? 1 : 0, oy = H >= 2 ? 1 : 0;
  const uint64_t base = ev_off[w];
  const uint32_t* tp = tile_ptr + (size_t)w * (TP.nT + 1);

  for (int i = tid; i < 9 * kPlane; i += kFwdThreads) acc[i] = 0u;
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    mbar_init(&empty[0], kFwdWarps);
    mbar_init(&empty[1], kFwdWarps);
    mbar_init(&rbar[0], 1);
    mbar_init(&rbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (wid == 0) {
    // ---------------- producer ----------------
    // ranges of reference r: precomputed list (prefetched one reference ahead)
    auto prefetch = [&](int r) {
      const size_t gid = ((size_t)w * NS + r) * TP.oT + T;
      const int q = (r - r0) & 1;
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_expect_tx(&rbar[q], kRgCap * (uint32_t)sizeof(uint2));
        bulk_g2s(rv[q], ranges + gid * kRgCap, kRgCap * (uint32_t)sizeof(uint2), &rbar[q]);
      }
    };
    uint32_t it = 0;
    // stage the rounds of one view; `final`: its last round ends reference r
    // fraction bits: a pixel's weight sum is bounded by the reference's candidate
    // count T (each record adds w <= 1), so T * 2^fb < 2^64 with fb <= 50
    const uint32_t nw_events = (uint32_t)(ev_off[w + 1] - base);
    auto rounds = [&](const Cat& cv, int r, bool final, uint32_t tbound) {
      const FwdRec* rr = recs + (size_t)r * n_total + base;
      const int fbits = min(50, 63 - bits_for(tbound));
      const int nl = cv.nl();
      const uint32_t total = cv.total();
      for (uint32_t rb = 0; rb < total || (rb == 0 && final); rb += kStageP) {
        const uint32_t n = total > rb ? min(total - rb, (uint32_t)kStageP) : 0u;
        const int b = it & 1;
        if (it >= 2) mbar_wait(&empty[b], ((it >> 1) - 1) & 1);
        FwdRec* sb = stage + b * kStageP;
        if (lane == 0) {
          desc[b].n = n;
          desc[b].r = r;
          desc[b].last = (final && rb + kStageP >= total) ? 1 : 0;
          desc[b].fb = fbits;
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive_expect_tx(&full[b], n * (uint32_t)sizeof(FwdRec));
        __syncwarp();
        int la = 0;  // first range ending after rb (prefixes are monotone)
        {
          int z = nl;
          while (la < z) {
            const int m = (la + z) >> 1;
            if (cv.pre(m + 1) > rb) z = m; else la = m + 1;
          }
        }
        for (int l = la + lane; l < nl && cv.pre(l) < rb + kStageP; l += 32) {
          const uint32_t lo = max(cv.pre(l), rb), hi = min(cv.pre(l + 1), rb + kStageP);
          if (lo < hi)
            bulk_g2s(sb + (lo - rb), rr + cv.rng(l) + (lo - cv.pre(l)),
                     (hi - lo) * (uint32_t)sizeof(FwdRec), &full[b]);
        }
        ++it;
        if (total == 0) break;
      }
    };
    prefetch(r0);
    for (int r = r0; r < r1; ++r) {
      if (r + 1 < r1) prefetch(r + 1);
      mbar_wait(&rbar[(r - r0) & 1], ((r - r0) >> 1) & 1);
      const uint2* v = rv[(r - r0) & 1];
      if (v[0].x != kOverflow) {
        rounds(make_cat(v, nullptr), r, true, v[0].y);
      } else {  // overflowed list: scan the sort-tile boxes batch by batch
        const size_t ws = (size_t)w * NS + r;
        if (lane == 0) bt.seg = -1;
        __syncwarp();
        int more = 1;
        while (more) {
          next_batch<1>(bt, lcount, lists, bbox, TP.nT, ox0, oy0,
                        [&](int) { return ws * TP.oT + T; }, [&](int) { return ws * TP.nT; },
                        [&](int, int S) { return make_uint2(tp[S], tp[S + 1]); });
          more = bt.more;
          batch_to_view(bt, fb);
          rounds(make_cat(fb, nullptr), r, !more, nw_events);  // total unknown: window bound
        }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int ct = tid - 32, cw = wid - 1;  // consumer thread / warp
  const uint32_t acc_s = smem_u32(acc);
  uint32_t it = 0;
  for (int r = r0; r < r1;) {
    const int b = it & 1;
    mbar_wait(&full[b], (it >> 1) & 1);
    const RoundDesc d = desc[b];
    const FwdRec* sb = stage + b * kStageP;
    const double esr = P.es[d.r], iwin = P.inv_window;
    const double fsc = ldexp(1.0, d.fb);  // 2^fb, exact scaling
    const double ifsc = ldexp(1.0, -d.fb);  // 2^-fb (exact; the epilogue's scale back)
    // splat_bilinear corners (warp.hpp:147-160) as exact fixed-point sums
    compacted<kFwdCons>(
        (uint32_t)cw * 32, d.n, wq[cw],
        [&](uint32_t v) {
          const uint32_t cell = sb[v].cell;
          const int lx = (int)(cell & 0xffffu) - ox0, ly = (int)((cell >> 16) & 0x7fffu) - oy0;
          return cell != kDead && lx + ox >= 0 && lx < kOwnW && ly + oy >= 0 && ly < kOwnH;
        },
        [&](uint32_t v) {
          const FwdRec rec = sb[v];
          const int lx = (int)(rec.cell & 0xffffu) - ox0, ly = (int)((rec.cell >> 16) & 0x7fffu) - oy0;
          double wx, ax, wy, ay;
          expand_frac(rec.fx, wx, ax);
          expand_frac(rec.fy, wy, ay);
          const double tb = fabs(dm((double)rec.dt, 1e-6) - esr) * iwin;  // engine.hpp:370
          // polarity_index plane set; corner weights pre-scaled by 2^fb (exact)
          const uint32_t pa = acc_s + (rec.cell >> 31) * (4 * kPlane * 4);
          const double sx0 = ax * fsc, sx1 = wx * fsc;
          const bool inx0 = lx >= 0, inx1 = lx + ox < kOwnW, iny0 = ly >= 0, iny1 = ly + oy < kOwnH;
          const int o00 = ly * kRowW + lx;
          // branch-free corners: a corner outside the tile adds a zero term to a
          // padding word of row 0 (x = 32 + lane % 8, never read), so the four
          // corners issue without divergent branches
          const int pad = kOwnW + (lane & 7);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const bool in = ((q & 1) ? inx1 : inx0) && ((q & 2) ? iny1 : iny0);
            const double wqq = ((q & 1) ? sx1 : sx0) * ((q & 2) ? wy : ay);
            const int o = in ? o00 + ((q & 2) ? oy * kRowW : 0) + ((q & 1) ? ox : 0) : pad;
            const double wv = in ? wqq : 0.0;
            const uint32_t a = pa + 4u * (uint32_t)o;
            const unsigned long long qc = fx_q(wv);  // wv <= 2^50
            if (wv > 0.0 && qc == 0ull) flag[o] = 1u;  // w > 0 below the fixed-point resolution
            fx_add(a, a + 4 * kPlane, qc);
            fx_add(a + 8 * kPlane, a + 12 * kPlane, fx_q(wv * tb));
          }
        });
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[b]);
    ++it;
    if (!d.last) continue;

    // reference r complete: refresh_active (warp.hpp:186-192), reference_loss
    // terms (:306-309), splat_position_grad factors (:346-349)
    consumer_sync(kFwdCons);
    double lsum = 0.0;
    unsigned actv = 0;
    for (int pxi = ct; pxi < kOwnPx; pxi += kFwdCons) {
      const int lx = pxi % kOwnW, ly = pxi / kOwnW;
      const int px = ox0 + lx, py = oy0 + ly;
      const int o = ly * kRowW + lx;
      if (px < W && py < H) {
        const double ifs = ifsc;  // 2^-fb
        const double C0 = (double)fx_read(acc + o, acc + kPlane + o) * ifs;
        const double S0 = (double)fx_read(acc + 2 * kPlane + o, acc + 3 * kPlane + o) * ifs;
        const double C1 = (double)fx_read(acc + 4 * kPlane + o, acc + 5 * kPlane + o) * ifs;
        const double S1 = (double)fx_read(acc + 6 * kPlane + o, acc + 7 * kPlane + o) * ifs;
        const int g = py * W + px;
        actv += (flag[o] || C0 > 0.0 || C1 > 0.0) ? 1u : 0u;  // refresh_active: some w > 0
        // correctly rounded reciprocals (== 1.0 / x, without the general divide)
        const double i0 = rcp_fast(C0 + kLossEps), i1 = rcp_fast(C1 + kLossEps);
        const double c0 = S0 * i0, c1 = S1 * i1;
        lsum += c0 * c0 + c1 * c1;
        // polarity-interleaved [w][r][px][pol]: the two polarities of a pixel
        // share a 32 B sector, so k_bwd_event's lanes of both polarities
        // gather from the same cache lines
        double2* cwp = coef + (((size_t)w * R + r) * HW + g) * 2;
        // one 32 B store per pixel (a warp's row of pixels stays one contiguous run)
        asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(cwp), "d"(c0), "d"(c0 * i0),
                     "d"(c1), "d"(c1 * i1)
                     : "memory");
        if (stack_out) {
          double2* so = stack_out + ((size_t)w * R + r) * 2 * HW;
          so[g] = make_double2(C0, S0);
          so[HW + g] = make_double2(C1, S1);
        }
      }
#pragma unroll
      for (int k = 0; k < 9; ++k) acc[k * kPlane + o] = 0u;  // this pixel's words, next reference
    }
    lsum = warp_sum(lsum);
    actv = __reduce_add_sync(kFull, actv);
    if (lane == 0) {
      s_red[r & 1][cw] = lsum;
      s_act[r & 1][cw] = actv;
    }
    consumer_sync(kFwdCons);
    if (ct == 0) {
      double sum = 0.0;
      unsigned a = 0;
      for (int m = 0; m < kFwdWarps; ++m) {
        sum += s_red[r & 1][m];
        a += s_act[r & 1][m];
      }
      const size_t slot = ((size_t)w * R + r) * TP.oT + T;
      part_acc[slot] = sum;
      part_act[slot] = a;
    }
    ++r;
  }
}

// ---------------------------------------------------------------------------
// backward: one CTA per (owner tile, window), warp specialised like the
// forward. For a reference r in 1..B-1 every alive event's record is the sink
// (BufferGradSink::add, warp.hpp:394-406) of exactly one bin: r - 1 when
// r <= j (backward leg: bin i sinks at pos[i+1]) and r otherwise (forward leg:
// bin i sinks at pos[i]); references 0 and B are never sinks
// (engine.hpp:475-504). Each bin also receives its events' source-pixel sink
// (the two partial steps, weight 1 at (x, y)). So the CTA streams the
// forward's per-reference candidate lists, references 1..B-1 in order, into
// two rolling fixed-point gradient tiles (bins r - 1 and r); after reference r
// (and the source sinks of bin r - 1) bin r - 1 is complete and feeds the fused
// depth_pose_to_flows_backward (geometry.hpp:300-322); d_depth sums the bins
// in order in registers.
//
// Staging layout: every record range gets an even-aligned slot region of
// roundup2(len + 2) slots; its 8 B sink values are bulk-copied as the 16 B-aligned
// superset starting at the region, and its records at the same slot offset, so
// slot s holds the record and value of one candidate; the slack slots of every
// region are flagged in a bitmask. Source ranges are 16 B {packed event, gx, gy}
// records in (bin, tile, time) order (k_bwd_event, k_src_base): one bulk copy
// each, no slack.
//
// Bin groups (gridDim.z > 1, owner_groups): CTA z owns bins [i0, i1) and
// streams groups i0..i1, where group i0 (i0 > 0) only primes bin i0 with the
// record sinks of reference i0 that belong to it. Every bin tile is then built
// from exactly the same terms as without groups (bit-identical, fixed point),
// and each bin's d_depth term is stored (dbin) for k_depth_bins to sum in bin
// order -- the same sum the single-group CTA forms in registers.

constexpr int kStageQ = 1536;  // slots per buffer
constexpr int kBufQ = 2;       // staging buffers (pipeline depth)
constexpr int kBwdThreads = kCons + 64;  // two producer warps
// each extra bin group re-streams one reference's records (its prime group)
constexpr int kMaxBwdGroups = 3;

struct BRound {
  uint32_t n;      // slots
  uint32_t split;  // slots [0, split): record sinks of reference r; [split, n): source sinks of bin r - 1
  int r;           // group
  int last;        // last round of the group: bin r - 1 is complete
};

template <bool kGrouped>
__global__ void __launch_bounds__(kBwdThreads, 2) k_bwd_cells(
    const uint2* __restrict__ sorted, const uint64_t* __restrict__ ev_off, WinParams P,
    TileParams TP, const uint32_t* __restrict__ tile_ptr, const uint32_t* __restrict__ bin_ptr,
    const FwdRec* __restrict__ recs, const float2* __restrict__ vals, uint64_t n_total,
    const uint32_t* __restrict__ gmax, const uint4* __restrict__ bbox,
    const uint32_t* __restrict__ lcount, const uint16_t* __restrict__ lists,
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ srcbase,
    const uint4* __restrict__ srcrec, const int* __restrict__ no_surv,
    const double* __restrict__ depth, const uint8_t* __restrict__ mask,
    const double* __restrict__ pose_tab, double fx, double fy, double cx, double cy, double ifx,
    double ify, double* __restrict__ d_depth, double* __restrict__ dbin,
    double* __restrict__ pose_part, double* __restrict__ grad_out) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint4* stage16 = reinterpret_cast<uint4*>(smem);                          // [kBufQ][kStageQ] records
  float2* stage8 = reinterpret_cast<float2*>(stage16 + kBufQ * kStageQ);    // [kBufQ][kStageQ] values
  uint32_t* acc = reinterpret_cast<uint32_t*>(stage8 + kBufQ * kStageQ);   // [tile][gu, gv][lo, hi][kPlane]
  __shared__ Batch bt;
  // round metadata (descriptor, slack bitmask) in 2 kBufQ sets: the set of
  // round it was last used by round it - 4, released before round it - 2 was
  // staged, so the producer fills it before waiting for the buffer of round it
  __shared__ BRound desc[2 * kBufQ];
  __shared__ uint32_t roffs[2][2 * kListCapO + 1 > kBatchCap ? 2 * kListCapO + 1 : kBatchCap];
  __shared__ uint32_t s_it;  // round counter hand-off after an overflowed group
  __shared__ uint32_t fake[2 * kBufQ][kStageQ / 32];  // slack slots of the staged round
  __shared__ __align__(16) uint2 rv[2][2][kRgCap];   // prefetched ranges (reference, source)
  __shared__ __align__(16) uint2 fb[kBatchCap + 1];  // overflow-path ranges
  __shared__ __align__(8) uint64_t full[kBufQ], empty[kBufQ], rbar[2];
  __shared__ uint16_t wq[kWarps][64];  // per-warp compaction queues
  __shared__ int s_kbits;              // fixed-point magnitude bits of the gradient terms
  __shared__ double s_pose[2][kWarps][kPoseSums];

  const int T = blockIdx.x, w = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int B = P.B, R = B + 1, NS = 2 * B + 1, W = P.W, H = P.H, HW = P.HW;
  const int ox0 = (T % TP.otx) * kOwnW, oy0 = (T / TP.otx) * kOwnH;
  const int ox = W >= 2 ? 1 : 0, oy = H >= 2 ? 1 : 0;
  const uint64_t base = ev_off[w];
  const uint32_t* tp = tile_ptr + (size_t)w * (TP.nT + 1);
  const uint32_t* bp = bin_ptr + (size_t)w * TP.nT * (B + 1);
  const bool run = !no_surv[w];
  // this CTA's bins [i0, i1); group gs = max(i0, 1) primes bin i0 when i0 > 0
  // (functions of blockIdx, re-formed where used rather than kept live)
  auto bin_lo = [&]() { return kGrouped ? (int)blockIdx.z * P.B / (int)gridDim.z : 0; };
  auto bin_hi = [&]() { return kGrouped ? ((int)blockIdx.z + 1) * P.B / (int)gridDim.z : P.B; };
  auto first_group = [&]() { return bin_lo() > 0 ? bin_lo() : 1; };
  auto prime_group = [&]() { return kGrouped && bin_lo() > 0 ? bin_lo() : -1; };

  for (int i = tid; i < 8 * kPlane; i += kBwdThreads) acc[i] = 0u;
  if (tid == 0) {
    for (int q = 0; q < kBufQ; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], kWarps);
    }
    mbar_init(&rbar[0], 1);
    mbar_init(&rbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (wid < 2) {
    // ---------------- producers ----------------
    // two producer warps: warp pw stages the rounds of parity pw (the
    // round sequence is a pure function of the prefetched ranges, so both walk
    // it in lockstep); an overflowed list is staged by warp 0 alone.
    const int pw = wid;
    auto pair_sync = [] { asm volatile("bar.sync 2, 64;" ::: "memory"); };
    // group g = 1..B: the record sinks of reference g (g < B, list slot g) then
    // the source-pixel sinks of bin g - 1 (list slot R + g - 1); after group g
    // bin g - 1 is complete. Ranges are prefetched one group ahead.
    auto prefetch = [&](int g) {  // warp 0 only
      const size_t gref = ((size_t)w * NS + g) * TP.oT + T;
      const size_t gsrc = ((size_t)w * NS + R + g - 1) * TP.oT + T;
      const int q = (g - first_group()) & 1;
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        const uint32_t one = kRgCap * (uint32_t)sizeof(uint2);
        mbar_arrive_expect_tx(&rbar[q], g < B ? 2 * one : one);
        if (g < B) bulk_g2s(rv[q][0], ranges + gref * kRgCap, one, &rbar[q]);
        bulk_g2s(rv[q][1], ranges + gsrc * kRgCap, one, &rbar[q]);
      }
    };
    uint32_t it = 0;
    auto rounds = [&](const Cat& cv, int g, bool final, bool all) {
      const FwdRec* rr = recs + (size_t)min(g, B) * n_total + base;
      const float2* v0 = vals + (size_t)(g - 1) * n_total;  // sinks at reference g
      const uint4* v1 = srcrec + base;  // source-pixel sinks with their events ((bin, tile) order)
      const int nl = cv.nl(), n0 = cv.n0;
      const uint32_t total = cv.total();
      // virtual candidates per round, leaving room for <= 3 slack slots per range
      const uint32_t capv = kStageQ - 3u * (uint32_t)nl;
      for (uint32_t rb = 0; rb < total || (rb == 0 && final); rb += capv) {
        const int b = (int)(it % kBufQ);
        if (!all && (int)(it & 1) != pw) {  // the other producer's round
          ++it;
          if (total == 0) break;
          continue;
        }
        // everything that does not touch buffer b is prepared before waiting
        // for it: the region offsets (this producer's own array) and the byte count
        uint32_t* const roff = roffs[pw];
        uint4* s16 = stage16 + b * kStageQ;
        float2* s8 = stage8 + b * kStageQ;
        const int ms = (int)(it % (2 * kBufQ));  // metadata set of this round
        uint32_t* fk = fake[ms];
        // the ranges that intersect this round: [la, lb) (prefixes are monotone)
        int la = 0, lb = nl;
        {
          int a = 0, z = nl;  // first l with pre(l + 1) > rb
          while (a < z) {
            const int m = (a + z) >> 1;
            if (cv.pre(m + 1) > rb) z = m; else a = m + 1;
          }
          la = a;
          z = nl;  // first l >= la with pre(l) >= rb + capv
          while (a < z) {
            const int m = (a + z) >> 1;
            if (cv.pre(m) >= rb + capv) z = m; else a = m + 1;
          }
          lb = a;
        }
        // region offsets: exclusive scan of roundup2(len + 2) over the record
        // ranges (their 8 B values are copied as 16 B-aligned supersets) and of
        // len over the source ranges (16 B records, no slack)
        uint32_t carry = 0;
        for (int l0 = la; l0 < lb; l0 += 32) {
          const int l = l0 + lane;
          uint32_t sz = 0;
          if (l < lb) {
            const uint32_t lo = max(cv.pre(l), rb), hi = min(cv.pre(l + 1), rb + capv);
            sz = lo < hi ? (l < n0 ? ((hi - lo + 3) & ~1u) : hi - lo) : 0u;
          }
          uint32_t x = sz;
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, x, o);
            if (lane >= o) x += y;
          }
          if (l < lb) roff[l] = carry + x - sz;
          carry += __shfl_sync(kFull, x, 31);
        }
        __syncwarp();
        const uint32_t nslots = carry;
        uint32_t bytes = 0;
        for (int l = la + lane; l < lb; l += 32) {
          const uint32_t lo = max(cv.pre(l), rb), hi = min(cv.pre(l + 1), rb + capv);
          if (lo >= hi) continue;
          const uint64_t k0 = cv.rng(l) + (lo - cv.pre(l)), len = hi - lo;
          const uint64_t a0 = (base + k0) & ~1ull, a1 = (base + k0 + len + 1) & ~1ull;
          bytes += (uint32_t)(len * 16) + (l < n0 ? (uint32_t)((a1 - a0) * 8) : 0u);
        }
        bytes = warp_sum_u32(bytes);
        for (int q = lane; q < kStageQ / 32; q += 32) fk[q] = 0u;
        __syncwarp();
        for (int l = la + lane; l < min(lb, n0); l += 32) {
          const uint32_t lo = max(cv.pre(l), rb), hi = min(cv.pre(l + 1), rb + capv);
          if (lo >= hi) continue;
          const uint64_t k0 = cv.rng(l) + (lo - cv.pre(l)), len = hi - lo;
          const uint32_t par = (uint32_t)((base + k0) & 1ull);  // n_total is even
          const uint32_t s0 = roff[l], sz = (uint32_t)((len + 3) & ~1ull);
          // slack slots (no candidate of this range): s0 if par, [s0+par+len, s0+sz)
          if (par) atomicOr(fk + (s0 >> 5), 1u << (s0 & 31));
          for (uint32_t q = s0 + par + (uint32_t)len; q < s0 + sz; ++q)
            atomicOr(fk + (q >> 5), 1u << (q & 31));
        }
        if (lane == 0) {
          desc[ms].n = nslots;
          desc[ms].split = n0 < la ? 0u : (n0 < lb ? roff[n0] : nslots);
          desc[ms].r = g;
          desc[ms].last = (final && rb + capv >= total) ? 1 : 0;
        }
        __syncwarp();
        // only now wait for the buffer itself (consumers done with round it - 2)
        if (it >= kBufQ) mbar_wait(&empty[b], ((it / kBufQ) - 1) & 1);
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive_expect_tx(&full[b], bytes);
        __syncwarp();
        for (int l = la + lane; l < lb; l += 32) {
          const uint32_t lo = max(cv.pre(l), rb), hi = min(cv.pre(l + 1), rb + capv);
          if (lo >= hi) continue;
          const uint64_t k0 = cv.rng(l) + (lo - cv.pre(l)), len = hi - lo;
          const uint32_t par = (uint32_t)((base + k0) & 1ull);
          const uint32_t s0 = roff[l];
          const uint64_t a0 = (base + k0) & ~1ull, a1 = (base + k0 + len + 1) & ~1ull;
          if (l < n0) {
            bulk_g2s(s8 + s0, v0 + a0, (uint32_t)((a1 - a0) * 8), &full[b]);
            bulk_g2s(s16 + s0 + par, rr + k0, (uint32_t)(len * sizeof(FwdRec)), &full[b]);
          } else {
            bulk_g2s(s16 + s0, v1 + k0, (uint32_t)(len * 16), &full[b]);
          }
        }
        ++it;
        if (total == 0) break;
      }
    };
    // overflowed list (more than kListCapO sort tiles): scan the boxes batch by batch
    auto scan_rounds = [&](int kind, int g, bool final) {
      const int slot = kind == 0 ? g : R + g - 1;
      const size_t ws = (size_t)w * NS + slot;
      if (lane == 0) bt.seg = -1;
      __syncwarp();
      int more = 1;
      while (more) {
        next_batch<1>(bt, lcount, lists, bbox, TP.nT, ox0, oy0,
                      [&](int) { return ws * TP.oT + T; }, [&](int) { return ws * TP.nT; },
                      [&](int, int S) {
                        if (kind == 0) return make_uint2(tp[S], tp[S + 1]);
                        const uint32_t* b = bp + (size_t)S * (B + 1);
                        const uint32_t lo = srcbase[((size_t)w * B + g - 1) * TP.nT + S];
                        return make_uint2(lo, lo + b[g] - b[g - 1]);
                      });
        more = bt.more;
        batch_to_view(bt, fb);
        rounds(kind == 0 ? make_cat(fb, nullptr) : make_cat(nullptr, fb), g, final && !more, true);
      }
    };
    // fixed-point headroom: a bin tile sums terms of two groups; bound every
    // group's candidate count (overflowed lists: the window's event count)
    if (pw == 0) {
      const uint32_t nwe = (uint32_t)(ev_off[w + 1] - base);
      uint32_t tmax = 0;
      for (int l = lane; l < 2 * B - 1; l += 32) {
        const int slot = l < B - 1 ? l + 1 : R + (l - (B - 1));
        const uint2 e0 = ranges[(((size_t)w * NS + slot) * TP.oT + T) * kRgCap];
        tmax = max(tmax, e0.x == kOverflow ? nwe : e0.y);
      }
      for (int o = 16; o > 0; o >>= 1) tmax = max(tmax, __shfl_xor_sync(kFull, tmax, o));
      if (lane == 0) s_kbits = min(49, 63 - bits_for(2u * min(tmax, 0x7fffffffu)));
      __syncwarp();
    }
    if (run) {
      if (pw == 0) prefetch(first_group());
      for (int g = first_group(); g <= bin_hi(); ++g) {
        pair_sync();  // both producers are done with the ranges of group g - 1
        if (pw == 0 && g + 1 <= bin_hi()) prefetch(g + 1);
        const int q = (g - first_group()) & 1;
        mbar_wait(&rbar[q], ((g - first_group()) >> 1) & 1);
        const bool prime = g == prime_group();  // record sinks of reference g only, bin g not complete
        const uint2* va = g < B ? rv[q][0] : nullptr;
        const uint2* vb = prime ? nullptr : rv[q][1];
        const bool oa = va && va[0].x == kOverflow, ob = vb && vb[0].x == kOverflow;
        if (!oa && !ob) {
          rounds(make_cat(va, vb), g, !prime, false);
        } else {
          if (pw == 0) {
            if (va) {
              if (oa) scan_rounds(0, g, false);
              else rounds(make_cat(va, nullptr), g, false, true);
            }
            if (vb) {
              if (ob) scan_rounds(1, g, true);
              else rounds(make_cat(nullptr, vb), g, true, true);
            }
            if (lane == 0) s_it = it;
          }
          pair_sync();
          it = s_it;
        }
      }
    } else {  // no survivors: every bin is zero, still finish each one
      for (int g = bin_lo() + 1; g <= bin_hi(); ++g) rounds(make_cat(nullptr, nullptr), g, true, false);
    }
    return;
  }

  // ---------------- consumers ----------------
  const int ct = tid - 64, cw = wid - 2;
  const uint32_t acc_s = smem_u32(acc);
  // fixed-point scale of this window's gradient terms: |w g| <= max|g| < 2^e,
  // scaled to 2^kbits (s_kbits is written by the producer before its first round)
  int e2 = 0;
  frexp((double)__uint_as_float(gmax[w]), &e2);
  double gsc = 0.0;
  double dd = 0.0;  // d_depth of this pixel, bins summed in order
  uint32_t it = 0;
  const int n_bins = bin_hi() - bin_lo();
  for (int done = 0; done < n_bins;) {
    const int b = (int)(it % kBufQ);
    mbar_wait(&full[b], (it / kBufQ) & 1);
    if (it == 0) gsc = ldexp(1.0, s_kbits - e2);
    const int ms = (int)(it % (2 * kBufQ));  // metadata set of this round
    const BRound d = desc[ms];
    const uint4* s16 = stage16 + b * kStageQ;
    const float2* s8 = stage8 + b * kStageQ;
    const uint32_t* fk = fake[ms];
    const uint32_t er = P.erel[d.r < B ? d.r : B];  // the sink test's threshold for this round
    // (prime group: re-formed from blockIdx.z here rather than kept live)
    const int lo_bin = kGrouped && d.r == (int)blockIdx.z * B / (int)gridDim.z ? d.r : 0;
    // record sinks of reference d.r (slots < split)
    compacted<kCons>(
        (uint32_t)cw * 32, d.split, wq[cw],
        [&](uint32_t v) {
          if ((fk[v >> 5] >> (v & 31)) & 1u) return false;
          const uint32_t cell = s16[v].x;
          const int lx = (int)(cell & 0xffffu) - ox0, ly = (int)((cell >> 16) & 0x7fffu) - oy0;
          // (zero sink values are not filtered here: they add zero terms, and the
          // test would cost a second shared load per candidate slot)
          return !(cell == kDead || lx + ox < 0 || lx >= kOwnW || ly + oy < 0 || ly >= kOwnH);
        },
        [&](uint32_t v) {
          const uint4 rec = s16[v];
          const int lx = (int)(rec.x & 0xffffu) - ox0, ly = (int)((rec.x >> 16) & 0x7fffu) - oy0;
          const float2 g = s8[v];
          // the bin this sink belongs to: r - 1 if r <= j else r, and for
          // 1 <= r <= B-1, r <= bin_of(t) (warp.hpp:284-288) iff erel[r] <= dt
          const int bin = (rec.y >= er) ? d.r - 1 : d.r;
          if (kGrouped && bin < lo_bin) return;  // a sink of bin i0 - 1 (another CTA's)
          const uint32_t pt = acc_s + (uint32_t)(bin & 1) * (4 * kPlane * 4);
          double wx, ax, wy, ay;
          expand_frac(__uint_as_float(rec.z), wx, ax);
          expand_frac(__uint_as_float(rec.w), wy, ay);
          const double gx = (double)g.x * gsc, gy = (double)g.y * gsc;
          const bool inx0 = lx >= 0, inx1 = lx + ox < kOwnW, iny0 = ly >= 0, iny1 = ly + oy < kOwnH;
          const int o00 = ly * kRowW + lx;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const bool in = ((q & 1) ? inx1 : inx0) && ((q & 2) ? iny1 : iny0);
            const double wqq = ((q & 1) ? wx : ax) * ((q & 2) ? wy : ay);
            if (in && wqq != 0.0) {
              const int o = o00 + ((q & 2) ? oy * kRowW : 0) + ((q & 1) ? ox : 0);
              const uint32_t a = pt + 4u * (uint32_t)o;
              fx_add(a, a + 4 * kPlane, fx_qs(wqq * gx));
              fx_add(a + 8 * kPlane, a + 12 * kPlane, fx_qs(wqq * gy));
            }
          }
        });
    // source-pixel sinks of bin d.r - 1 (slots >= split): weight 1 at the event's
    // pixel; each slot a 16 B {packed event, gx, gy} record, no slack slots
    {
      const uint32_t pt = acc_s + (uint32_t)((d.r - 1) & 1) * (4 * kPlane * 4);
      for (uint32_t v = d.split + ct; v < d.n; v += kCons) {
        const uint4 sr = s16[v];
        const uint2 e = make_uint2(sr.x, sr.y);
        const int lx = ev_x(e) - ox0, ly = ev_y(e) - oy0;
        if (lx < 0 || lx >= kOwnW || ly < 0 || ly >= kOwnH) continue;
        const float2 g = make_float2(__uint_as_float(sr.z), __uint_as_float(sr.w));
        if (g.x == 0.f && g.y == 0.f) continue;
        const uint32_t a = pt + 4u * (uint32_t)(ly * kRowW + lx);
        fx_add(a, a + 4 * kPlane, fx_qs((double)g.x * gsc));
        fx_add(a + 8 * kPlane, a + 12 * kPlane, fx_qs((double)g.y * gsc));
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[b]);
    ++it;
    if (!d.last) continue;

    // bin i = d.r - 1 complete: fused depth_pose_to_flows_backward (geometry.hpp:300-322)
    const int i = d.r - 1;
    // per-pixel constants, re-formed per bin (not held across the streaming loop:
    // the register budget of two 576-thread CTAs per SM is 56); the depth load is
    // issued before the barrier so its latency overlaps the wait
    const int lxp = ct % kOwnW, lyp = ct / kOwnW;
    const int px = ox0 + lxp, py = oy0 + lyp;
    const bool own_px = px < W && py < H;
    const int gq = py * W + px, op = lyp * kRowW + lxp;
    const double dpx = own_px && depth ? __ldg(depth + (size_t)w * HW + gq) : 0.0;
    consumer_sync(kCons);
    const double igsc = ldexp(1.0, e2 - s_kbits);
    // pose sums of this pixel (see kPoseSums): N = d v r^T (0..8), v (9..11),
    // generated from (d, v, r^) in two passes (fewer live registers than all 12)
    double mv0 = 0.0, mv1 = 0.0, mv2 = 0.0, mdp = 0.0, mrx = 0.0, mry = 0.0;
    double ddi = 0.0;  // this bin's d_depth term
    {
      const uint32_t* at = acc + (i & 1) * 4 * kPlane;
      const double gu = (double)(long long)fx_read(at + op, at + kPlane + op) * igsc;
      const double gv = (double)(long long)fx_read(at + 2 * kPlane + op, at + 3 * kPlane + op) * igsc;
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[((i & 1) * 4 + k) * kPlane + op] = 0u;  // tile of bin i + 2
      if (own_px) {
        if (grad_out) {
          grad_out[((size_t)w * B + i) * 2 * HW + gq] = gu;
          grad_out[(((size_t)w * B + i) * 2 + 1) * HW + gq] = gv;
        }
        const bool dok = depth && pose_tab && (!mask || mask[(size_t)w * HW + gq]) && dpx > 0.0;
        if (dok && (gu != 0.0 || gv != 0.0)) {
          // backproject(x, 1.0, k) (geometry.hpp:147-149)
          // (times the reciprocal focal lengths: within 1 ulp of the division)
          const double rx = ((double)px - cx) * ifx, ry = ((double)py - cy) * ify;
          const double* ptab = pose_tab + ((size_t)w * B + i) * kPoseTab;
          const double rr0 = ptab[0] * rx + ptab[1] * ry + ptab[2];
          const double rr1 = ptab[3] * rx + ptab[4] * ry + ptab[5];
          const double rr2 = ptab[6] * rx + ptab[7] * ry + ptab[8];
          const double p0 = dpx * rr0 + ptab[36], p1 = dpx * rr1 + ptab[37], p2 = dpx * rr2 + ptab[38];
          if (p2 > 0.0) {
            const double inv_dt = ptab[39], iz = rcp_fast(p2);  // 1 / p2 to 1 ulp
            // reproject_with_grads (geometry.hpp:185-209) folded into the adjoint:
            // v = (gu du/dX, gv dv/dY, gu du/dZ + gv dv/dZ) / dt with du/dX = fx/Z,
            // du/dZ = -fx X/Z^2 (dv alike) -- the translation gradient; d_depth adds
            // v . (R r^) and d_omega_a = d v . (dR_a r^), r^ = (rx, ry, 1), summed as
            // the moments N = sum d v r^T, contracted with dR_a once per (window,
            // bin) (k_pose_contract)
            const double sc = iz * inv_dt;
            const double v0 = gu * fx * sc, v1 = gv * fy * sc;
            const double v2 = -(v0 * p0 + v1 * p1) * iz;
            // the add is explicitly rounded: k_depth_bins re-forms this sum from the stored terms
            ddi = v0 * rr0 + v1 * rr1 + v2 * rr2;
            dd = __dadd_rn(dd, ddi);
            mv0 = v0;
            mv1 = v1;
            mv2 = v2;
            mdp = dpx;
            mrx = rx;
            mry = ry;
          }
        }
      }
    }
    if (kGrouped && dbin && own_px) dbin[((size_t)w * B + i) * HW + gq] = ddi;
    if (pose_part) {
      // warp sums by transposition (warp_comp_sum), fixed order: deterministic
      {
        const double d0 = mdp * mv0, d1 = mdp * mv1, d2 = mdp * mv2;
        double c[8] = {d0 * mrx, d0 * mry, d0, d1 * mrx, d1 * mry, d1, d2 * mrx, d2 * mry};
        const double v = warp_comp_sum(c, lane);
        if ((lane & 3) == 0) s_pose[i & 1][cw][(lane >> 2) & 7] = v;
      }
      {
        double c[4] = {mdp * mv2, mv0, mv1, mv2};
        const double v = warp_comp_sum(c, lane);
        if ((lane & 7) == 0) s_pose[i & 1][cw][8 + ((lane >> 3) & 3)] = v;
      }
    }
    consumer_sync(kCons);  // also: the zeroed tile is ready for bin i + 2
    if (pose_part && ct < kPoseSums) {
      double sum = 0.0;
      for (int m = 0; m < kWarps; ++m) sum += s_pose[i & 1][m][ct];
      pose_part[(((size_t)w * B + i) * kPoseSums + ct) * TP.oT + T] = sum;  // [w][bin][moment][part]
    }
    ++done;
  }
  {
    const int px = ox0 + ct % kOwnW, py = oy0 + ct / kOwnW;
    if (d_depth && !(kGrouped && dbin) && px < W && py < H) d_depth[(size_t)w * HW + py * W + px] = dd;
  }
  (void)H;
}

// d_depth of grouped backward CTAs: each pixel's bin terms summed in bin order
// from 0.0, exactly the register sum of an ungrouped CTA
__global__ void k_depth_bins(const double* __restrict__ dbin, int B, int HW, int n_windows,
                             double* __restrict__ d_depth) {
  const size_t n = (size_t)n_windows * HW;
  for (size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (size_t)gridDim.x * blockDim.x) {
    const size_t w = k / HW, p = k % HW;
    double dd = 0.0;
    for (int i = 0; i < B; ++i) dd = __dadd_rn(dd, dbin[(w * B + i) * HW + p]);
    d_depth[k] = dd;
  }
}

// ---------------------------------------------------------------------------
// launchers

static size_t fwd_cells_smem() {
  return 2 * (size_t)kStageP * sizeof(FwdRec) + 9 * kPlane * sizeof(uint32_t);
}
static size_t bwd_cells_smem() {
  return (size_t)kBufQ * kStageQ * (16 + 8) + 8 * kPlane * sizeof(uint32_t);
}
static void smem_attr(const void* fn, size_t bytes) {
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

void launch_fwd_cells(cudaStream_t s, const uint64_t* ev_off, const WinParams& P,
                      const TileParams& TP, const uint32_t* tile_ptr, const FwdRec* recs,
                      uint64_t n_total, const uint4* bbox, const uint32_t* lcount,
                      const uint16_t* lists, const uint2* ranges, double2* coef, double2* stack_out,
                      double* part_acc, unsigned long long* part_act, int groups) {
  static bool attr = false;
  if (!attr) {
    smem_attr(reinterpret_cast<const void*>(k_fwd_cells<false>), fwd_cells_smem());
    smem_attr(reinterpret_cast<const void*>(k_fwd_cells<true>), fwd_cells_smem());
  }
  attr = true;
  count_launch();
  groups = std::max(1, std::min(groups, P.B + 1));
  auto* kern = groups > 1 ? k_fwd_cells<true> : k_fwd_cells<false>;
  kern<<<dim3(TP.oT, P.n_windows, groups), kFwdThreads, fwd_cells_smem(), s>>>(
      ev_off, P, TP, tile_ptr, recs, n_total, bbox, lcount, lists, ranges, coef, stack_out,
      part_acc, part_act);
}

void launch_bwd_cells(cudaStream_t s, const uint2* sorted, const uint64_t* ev_off,
                      const WinParams& P, const TileParams& TP, const uint32_t* tile_ptr,
                      const uint32_t* bin_ptr, const FwdRec* recs, const float2* bwd,
                      uint64_t n_total, const uint32_t* gmax, const uint4* bbox,
                      const uint32_t* lcount, const uint16_t* lists, const uint2* ranges,
                      const uint32_t* srcbase, const uint4* srcrec, const int* no_surv,
                      const double* depth, const uint8_t* mask, const double* pose_tab,
                      const double* K, double* d_depth, double* pose_part, double* grad_out,
                      int groups, double* dbin) {
  const double k0 = K ? K[0] : 1.0, k1 = K ? K[1] : 1.0, k2 = K ? K[2] : 0.0, k3 = K ? K[3] : 0.0;
  static bool attr = false;
  if (!attr) {
    smem_attr(reinterpret_cast<const void*>(k_bwd_cells<false>), bwd_cells_smem());
    smem_attr(reinterpret_cast<const void*>(k_bwd_cells<true>), bwd_cells_smem());
  }
  attr = true;
  count_launch();
  groups = std::max(1, std::min(groups, P.B));
  if (groups == 1 || !d_depth) dbin = nullptr;
  auto* kern = groups > 1 ? k_bwd_cells<true> : k_bwd_cells<false>;
  kern<<<dim3(TP.oT, P.n_windows, groups), kBwdThreads, bwd_cells_smem(), s>>>(
      sorted, ev_off, P, TP, tile_ptr, bin_ptr, recs, bwd, n_total, gmax, bbox, lcount, lists, ranges,
      srcbase, srcrec, no_surv, depth, mask, pose_tab, k0, k1, k2, k3, 1.0 / k0, 1.0 / k1, d_depth, dbin, pose_part,
      grad_out);
  if (dbin) {
    count_launch();
    const size_t n = (size_t)P.n_windows * P.HW;
    k_depth_bins<<<(unsigned)std::min<size_t>((n + 255) / 256, 148 * 8), 256, 0, s>>>(dbin, P.B, P.HW,
                                                                                    P.n_windows, d_depth);
  }
}

static int env_int(const char* name) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : 0;
}

int owner_groups(const TileParams& TP, const WinParams& P, bool backward) {
  static const int env_f = env_int("EVCM_FWD_GROUPS"), env_b = env_int("EVCM_BWD_GROUPS");
  const int env = backward ? env_b : env_f;
  const int max_groups = backward ? P.B : P.B + 1;
  const long ctas = (long)TP.oT * P.n_windows;
  const long target = 4L * 2 * 148;
  int g = (int)std::min<long>((target + ctas - 1) / ctas, max_groups);
  if (backward) g = std::min(g, kMaxBwdGroups);
  if (env > 0) g = env;
  return std::max(1, std::min(g, max_groups));
}

void launch_ranges(cudaStream_t s, const uint32_t* lcount, const uint16_t* lists,
                   const uint32_t* tile_ptr, const uint32_t* bin_ptr, const uint32_t* srcbase,
                   const WinParams& P, const TileParams& TP, uint2* ranges) {
  const size_t lists_n = (size_t)P.n_windows * (2 * P.B + 1) * TP.oT;
  count_launch();
  k_ranges<<<(unsigned)((lists_n * 32 + 255) / 256), 256, 0, s>>>(lcount, lists, tile_ptr, bin_ptr,
                                                                  srcbase, P, TP, ranges);
}

}  // namespace evcm_b200
