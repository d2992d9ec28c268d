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
// Precision: the IWE weights w and w*tb lie in [0, 1] and use k = 50 (2^-51
// absolute rounding per term; per-pixel sums below 2^14 per window, reference
// and polarity). The reference's sensitive quantity is the splat_position_grad
// factor a*inv*(tb - a), largest where C ~ eps = 1e-9; there a term's relative
// error is ~2^-51 / 1e-9 ~ 4e-7. Gradient terms w*g use k = 49 - e with
// 2^e > max|g| of the window (k_bwd_event). n_active is exact: a pixel is
// active iff some contribution has w > 0, recorded as a flag.
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
constexpr int kStageF = 3072;                      // staged candidates per forward round
constexpr int kStageB = 2048;                      // staged candidates per backward round
constexpr int kBatchCap = 3 * kListCapO;           // sort-tile ranges per batch
constexpr int kRowW = kOwnW + 1;                   // padded accumulator row (bank spread)
constexpr int kPlane = kOwnH * kRowW;              // words per accumulator plane
constexpr int kFxFwd = 50;                         // fractional bits of the IWE sums

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
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// wait for phase `parity`; back off between polls so that waiting warps leave
// the issue slots to the CTAs that still compute
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) __nanosleep(64);
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
// forward: one CTA per (owner tile, window), references in order, warp
// specialised. Warp 0 (producer) builds each round's candidate ranges and
// stages them with cp.async.bulk into one of two buffers (full/empty mbarrier
// pair per buffer), running up to two rounds ahead; warps 1..16 (consumers, one
// pixel each in the pixel phase) accumulate a round, release its buffer and,
// after the last round of a reference, turn the tile into loss partials and
// coefficient planes.

constexpr int kCons = kThreads;                 // consumer threads (16 warps)
constexpr int kFwdThreads = kCons + 32;         // + producer warp
constexpr int kStageP = 2048;                   // candidates per buffer

struct RoundDesc {
  uint32_t n;  // staged candidates
  int r;       // reference
  int last;    // last round of this reference
};

__global__ void __launch_bounds__(kFwdThreads, 2) k_fwd_cells(
    const uint64_t* __restrict__ ev_off, WinParams P, TileParams TP,
    const uint32_t* __restrict__ tile_ptr, const FwdRec* __restrict__ recs, uint64_t n_total,
    const uint4* __restrict__ bbox, const uint32_t* __restrict__ lcount,
    const uint16_t* __restrict__ lists, double2* __restrict__ coef, double2* __restrict__ stack_out,
    double* __restrict__ part_acc, unsigned long long* __restrict__ part_act) {
  extern __shared__ __align__(16) unsigned char smem[];
  FwdRec* stage = reinterpret_cast<FwdRec*>(smem);                    // [2][kStageP]
  uint32_t* acc = reinterpret_cast<uint32_t*>(stage + 2 * kStageP);   // [pol][C, S][lo, hi][kPlane]
  uint32_t* flag = acc + 8 * kPlane;                                  // [kPlane] some w > 0
  __shared__ Batch bt;
  __shared__ RoundDesc desc[2];
  __shared__ __align__(8) uint64_t full[2], empty[2];
  __shared__ double s_red[2][kWarps];
  __shared__ unsigned s_act[2][kWarps];

  const int T = blockIdx.x, w = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int R = P.B + 1, NS = 2 * P.B + 1, W = P.W, H = P.H, HW = P.HW;
  const int ox0 = (T % TP.otx) * kOwnW, oy0 = (T / TP.otx) * kOwnH;
  const int ox = W >= 2 ? 1 : 0, oy = H >= 2 ? 1 : 0;
  const uint64_t base = ev_off[w];
  const uint32_t* tp = tile_ptr + (size_t)w * (TP.nT + 1);

  for (int i = tid; i < 9 * kPlane; i += kFwdThreads) acc[i] = 0u;
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    mbar_init(&empty[0], kWarps);
    mbar_init(&empty[1], kWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (wid == 0) {
    // ---------------- producer ----------------
    uint32_t it = 0;
    for (int r = 0; r < R; ++r) {
      const FwdRec* rr = recs + (size_t)r * n_total + base;
      const size_t ws = (size_t)w * NS + r;
      if (lane == 0) bt.seg = -1;
      __syncwarp();
      int more = 1;
      while (more) {
        next_batch<1>(bt, lcount, lists, bbox, TP.nT, ox0, oy0,
                      [&](int) { return ws * TP.oT + T; }, [&](int) { return ws * TP.nT; },
                      [&](int, int S) { return make_uint2(tp[S], tp[S + 1]); });
        const int nl = bt.nl;
        const uint32_t total = nl > 0 ? bt.pre[nl] : 0u;
        more = bt.more;
        // rounds of this batch (an empty final batch still emits one round)
        for (uint32_t rb = 0; rb < total || (rb == 0 && !more); rb += kStageP) {
          const uint32_t n = total > rb ? min(total - rb, (uint32_t)kStageP) : 0u;
          const int b = it & 1;
          if (it >= 2) mbar_wait(&empty[b], ((it >> 1) - 1) & 1);
          FwdRec* sb = stage + b * kStageP;
          if (lane == 0) {
            desc[b].n = n;
            desc[b].r = r;
            desc[b].last = (!more && rb + kStageP >= total) ? 1 : 0;
          }
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) mbar_arrive_expect_tx(&full[b], n * (uint32_t)sizeof(FwdRec));
          __syncwarp();
          for (int l = lane; l < nl; l += 32) {
            uint32_t lo, hi;
            clip(bt, l, rb, kStageP, lo, hi);
            if (lo < hi)
              bulk_g2s(sb + (lo - rb), rr + bt.rng[l] + (lo - bt.pre[l]),
                       (hi - lo) * (uint32_t)sizeof(FwdRec), &full[b]);
          }
          ++it;
          if (total == 0) break;
        }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int ct = tid - 32, cw = wid - 1;  // consumer thread / warp
  const uint32_t acc_s = smem_u32(acc);
  uint32_t it = 0;
  for (int r = 0; r < R;) {
    const int b = it & 1;
    mbar_wait(&full[b], (it >> 1) & 1);
    const RoundDesc d = desc[b];
    const FwdRec* sb = stage + b * kStageP;
    const double esr = P.es[d.r], iwin = P.inv_window;
    // splat_bilinear corners (warp.hpp:147-160) as exact fixed-point sums
    for (uint32_t v = ct; v < d.n; v += kCons) {
      const FwdRec rec = sb[v];
      const int lx = (int)(rec.cell & 0xffffu) - ox0, ly = (int)((rec.cell >> 16) & 0x7fffu) - oy0;
      if (rec.cell == kDead || lx + ox < 0 || lx >= kOwnW || ly + oy < 0 || ly >= kOwnH) continue;
      double wx, ax, wy, ay;
      expand_frac(rec.fx, wx, ax);
      expand_frac(rec.fy, wy, ay);
      const double tb = fabs(dm((double)rec.dt, 1e-6) - esr) * iwin;  // engine.hpp:370
      // polarity_index plane set; corner weights pre-scaled by 2^50 (exact)
      const uint32_t pa = acc_s + (rec.cell >> 31) * (4 * kPlane * 4);
      const double sx0 = ax * 0x1p50, sx1 = wx * 0x1p50;
      const bool inx0 = lx >= 0, inx1 = lx + ox < kOwnW, iny0 = ly >= 0, iny1 = ly + oy < kOwnH;
      const int o00 = ly * kRowW + lx;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const bool in = ((q & 1) ? inx1 : inx0) && ((q & 2) ? iny1 : iny0);
        const double wq = ((q & 1) ? sx1 : sx0) * ((q & 2) ? wy : ay);
        if (in && wq > 0.0) {
          const int o = o00 + ((q & 2) ? oy * kRowW : 0) + ((q & 1) ? ox : 0);
          flag[o] = 1u;
          const uint32_t a = pa + 4u * (uint32_t)o;
          fx_add(a, a + 4 * kPlane, __double2ull_rn(wq));
          fx_add(a + 8 * kPlane, a + 12 * kPlane, __double2ull_rn(wq * tb));
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[b]);
    ++it;
    if (!d.last) continue;

    // reference r complete: refresh_active (warp.hpp:186-192), reference_loss
    // terms (:306-309), splat_position_grad factors (:346-349)
    consumer_sync(kCons);
    double lsum = 0.0;
    unsigned actv = 0;
    {
      const int lx = ct % kOwnW, ly = ct / kOwnW;
      const int px = ox0 + lx, py = oy0 + ly;
      const int o = ly * kRowW + lx;
      if (px < W && py < H) {
        const double C0 = (double)fx_read(acc + o, acc + kPlane + o) * 0x1p-50;
        const double S0 = (double)fx_read(acc + 2 * kPlane + o, acc + 3 * kPlane + o) * 0x1p-50;
        const double C1 = (double)fx_read(acc + 4 * kPlane + o, acc + 5 * kPlane + o) * 0x1p-50;
        const double S1 = (double)fx_read(acc + 6 * kPlane + o, acc + 7 * kPlane + o) * 0x1p-50;
        const int g = py * W + px;
        actv = flag[o];
        const double i0 = 1.0 / (C0 + kLossEps), i1 = 1.0 / (C1 + kLossEps);
        const double c0 = S0 * i0, c1 = S1 * i1;
        lsum = c0 * c0 + c1 * c1;
        double2* cwp = coef + ((size_t)w * R + r) * 2 * HW;
        cwp[g] = make_double2(c0, c0 * i0);
        cwp[HW + g] = make_double2(c1, c1 * i1);
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
    actv = warp_sum_u32(actv);
    if (lane == 0) {
      s_red[r & 1][cw] = lsum;
      s_act[r & 1][cw] = actv;
    }
    consumer_sync(kCons);
    if (ct == 0) {
      double sum = 0.0;
      unsigned a = 0;
      for (int m = 0; m < kWarps; ++m) {
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
// backward: one CTA per (owner tile, bin, window). For bin i the candidates
// are: events with j > i at their reference-(i+1) cell (backward leg), events
// with j < i at their reference-i cell (forward leg), events with j == i at
// their source pixel (the two partial steps), each with its per-bin adjoint
// value (k_bwd_event) -- BufferGradSink::add (warp.hpp:394-406). The finished
// gradient tile of bin i feeds the flows backward of bin i
// (geometry.hpp:300-322): per-bin d_depth planes (summed over bins in order by
// k_ddepth_sum) and per-(tile, bin) pose partials.
//
// Staging: records (16 B, legs A/B) go to stage16 at their candidate index;
// the 8 B adjoint values (and, for the source-pixel leg, the 8 B packed events)
// are copied as 16 B-aligned supersets into per-range slots of stage8v/stage8e.

__global__ void __launch_bounds__(kThreads, 2) k_bwd_cells(
    const uint2* __restrict__ sorted, const uint64_t* __restrict__ ev_off, WinParams P,
    TileParams TP, const uint32_t* __restrict__ tile_ptr, const uint32_t* __restrict__ bin_ptr,
    const FwdRec* __restrict__ recs, const float2* __restrict__ bwd, uint64_t n_total,
    const uint32_t* __restrict__ gmax, const uint4* __restrict__ bbox,
    const uint32_t* __restrict__ lcount, const uint16_t* __restrict__ lists,
    const int* __restrict__ no_surv, const double* __restrict__ depth,
    const uint8_t* __restrict__ mask, const double* __restrict__ pose_tab, double fx, double fy,
    double cx, double cy, double* __restrict__ d_depth, double* __restrict__ pose_part,
    double* __restrict__ grad_out) {
  constexpr int k8 = kStageB + 3 * kBatchCap;  // 8 B slots incl. per-range alignment slack
  extern __shared__ __align__(16) unsigned char smem[];
  uint4* stage16 = reinterpret_cast<uint4*>(smem);                 // kStageB
  float2* stage8v = reinterpret_cast<float2*>(stage16 + kStageB);  // k8 adjoint values
  uint2* stage8e = reinterpret_cast<uint2*>(stage8v + k8);         // k8 packed events
  uint32_t* acc = reinterpret_cast<uint32_t*>(stage8e + k8);       // [gu, gv][lo, hi][kPlane]
  uint32_t* tl = acc + 4 * kPlane;                                 // touching candidates
  const uint32_t acc_s = smem_u32(acc);
  __shared__ Batch bt;
  __shared__ int s_nt;
  __shared__ uint32_t off8[kBatchCap];
  __shared__ __align__(8) uint64_t bar;
  __shared__ double s_pose[kWarps][6];

  const int T = blockIdx.x, i = blockIdx.y, w = blockIdx.z;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int B = P.B, R = B + 1, NS = 2 * B + 1, W = P.W, H = P.H, HW = P.HW;
  const int ox0 = (T % TP.otx) * kOwnW, oy0 = (T / TP.otx) * kOwnH;
  const int ox = W >= 2 ? 1 : 0, oy = H >= 2 ? 1 : 0;
  const uint64_t base = ev_off[w];
  const uint32_t* tp = tile_ptr + (size_t)w * (TP.nT + 1);
  const uint32_t* bp = bin_ptr + (size_t)w * TP.nT * (B + 1);
  const bool run = !no_surv[w];
  const int lxp = tid % kOwnW, lyp = tid / kOwnW;
  const int px = ox0 + lxp, py = oy0 + lyp;
  const bool own_px = px < W && py < H;
  const int gq = py * W + px, op = lyp * kRowW + lxp;
  const double dpx = own_px && depth ? depth[(size_t)w * HW + gq] : 0.0;
  const bool dok = own_px && depth && pose_tab && (!mask || mask[(size_t)w * HW + gq]) && dpx > 0.0;
  // fixed-point scale of this window's gradient terms: |w g| <= max|g| < 2^e
  int e2 = 0;
  frexp((double)__uint_as_float(gmax[w]), &e2);
  const double gsc = ldexp(1.0, 49 - e2), igsc = ldexp(1.0, e2 - 49);
  double dd = 0.0;  // this bin's d_depth of the pixel
  uint32_t phase = 0;

  for (int k = tid; k < 4 * kPlane; k += kThreads) acc[k] = 0u;
  if (tid == 0) {
    s_nt = 0;
    bt.seg = -1;
    mbar_init(&bar, 1);
  }
  __syncthreads();
  {
    const uint64_t vbase = (uint64_t)i * n_total + base;  // bwd[i] of this window
    const FwdRec* rA = recs + (size_t)(i + 1) * n_total + base;  // backward-leg cells (j > i)
    const FwdRec* rB = recs + (size_t)i * n_total + base;        // forward-leg cells (j < i)
    int more = run ? 1 : 0;
    while (more) {
      if (wid == 0)
        next_batch<3>(
            bt, lcount, lists, bbox, TP.nT, ox0, oy0,
            [&](int s) {
              const int slot = s == 0 ? i + 1 : (s == 1 ? i : R + i);
              return ((size_t)w * NS + slot) * TP.oT + T;
            },
            [&](int s) {
              const int slot = s == 0 ? i + 1 : (s == 1 ? i : R + i);
              return ((size_t)w * NS + slot) * TP.nT;
            },
            [&](int s, int S) {
              const uint32_t* b = bp + (size_t)S * (B + 1);
              if (s == 0) return make_uint2(b[i + 1], tp[S + 1]);
              if (s == 1) return make_uint2(tp[S], b[i]);
              return make_uint2(b[i], b[i + 1]);
            });
      __syncthreads();
      const int nl = bt.nl;
      const uint32_t total = nl > 0 ? bt.pre[nl] : 0u;
      more = bt.more;
      auto seg_of = [&](int l) {
        const uint32_t v = bt.pre[l];
        return (v >= bt.seg_end[0] ? 1 : 0) + (v >= bt.seg_end[1] ? 1 : 0);
      };
      for (uint32_t rb = 0; rb < total; rb += kStageB) {
        if (wid == 0) {
          // per-range 8 B slot offsets (exclusive scan of the even slot sizes)
          uint32_t carry = 0;
          for (int l0 = 0; l0 < nl; l0 += 32) {
            const int l = l0 + lane;
            uint32_t n8 = 0;
            if (l < nl) {
              uint32_t lo, hi;
              clip(bt, l, rb, kStageB, lo, hi);
              n8 = lo < hi ? ((hi - lo + 3) & ~1u) : 0;
            }
            uint32_t x = n8;
            for (int o = 1; o < 32; o <<= 1) {
              const uint32_t y = __shfl_up_sync(kFull, x, o);
              if (lane >= o) x += y;
            }
            if (l < nl) off8[l] = carry + x - n8;
            carry += __shfl_sync(kFull, x, 31);
          }
          __syncwarp();
          uint32_t bytes = 0;
          for (int l = lane; l < nl; l += 32) {
            uint32_t lo, hi;
            clip(bt, l, rb, kStageB, lo, hi);
            if (lo >= hi) continue;
            const int sg = seg_of(l);
            const uint64_t k0 = bt.rng[l] + (lo - bt.pre[l]), nn = hi - lo;
            if (sg < 2) bytes += (uint32_t)(nn * sizeof(FwdRec));
            const uint64_t a0 = (vbase + k0) & ~1ull, a1 = (vbase + k0 + nn + 1) & ~1ull;
            bytes += (uint32_t)((a1 - a0) * 8);
            if (sg == 2) {
              const uint64_t e0 = (base + k0) & ~1ull, e1 = (base + k0 + nn + 1) & ~1ull;
              bytes += (uint32_t)((e1 - e0) * 8);
            }
          }
          bytes = warp_sum_u32(bytes);
          fence_proxy_async();
          if (lane == 0) mbar_arrive_expect_tx(&bar, bytes);
          __syncwarp();
          for (int l = lane; l < nl; l += 32) {
            uint32_t lo, hi;
            clip(bt, l, rb, kStageB, lo, hi);
            if (lo >= hi) continue;
            const int sg = seg_of(l);
            const uint64_t k0 = bt.rng[l] + (lo - bt.pre[l]), nn = hi - lo;
            if (sg < 2)
              bulk_g2s(stage16 + (lo - rb), (sg == 0 ? rA : rB) + k0, (uint32_t)(nn * sizeof(FwdRec)),
                       &bar);
            const uint64_t a0 = (vbase + k0) & ~1ull, a1 = (vbase + k0 + nn + 1) & ~1ull;
            bulk_g2s(stage8v + off8[l], bwd + a0, (uint32_t)((a1 - a0) * 8), &bar);
            if (sg == 2) {
              const uint64_t e0 = (base + k0) & ~1ull, e1 = (base + k0 + nn + 1) & ~1ull;
              bulk_g2s(stage8e + off8[l], sorted + e0, (uint32_t)((e1 - e0) * 8), &bar);
            }
          }
        }
        __syncthreads();  // off8 visible
        mbar_wait(&bar, phase);
        phase ^= 1;
        // pass 1, one warp per range: compact the candidates whose cell touches
        // the tile as (candidate index, range)
        for (int l = wid; l < nl; l += kWarps) {
          uint32_t lo, hi;
          clip(bt, l, rb, kStageB, lo, hi);
          if (lo >= hi) continue;
          const int sg = seg_of(l);
          const uint32_t pe = (uint32_t)((base + bt.rng[l] + (lo - bt.pre[l])) & 1ull) + off8[l];
          for (uint32_t v0 = lo; v0 < hi; v0 += 32) {
            const uint32_t v = v0 + lane;
            bool hit = false;
            if (v < hi) {
              int x0, y0;
              if (sg < 2) {
                const uint32_t cell = stage16[v - rb].x;
                x0 = (int)(cell & 0xffffu);
                y0 = (int)((cell >> 16) & 0x7fffu);
                hit = cell != kDead;  // masked event (engine.hpp:564)
              } else {
                const uint2 e = stage8e[pe + (v - lo)];
                x0 = W >= 2 ? min(ev_x(e), W - 2) : 0;
                y0 = H >= 2 ? min(ev_y(e), H - 2) : 0;
                hit = true;
              }
              const int lx = x0 - ox0, ly = y0 - oy0;
              hit = hit && lx + ox >= 0 && lx < kOwnW && ly + oy >= 0 && ly < kOwnH;
            }
            const unsigned bal = __ballot_sync(kFull, hit);
            int b0 = 0;
            if (lane == 0 && bal) b0 = atomicAdd(&s_nt, __popc(bal));
            b0 = __shfl_sync(kFull, b0, 0);
            if (hit) tl[b0 + __popc(bal & ((1u << lane) - 1u))] = (v - rb) | ((uint32_t)l << 16);
          }
        }
        __syncthreads();
        // pass 2 (full warps): BufferGradSink::add corners as exact fixed-point sums
        const int nt = s_nt;
        for (int t = tid; t < nt; t += kThreads) {
          const uint32_t ent = tl[t];
          const uint32_t idx = ent & 0xffffu;
          const int l = (int)(ent >> 16);
          const int sg = seg_of(l);
          const uint32_t lo = max(bt.pre[l], rb);
          const uint64_t k0 = bt.rng[l] + (lo - bt.pre[l]);
          const uint32_t p = idx + rb - lo;
          int x0, y0;
          double wx, ax, wy, ay;
          if (sg < 2) {
            const uint4 rec = stage16[idx];
            x0 = (int)(rec.x & 0xffffu);
            y0 = (int)((rec.x >> 16) & 0x7fffu);
            expand_frac(__uint_as_float(rec.z), wx, ax);
            expand_frac(__uint_as_float(rec.w), wy, ay);
          } else {
            // bilin_cell at the integer source pixel: weight 0 or 1 (border
            // cell); masked events carry a zero adjoint value (k_bwd_event)
            const uint2 e = stage8e[(uint32_t)((base + k0) & 1ull) + off8[l] + p];
            const int ex = ev_x(e), ey = ev_y(e);
            x0 = W >= 2 ? min(ex, W - 2) : 0;
            y0 = H >= 2 ? min(ey, H - 2) : 0;
            wx = ex > x0 ? 1.0 : 0.0;
            wy = ey > y0 ? 1.0 : 0.0;
            ax = 1.0 - wx;
            ay = 1.0 - wy;
          }
          const float2 g = stage8v[(uint32_t)((vbase + k0) & 1ull) + off8[l] + p];
          const double gx = (double)g.x * gsc, gy = (double)g.y * gsc;
          const int lx = x0 - ox0, ly = y0 - oy0;
          const bool inx0 = lx >= 0, inx1 = lx + ox < kOwnW, iny0 = ly >= 0, iny1 = ly + oy < kOwnH;
          const int o00 = ly * kRowW + lx;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const bool in = ((q & 1) ? inx1 : inx0) && ((q & 2) ? iny1 : iny0);
            const double wq = ((q & 1) ? wx : ax) * ((q & 2) ? wy : ay);
            if (in && wq != 0.0) {
              const int o = o00 + ((q & 2) ? oy * kRowW : 0) + ((q & 1) ? ox : 0);
              const uint32_t a = acc_s + 4u * (uint32_t)o;
              fx_add(a, a + 4 * kPlane, (unsigned long long)__double2ll_rn(wq * gx));
              fx_add(a + 8 * kPlane, a + 12 * kPlane, (unsigned long long)__double2ll_rn(wq * gy));
            }
          }
        }
        if (tid == 0) s_nt = 0;
        __syncthreads();  // stage buffers are free for the next round
      }
    }
    // fused depth_pose_to_flows_backward for bin i (geometry.hpp:300-322)
    double c6[6] = {0, 0, 0, 0, 0, 0};
    if (own_px) {
      const double gu = (double)(long long)fx_read(acc + op, acc + kPlane + op) * igsc;
      const double gv = (double)(long long)fx_read(acc + 2 * kPlane + op, acc + 3 * kPlane + op) * igsc;
      if (grad_out) {
        grad_out[((size_t)w * B + i) * 2 * HW + gq] = gu;
        grad_out[(((size_t)w * B + i) * 2 + 1) * HW + gq] = gv;
      }
      if (dok && (gu != 0.0 || gv != 0.0)) {
        const double* pt = pose_tab + ((size_t)w * B + i) * kPoseTab;
        const double rx = 1.0 * ((double)px - cx) / fx;  // backproject(x, 1.0, k)
        const double ry = 1.0 * ((double)py - cy) / fy;
        const double rr0 = pt[0] * rx + pt[1] * ry + pt[2];
        const double rr1 = pt[3] * rx + pt[4] * ry + pt[5];
        const double rr2 = pt[6] * rx + pt[7] * ry + pt[8];
        const double p0 = dpx * rr0 + pt[36], p1 = dpx * rr1 + pt[37], p2 = dpx * rr2 + pt[38];
        if (p2 > 0.0) {
          const double inv_dt = pt[39], iz = 1.0 / p2;
          const double ju0 = fx * iz, ju2 = -fx * p0 * iz * iz;
          const double jv1 = fy * iz, jv2 = -fy * p1 * iz * iz;
          dd += (gu * (ju0 * rr0 + ju2 * rr2) + gv * (jv1 * rr1 + jv2 * rr2)) * inv_dt;
          c6[3] = gu * ju0 * inv_dt;
          c6[4] = gv * jv1 * inv_dt;
          c6[5] = (gu * ju2 + gv * jv2) * inv_dt;
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            const double* dR = pt + 9 + 9 * a;
            const double m0 = dR[0] * rx + dR[1] * ry + dR[2];
            const double m1 = dR[3] * rx + dR[4] * ry + dR[5];
            const double m2 = dR[6] * rx + dR[7] * ry + dR[8];
            c6[a] = (gu * (ju0 * dpx * m0 + ju2 * dpx * m2) + gv * (jv1 * dpx * m1 + jv2 * dpx * m2)) *
                    inv_dt;
          }
        }
      }
    }
    if (pose_part) {
#pragma unroll
      for (int a = 0; a < 6; ++a) {
        const double v = warp_sum(c6[a]);
        if (lane == 0) s_pose[wid][a] = v;
      }
      __syncthreads();
      if (tid < 6) {
        double sum = 0.0;
        for (int m = 0; m < kWarps; ++m) sum += s_pose[m][tid];
        pose_part[(((size_t)w * TP.oT + T) * B + i) * 6 + tid] = sum;
      }
    }
  }
  if (d_depth && own_px) d_depth[((size_t)w * B + i) * HW + gq] = dd;
  (void)H;
}

// ---------------------------------------------------------------------------
// launchers

static size_t fwd_cells_smem() {
  return 2 * (size_t)kStageP * sizeof(FwdRec) + 9 * kPlane * sizeof(uint32_t);
}
static size_t bwd_cells_smem() {
  const size_t k8 = kStageB + 3 * kBatchCap;
  return (size_t)kStageB * 16 + 2 * k8 * 8 + 4 * kPlane * sizeof(uint32_t) +
         kStageB * sizeof(uint32_t);
}
static void smem_attr(const void* fn, size_t bytes) {
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

void launch_fwd_cells(cudaStream_t s, const uint64_t* ev_off, const WinParams& P,
                      const TileParams& TP, const uint32_t* tile_ptr, const FwdRec* recs,
                      uint64_t n_total, const uint4* bbox, const uint32_t* lcount,
                      const uint16_t* lists, double2* coef, double2* stack_out, double* part_acc,
                      unsigned long long* part_act) {
  static bool attr = false;
  if (!attr) smem_attr(reinterpret_cast<const void*>(k_fwd_cells), fwd_cells_smem());
  attr = true;
  count_launch();
  k_fwd_cells<<<dim3(TP.oT, P.n_windows), kFwdThreads, fwd_cells_smem(), s>>>(
      ev_off, P, TP, tile_ptr, recs, n_total, bbox, lcount, lists, coef, stack_out, part_acc,
      part_act);
}

void launch_bwd_cells(cudaStream_t s, const uint2* sorted, const uint64_t* ev_off,
                      const WinParams& P, const TileParams& TP, const uint32_t* tile_ptr,
                      const uint32_t* bin_ptr, const FwdRec* recs, const float2* bwd,
                      uint64_t n_total, const uint32_t* gmax, const uint4* bbox,
                      const uint32_t* lcount, const uint16_t* lists, const int* no_surv,
                      const double* depth, const uint8_t* mask, const double* pose_tab,
                      const double* K, double* d_depth_bins, double* pose_part, double* grad_out) {
  const double k0 = K ? K[0] : 1.0, k1 = K ? K[1] : 1.0, k2 = K ? K[2] : 0.0, k3 = K ? K[3] : 0.0;
  static bool attr = false;
  if (!attr) smem_attr(reinterpret_cast<const void*>(k_bwd_cells), bwd_cells_smem());
  attr = true;
  count_launch();
  k_bwd_cells<<<dim3(TP.oT, P.B, P.n_windows), kThreads, bwd_cells_smem(), s>>>(
      sorted, ev_off, P, TP, tile_ptr, bin_ptr, recs, bwd, n_total, gmax, bbox, lcount, lists, no_surv,
      depth, mask, pose_tab, k0, k1, k2, k3, d_depth_bins, pose_part, grad_out);
}

}  // namespace evcm_b200
