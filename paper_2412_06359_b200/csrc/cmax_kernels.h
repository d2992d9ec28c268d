// Host-side declarations of the kernel launchers (internal to libevcm_cuda).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/evcm_cuda.h"
#include "cmax_device.cuh"

namespace evcm_b200 {

constexpr int kEvBlock = 128;        // threads per block of the per-event kernels
constexpr int kPxBlock = 256;        // threads per block of the per-pixel kernels
constexpr int kPoseTab = 40;         // R[9], dR[27], t[3], inv_dt per (window, bin)
constexpr size_t kEvSmemHeader = 512;  // es + erel tables ahead of the position columns

void reset_launch_count();
void count_launch();
void launch_loss_finalize(cudaStream_t s, const double* part_acc, const unsigned long long* part_act,
                          int n_parts, const WinParams& P, double* loss, int* no_surv,
                          long long* n_active, double* scale);
// owner backward: per-part pose moments (kPoseSums per (window, bin)) summed in
// part order, then contracted with the pose table's dR into d_poses [w][B][6]
constexpr int kPoseSums = 12;
void launch_pose_contract(cudaStream_t s, const double* pose_part, int n_parts, int B, int n_windows,
                          const double* pose_tab, double* d_poses);
int launch_count();

size_t ev_smem_bytes(const WinParams& P);
int loss_parts(const WinParams& P);
int flows_bwd_parts(const WinParams& P);

void launch_stage(cudaStream_t s, const evcm_event* ev, const uint64_t* ev_off, const WinParams& P,
                  uint64_t max_n, uint2* packed, unsigned long long* err);
void launch_pose_table(cudaStream_t s, const double* poses, int n_windows, int B,
                       const double* inv_dt, double* tab, int* bad);
// Chain prologue (k_chain_init): offsets, validation words, device pose table.
constexpr int kInitMaxWin = 256;  // windows whose offsets fit the kernel parameters
constexpr uint64_t kOwnerMinEvents = 250000;  // algo auto: smaller calls take the atomic pipeline
struct ChainInit {
  uint64_t off[kInitMaxWin + 1];
  int nw, B;
  const double* poses;       // device poses [nw][B][6], or null (host-built table)
  double* tab;               // pose table out [nw][B][kPoseTab]
  uint64_t* ev_off;          // device offsets out [nw + 1]
  unsigned long long* err;   // [nw]: ~0 (no error); [nw]: pose validation flag
};
void launch_chain_init(cudaStream_t s, const ChainInit& a, const WinParams& P);
void launch_window_sums(cudaStream_t s, const double* loss, const double* d_depth,
                        const double* d_poses, int nw, int HW, int B6, double* out);
void launch_interleave_flows(cudaStream_t s, const double* uv, int B, int HW, double2* out,
                             float2* out32 = nullptr);
void launch_motion_field(cudaStream_t s, const double* depth, const uint8_t* mask,
                         const double* pose_tab, const WinParams& P, const double* K,
                         double2* flows, uint8_t* valid, float2* flows32 = nullptr);
template <typename S2>
void launch_fwd_splat(cudaStream_t s, const uint2* packed, const uint64_t* ev_off,
                      const WinParams& P, uint64_t max_n, const double2* flows, S2* stack);
template <typename S2>
void launch_loss(cudaStream_t s, const S2* stack, const WinParams& P, S2* coef,
                 double* part_acc, unsigned long long* part_act, double* loss, int* no_surv,
                 long long* n_active, double* scale);
template <typename C2, typename G2>
void launch_bwd(cudaStream_t s, const uint2* packed, const uint64_t* ev_off, const WinParams& P,
                uint64_t max_n, const double2* flows, const C2* coef, const double* scale,
                const int* no_surv, G2* grad);
template <typename G2>
void launch_flows_bwd(cudaStream_t s, const double* depth, const uint8_t* mask,
                      const double* pose_tab, const WinParams& P, const double* K, const G2* grad,
                      double* d_depth, double* pose_part, double* d_poses);
template <typename S2>
void launch_unpack_stack(cudaStream_t s, const S2* stack, size_t planes, int HW, double* count,
                         double* tsum);
template <typename G2>
void launch_unpack_grad(cudaStream_t s, const G2* g, int B, int HW, double* out);
void launch_traj_products(cudaStream_t s, const uint2* packed, uint64_t n, const WinParams& P,
                          const double2* flows, uint8_t* alive, int32_t* bin, double* pos);

// Predictor decode chain (predictor.cu)
void launch_decode(cudaStream_t s, const double* params, int sw, int sh, int factor, double* depth);
void launch_decode_adjoint(cudaStream_t s, const double* params, const double* d_depth, int sw,
                           int sh, int factor, double* d_params);
void launch_adam(cudaStream_t s, double* slots, const double* grads, double* m, double* v, size_t n,
                 double lr, double b1, double b2, double eps, double c1, double c2);

// Event ingestion (ingest.cu)
void launch_validate_events(cudaStream_t s, const evcm_event* ev, uint64_t n, int W, int H,
                            int check_window, uint64_t t_lo, uint64_t t_hi,
                            unsigned long long* first);
void launch_window_offsets(cudaStream_t s, const evcm_event* ev, uint64_t n, uint64_t t0,
                           uint64_t window_us, int n_windows, uint64_t* offsets);

// Geometry-consistency loss (geo.cu)
struct GeoArgs {
  int W, H, n_poses, want_grad;
  const double* d0;
  const uint8_t* m0;  // may be null (all valid)
  const double* d1;
  const uint8_t* m1;
  const double* tab;  // pose table [n_poses][kPoseTab]
  double K[4];
  double upstream;
  // workspace
  unsigned long long* zkey;  // [n_poses][HW]
  unsigned* winner;          // [n_poses][HW]
  double* dd0_raw;           // [n_poses][HW]   (want_grad)
  double* gb_src;            // [n_poses][HW]   (want_grad)
  double2* land;             // [n_poses][HW]   (want_grad)
  double* parts;             // [n_poses][geo_parts][8]
  double* scale;             // [n_poses]
  // outputs (device; null = not wanted)
  double* value;             // [n_poses]
  long long* n_valid;        // [n_poses]
  double* projected;         // [n_poses][HW]
  double* interpolated;      // [n_poses][HW]
  uint8_t* valid;            // [n_poses][HW]
  double* d_d0;              // [n_poses][HW]
  double* d_d1;              // [n_poses][HW]
  double* d_poses;           // [n_poses][6]
  const double* add_poses;   // d_poses = add_poses + scale * g (may alias d_poses)
  double* d_depth_sum;       // [HW] sum_i (d_d0_i + d_d1_i)
  const double* add_depth;   // d_depth_sum = add_depth + extra (may alias)
  const double* l_cm;        // predictor: losses = {l_cm, l_geo, l_cm + lambda * l_geo}
  double lambda;
  double* losses;
};
int geo_parts(int W, int H);
void launch_geo(cudaStream_t s, const GeoArgs& g);
void launch_geo_losses_off(cudaStream_t s, const double* l_cm, double lambda, double* losses);

}  // namespace evcm_b200
