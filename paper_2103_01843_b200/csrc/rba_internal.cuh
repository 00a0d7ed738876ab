// rba_internal.cuh -- context layout, arena layout and kernel launcher prototypes of librba.
// Product path only (no oracle code).  See DESIGN.md §4 for the HBM layout.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/rba.h"

namespace rba {

constexpr int KSMALL = 32;    // k <= KSMALL: one tile per landmark, warp-group kernels
constexpr int TILE_H = 4;     // R2 rows per tile for k > KSMALL
constexpr int KMAX = 512;     // largest track length supported by this build's large-k kernels

// ---- landmark-block arena layout ------------------------------------------
// Per landmark (internal order), two 16-byte aligned regions:
//  R2   = A_j = Q^_2^T J_p: logical rows 3..2k+2 (2k rows) x 9k pose columns, stored in row tiles
//         of height H (H = 2k if k <= KSMALL else TILE_H); inside a tile, camera-block-major:
//         block o is an H x 9 row-major slab.  The tile is the unit the matvec streams.
//  side = R1 (logical rows 0..2, 3 x 9k row-major: Q^_1^T J_p)  | pad4
//         TL ((2k+3) float4: [landmark columns | residual] of every logical row)
//         G  (6 x (c, s) damping rotations)                       | pad4
__host__ __device__ inline int64_t pad4(int64_t x) { return (x + 3) & ~int64_t(3); }
__host__ __device__ inline int tile_h(int k) { return k <= KSMALL ? 2 * k : TILE_H; }
__host__ __device__ inline int n_tiles(int k) { return k <= KSMALL ? 1 : (2 * k + TILE_H - 1) / TILE_H; }
__host__ __device__ inline int tile_rows(int k, int t) {
    int H = tile_h(k);
    int r = 2 * k - t * H;
    return r < H ? r : H;
}
// float offset of tile t inside the landmark's R2 region (all tiles but the last are full)
__host__ __device__ inline int64_t tile_off(int k, int t) { return (int64_t)t * pad4((int64_t)9 * k * tile_h(k)); }
__host__ __device__ inline int64_t r2_floats(int k) {
    int T = n_tiles(k);
    return tile_off(k, T - 1) + pad4((int64_t)9 * k * tile_rows(k, T - 1));
}
// float offset of element (R2 row a, camera block o, param q)
__host__ __device__ inline int64_t r2_index(int k, int a, int o, int q) {
    int H = tile_h(k);
    int t = a / H;
    int h = tile_rows(k, t);
    return tile_off(k, t) + (int64_t)o * 9 * h + (int64_t)(a - t * H) * 9 + q;
}
__host__ __device__ inline int64_t side_r1_floats(int k) { return pad4(27 * (int64_t)k); }
__host__ __device__ inline int64_t side_floats(int k) { return side_r1_floats(k) + 4 * (2 * (int64_t)k + 3) + 12; }
// side sub-offsets
__host__ __device__ inline int64_t side_tl(int k) { return side_r1_floats(k); }
__host__ __device__ inline int64_t side_g(int k) { return side_r1_floats(k) + 4 * (2 * (int64_t)k + 3); }

struct PcgState {
    double rz;  // rho^T z
    double r0;  // |rho_0|
    double rn;  // |rho_k|
    int it, done, reason, active;
};

// double scalars on the device (single buffer so one all-reduce covers them)
// [E, BAD] reduced at linearize; [ET, BADT, Q1R2, DAMPL] reduced after a trial; MODELP replicated
enum { SC_E = 0, SC_BAD, SC_ET, SC_BADT, SC_Q1R2, SC_DAMPL, SC_MODELP, SC_N = 8 };

enum { KID_LIN = 0, KID_MARG, KID_DAMP, KID_PRE, KID_MATVEC, KID_PCG, KID_BACKSUB, KID_COST, KID_N };

struct LargeItem {
    int32_t lm, t0, t1, pad;
};

struct DevProblem {
    int64_t n_p, n_l, n_obs;  // local counts (landmarks / observations of this shard)
    // state
    float *cams, *cams_trial, *pts, *pts_trial;
    // landmark metadata (internal order, sorted by k)
    int32_t *lm_k, *lm_obs0;
    int64_t *lm_r2, *lm_side;
    int32_t *obs_cam, *obs_lm;
    float2 *obs_uv;
    // scaling / damping
    float *cam_n2, *sp, *Dp2;
    float *lm_s, *lm_D;
    // arena
    float *arena;
    // reduced system / PCG
    float *pacc;  // 54 per camera: 45 upper-triangle of P_i + 9 of b~
    float *bt, *Minv;
    float *x, *r, *z, *p, *w;
    float *dl;
    double *scal;
    PcgState *pcg;
    LargeItem *large_items;
};

struct Launch {
    int kid;
    cudaEvent_t a, b;
    double bytes;
};

}  // namespace rba

struct rba_ctx {
    rba_options opt;
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int world = 1, rank = 0;
    ncclComm_t comm = nullptr;
    bool have_comm = false;
    int64_t n_p = 0, n_l_global = 0, n_obs_global = 0;
    rba::DevProblem d{};
    // host plan
    std::vector<int32_t> lm_orig;     // internal -> caller landmark index
    std::vector<int32_t> orig_to_int; // caller landmark -> internal (-1 if not owned)
    std::vector<int32_t> h_k;
    std::vector<int64_t> h_r2, h_side;
    int64_t small_lo[4] = {0, 0, 0, 0}, small_hi[4] = {0, 0, 0, 0};  // G = 4, 8, 16, 32 ranges
    int64_t large_lo = 0, large_hi = 0;
    int64_t n_large_items = 0, max_large_k = 0;
    int64_t arena_floats = 0, logical_bytes = 0;
    double marg_bytes = 0, matvec_bytes = 0;  // algorithmic bytes per launch
    std::vector<void *> allocations;
    // pinned host scratch
    double *h_scal = nullptr;
    rba::PcgState *h_pcg = nullptr;
    // solver state
    bool linearized = false, marginalized = false, solved = false, backsubbed = false;
    double lambda_blocks = 0.0;
    double cost = 0.0;
    double lm_lambda = 1e-4, lm_nu = 2.0;
    bool need_lin = true;
    int64_t iteration = 0;
    int64_t launches = 0;
    // profiling
    bool profiling = false;
    std::vector<rba::Launch> prof;
    std::vector<cudaEvent_t> ev_pool;
};

namespace rba {
// kernel launchers (rba_kernels.cu); each returns cudaGetLastError()
cudaError_t launch_check_depth(rba_ctx *c, int *d_bad);
cudaError_t launch_linearize(rba_ctx *c);
cudaError_t launch_cam_scale(rba_ctx *c);
cudaError_t launch_marginalize(rba_ctx *c, float lambda);
cudaError_t launch_redamp(rba_ctx *c, float lambda_new);
cudaError_t launch_precond_rhs(rba_ctx *c);
cudaError_t launch_precond_finalize(rba_ctx *c, float lambda);
cudaError_t launch_matvec(rba_ctx *c, const float *v, float *out);
cudaError_t launch_matvec_pcg(rba_ctx *c);
cudaError_t launch_pcg_init(rba_ctx *c, float tol, int max_iters);
cudaError_t launch_pcg_step(rba_ctx *c, float lambda, float tol, int max_iters);
cudaError_t launch_backsub(rba_ctx *c, float lambda);
cudaError_t launch_trial_cost(rba_ctx *c);
cudaError_t launch_cost(rba_ctx *c, int at_trial, int slot);
cudaError_t launch_commit(rba_ctx *c);
cudaError_t launch_add_damping(rba_ctx *c, const float *v, float *out, float lambda);
// profiling scope: CUDA events on the context stream around one launch (rba_api.cu)
struct Prof {
    rba_ctx *c;
    int kid;
    double bytes;
    cudaEvent_t a = nullptr;
    Prof(rba_ctx *c_, int kid_, double bytes_);
    void end();
};
}  // namespace rba
