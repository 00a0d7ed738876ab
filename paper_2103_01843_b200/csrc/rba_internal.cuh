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

// RBA_CHECKS build (tools/checked_build.py): device-side bounds checks on the staged / indexed
// accesses of the kernels (compute-sanitizer is closed on this pool); a failed check traps, the
// context's next call reports a CUDA error.
#ifdef RBA_CHECKS
#define RBA_CHECK(cond)              \
    do {                             \
        if (!(cond)) __trap();       \
    } while (0)
#else
#define RBA_CHECK(cond) \
    do {                \
    } while (0)
#endif

constexpr int KSMALL = 16;    // k <= KSMALL: warp-group kernels over packs of same-k landmarks
constexpr int KLARGE = 512;   // k <= KLARGE: one thread per camera block in the large-k kernels
constexpr int KMAX = 3072;    // largest track length supported (k > KLARGE: "huge" path, smem-bound)
constexpr int KMAX64 = 1024;
constexpr int S64_STAGE_DBL = 6144;  // sqrt-BA-64 small-k TMA stage: 48 KB
constexpr int SC_BS = 84;            // explicit SC: stored elements per 9 x 9 block (81 + 3 pad: 16-byte rows of float4)
constexpr int CAMPRE = 24;    // doubles of a camera's precomputed model (R, J_left, t, f, k1, k2)  // sqrt-BA-64 (f2): largest track length (registers of the FP64 product)

// ---- landmark-block arena layout ------------------------------------------
// Logical block of a landmark with k observations: rows 0..2k+2, columns [J_p (9k) | J_l | r].
// R2 = A_j = Q^_2^T J_p = logical rows 3..2k+2 (2k rows "a" = 0..2k-1) x 9k pose columns is what
// the PCG matvec streams; it is stored so that every warp load is one contiguous run:
//  * small k (<= KSMALL): landmarks are grouped in packs of np <= 32/G same-k landmarks (G = lanes
//    per landmark).  A pack is row-pair major: for row pair p (rows 2p, 2p+1), slab chunk c (9
//    float2 of the 2 x 9 slab of camera block o), landmark m, block o:
//       float2 index ((p*9 + c)*np*k + m*k + o)
//    The slab's 18 values (row r, column q) sit in the chunks as: c = 0..3 row 0 (q, q+1) pairs,
//    c = 4..7 row 1 pairs, c = 8 (row 0 q 8, row 1 q 8) -- so K2 emits each pair with one packed
//    FP32 FMA (FFMA2) per term and the product reads whole rows (slab_elem below).
//  * large k (> KSMALL): tiles of 4 rows (rows >= 2k are zero padding), tile t at 36 k t; in a
//    tile, camera blocks in groups of 32 (n_g = min(32, k - 32 g)); the 4 x 9 slab of block o is
//    9 float4 chunks:  float4 index (36*32*g)/4 + c*n_g + (o & 31)
// Side region per landmark (16-byte aligned):  R1 = logical rows 0..2 pose columns (3 x 9k
// row-major) | pad4 | TL: (2k+3) float4 [J_l row | residual] of every logical row | G: 6 x (c, s).
__host__ __device__ constexpr int64_t pad4(int64_t x) { return (x + 3) & ~int64_t(3); }
__host__ __device__ inline int large_tiles(int k) { return (k + 1) >> 1; }  // ceil(2k / 4)
__host__ __device__ inline int64_t small_pack_floats(int k, int np) { return (int64_t)18 * k * k * np; }
__host__ __device__ inline int64_t large_r2_floats(int k) { return (int64_t)36 * k * large_tiles(k); }
// slab element (9 r + q) held by half h of small-k chunk c (see above)
__host__ __device__ constexpr int slab_elem(int c, int h) { return c < 4 ? 2 * c + h : (c < 8 ? 2 * c + 1 + h : 8 + 9 * h); }
__host__ __device__ inline int64_t small_index(int k, int np, int m, int a, int o, int q) {
    const int p = a >> 1, r = a & 1;
    const int c = q < 8 ? 4 * r + (q >> 1) : 8, h = q < 8 ? (q & 1) : r;
    return ((int64_t)((p * 9 + c) * np + m) * k + o) * 2 + h;
}
__host__ __device__ inline int64_t large_index(int k, int a, int o, int q) {
    const int t = a >> 2, e = 9 * (a & 3) + q, c = e >> 2;
    const int g = o >> 5, ng = (k - 32 * g) < 32 ? (k - 32 * g) : 32;
    return (int64_t)36 * k * t + 36 * 32 * g + (c * ng + (o & 31)) * 4 + (e & 3);
}
// lm_pk[j] = m | (np << 8) for small landmarks (pack slot, pack size); 0 for large ones.
__host__ __device__ inline int64_t r2_index(int k, int32_t pk, int a, int o, int q) {
    return k <= KSMALL ? small_index(k, pk >> 8, pk & 255, a, o, q) : large_index(k, a, o, q);
}
__host__ __device__ constexpr int64_t side_r1_floats(int k) { return pad4(27 * (int64_t)k); }
__host__ __device__ constexpr int64_t side_floats(int k) { return side_r1_floats(k) + 4 * (2 * (int64_t)k + 3) + 12; }
__host__ __device__ inline int64_t side_tl(int k) { return side_r1_floats(k); }
__host__ __device__ inline int64_t side_g(int k) { return side_r1_floats(k) + 4 * (2 * (int64_t)k + 3); }

// fast exact n / d for n, d < 2^16:  __umulhi(n, magic(d))
__host__ __device__ inline uint32_t divmagic(uint32_t d) { return (uint32_t)((0x100000000ull + d - 1) / d); }

struct Pack {
    int32_t lm0, np;  // first landmark (internal index) and number of landmarks (same k)
    int64_t base;     // float offset of the pack's R2 region
    int32_t obs0, k;  // first observation of the pack (its observations are contiguous) and k
    int32_t q0, pad1; // offset of the first landmark's q in qpk (landmark m: q0 + 2 k m)
};

// A stage of the small-k pipeline: consecutive packs whose R2 regions are contiguous, their
// camera indices and a table of work units (pack slot | row-pair range << 8).
struct SmallChunk {
    int32_t p0, np;          // packs [p0, p0 + np)
    int64_t base;            // float offset of the first pack's R2
    int32_t bytes;           // R2 bytes (multiple of 16)
    int32_t cam0, ncam;      // obs_cam[cam0 .. cam0 + ncam): 16-byte aligned superset of the packs' cameras
    int32_t unit0;           // units[unit0 .. unit0 + nunit) (nunit a multiple of 8, 0xFFFF = none)
    int32_t nunit;
    int32_t q0, nq;          // qpk[q0 .. q0 + nq): 16-byte aligned superset of the packs' q (K4 only)
    int32_t nreal;           // units before the 0xFFFF padding
};
constexpr int PACC_STRIDE = 56;             // per-camera slot of the preconditioner accumulator
#ifndef RBA_SP_STAGE_KB
#define RBA_SP_STAGE_KB 40
#endif
constexpr int SMALL_STAGE_BYTES = RBA_SP_STAGE_KB * 1024;  // >= largest pack (k = 16, np = 2: 36,864 B)
constexpr int SP_QCAP = 640;                   // q floats per small-pipe stage (K4; host guarantees)

struct PcgState {
    double rz;  // rho^T z
    double r0;  // |rho_0|
    double rn;  // |rho_k|
    int it, done, reason, active;
    double alpha, beta;       // step lengths of the current iteration (multi-CTA update kernels)
    unsigned int ctr_a, ctr_b;  // last-CTA-done counters of k_pcg_a / k_pcg_b (reset by that CTA)
    double tol;                 // stop when |rho| <= tol |rho_0| (reading C11); set by the host
    int max_iters, pad_;        // (rba_set_pcg_limits), read by k_pcg_init / k_pcg_b
};

// double scalars on the device (single buffer so one all-reduce covers them)
// [E, BAD] reduced at linearize; [ET, BADT, Q1R2, DAMPL] reduced after a trial; MODELP replicated;
// LAM = the damping lambda of the current attempt (every kernel that needs lambda reads it here, in
// FP64, so the device-side LM control can change it without the host); NSPD = preconditioner
// blocks found not SPD (the attempt is then treated as indefinite)
enum { SC_E = 0, SC_BAD, SC_ET, SC_BADT, SC_Q1R2, SC_DAMPL, SC_MODELP, SC_LAM, SC_NSPD, SC_N = 9 };

// Device-side Levenberg-Marquardt control (readings C9, C10, C13): the schedule lives in
// device memory and is advanced by k_lm_control, so an LM iteration (or a whole rba_lm_solve) runs
// without a host round trip.  Timestamps are %globaltimer (ns).
enum { TS_BEGIN = 0, TS_LIN, TS_MARG, TS_PRE, TS_PCG, TS_TRIAL, TS_END, TS_N };
struct LmDev {
    double lambda, nu;        // damping of the next attempt and the rejection multiplier
    double cost;              // E at the current state
    double min_rel_decrease;  // accept iff gain ratio > this (C9)
    double ftol;              // rba_lm_solve: stop once an accepted step decreases E by < ftol E
    int need_lin;             // the next attempt relinearizes (state changed / accepted)
    int stop;                 // 0 running, 1 converged (ftol), 2 error (point behind a camera / non-finite E)
    int lin_now;              // this attempt relinearized
    int accepted_now;         // this attempt was accepted (k_lm_commit copies the trial state)
    int64_t iter;             // LM iteration counter (every attempt counts, C13)
    int64_t target, n_done;   // rba_lm_solve: attempts requested / done in this call
    int64_t rep_cap;          // capacity of the device report array
    unsigned long long ts[TS_N];
};

enum { KID_LIN = 0, KID_MARG, KID_DAMP, KID_PRE, KID_MATVEC, KID_PCG, KID_BACKSUB, KID_COST, KID_N };

struct TileRef {
    int32_t lm, t;   // landmark (internal index) and 4-row tile index
    int64_t off;     // float offset of the tile in the arena
    int32_t k, obs0;  // track length (tile bytes = 144 k) and the landmark's first observation
    int64_t tl;      // float offset of the tile's 4 TL rows 3 + 4t .. 6 + 4t (K4's residual entries)
};

struct LargeItem {
    int32_t lm, t0, t1, pad;  // landmark (internal index) and tile range [t0, t1)
};

// Huge landmarks (k > KLARGE): work item of the two-pass matvec / preconditioner.
//  y pass:  (lm, t0 = t1 - 1 = tile)            y[yoff + 4t + r] = (A v) of row 4t + r
//  out pass: (lm, o0 = first camera block, [t0, t1) tiles)   out_o += sum_t slab_{o,t}^T y_t
struct HugeItem {
    int32_t lm, o0, t0, t1;
    int64_t yoff;
};
constexpr int HUGE_NT = 256;  // threads per CTA of the huge-k passes (camera blocks per out item)
constexpr int HUGE_TPO = (1 << 20) / (144 * HUGE_NT);  // tiles per out / preconditioner item (~1 MB)
constexpr int PIPE_NSLOT[5] = {8, 4, 2, 1, 1};          // consumer slots per CTA of the large-pipe classes
constexpr int DET_PART = 2048;  // deterministic scalar sums: per-CTA partials per sum (>= any grid used)
enum { DS_E = 0, DS_ET, DS_Q1R2, DS_DAMPL, DS_N };

struct DevProblem {
    int64_t n_p, n_l, n_obs;  // local counts (landmarks / observations of this shard)
    double huber;             // Huber parameter (px), 0 = squared loss
    // state
    double *cams, *cams_trial, *pts, *pts_trial;  // FP64 state (reading C23)
    double *campre, *campre_trial;                // per camera R, J_left, t, f, k1, k2 (24 doubles)
    int32_t *lm_orig;                             // internal -> caller landmark index (state I/O)
    double *pts_io;                               // 3 n_l(global) staging of the caller-order points
    // landmark metadata (internal order, sorted by k)
    int32_t *lm_k, *lm_obs0, *lm_pk;
    int32_t *lm_q;  // small landmarks: offset of their residual entries q (rows 3..2k+2) in qpk; -1 else
    float *qpk;     // copy of q of the small landmarks, consecutive (TMA-staged by the small K4 pipe)
    int64_t *lm_r2, *lm_side;
    int32_t *obs_cam, *obs_lm;
    double2 *obs_uv;
    // scaling / damping
    float *sp, *Dp2;
    double *cam_n2d;       // camera column norms^2 in FP64 (9 per camera): FP32 slices summed, or FP64 sums (sqrt-BA-64)
    double *sp64, *Dp264;  // FP64 copies of S_p and D_p^2 (exact FP64 values for sqrt-BA-64)
    float *lm_s, *lm_D;
    // arena
    float *arena;
    // reduced system / PCG
    // camera-space sums of K4 / K5: FP32 per-SM slices (nslice of them), FP64 after k_reduce_slices
    float *psl;   // K4: PACC_STRIDE per camera per slice: 45 upper-triangle of P_i + 9 of b~ (+2 pad)
    float *wsl;   // K5: 12 per camera per slice (9 used; 16-byte aligned float4 atomics)
    double *pd;   // K4 reduced: 54 per camera
    double *wd;   // K5 reduced: 9 per camera
    int nslice;
    double *bt, *Minv;                // b~ (9 n_p), block-Jacobi inverse (81 n_p), FP64
    double *x, *r, *z, *p, *w;        // PCG vectors (FP64, reading C24)
    float *p32;                       // p rounded to FP32: the matvec input
    float *dl;
    double *scal;
    PcgState *pcg;
    LmDev *lm;                // device-side LM schedule (rba_lm.cu)
    rba_lm_report *reps;      // device reports of the iterations of one rba_lm_step / rba_lm_solve call
    double *pcg_part;  // per-CTA partial dot products of the PCG update kernels (fixed-order sums)
    Pack *packs;            // small-k packs, classes G = 2, 4, 8, 16 back to back
    Pack *mid_packs;        // 17 <= k <= 32 (dense FP32): one landmark per "pack" for k_marg_small<32>
    uint16_t *units;        // small-k work units per stage
    LargeItem *marg_items;  // K2 work items (~1 MB of output each), classes NT = 64, 128, 256, 512
    TileRef *tiles;         // K4/K5 tile stream of the large landmarks, classes k <= 32, 64, 128, 256, 512
    SmallChunk *chunks;     // K4/K5 stage stream of the small-k packs
    int64_t *chunk_lo;      // tile-range boundaries of the persistent CTAs over the chunks
    int64_t *cta_lo;        // per class: tile range boundaries of the persistent CTAs (bytes-balanced)
    HugeItem *huge_y, *huge_out;  // k > KLARGE: y-pass items (one per tile), out/precond items
    HugeItem *huge_fused;         // k > KLARGE: fused-product items (landmark, ~1 MB tile range)
    float *ybuf;                  // k > KLARGE: y = A v, 4 floats per 4-row tile
    // explicit Schur-complement baseline (f3, rba_sc.cu): sc = 0 off (sqrt-BA), 1 FP32, 2 FP64
    int sc;
    int64_t nnzb;                 // 9 x 9 blocks of H~ on the covisibility graph (both triangles)
    int32_t *bsr_ptr, *bsr_col;   // BSR rows per camera, columns ascending
    void *bsr_val;                // nnzb x 81 (FP32 or FP64), row-major blocks
    void *sc_b;                   // b~ accumulator, 9 n_p
    void *sc_scratch;             // per observation: G_a (27) and L_a = G_a H_ll^-1 (27)
    // factored storage (f4, rba_factored.cu): landmark j's factors at arena + lm_r2[j]
    int fac;
    // sqrt-BA-64 (f2, rba_sqrtba64.cu): row-major FP64 blocks at arena64 + lm_r2[j]
    int s64;
    double *arena64, *lm_s64, *lm_D64;
    LargeItem *rcs_items;  // sqrt-BA-64 product / block-Jacobi items: (landmark, rows [t0, t1) of 3..2k+2)
    double *wsl64;         // sqrt-BA-64: per-SM FP64 slices of the product (nslice x 9 n_p), summed into wd
    int4 *s64_batches;     // sqrt-BA-64, k <= 16: TMA batches {count, stage doubles, first camera index (16-B
                           // aligned), camera indices staged}
    int4 *s64_brec;        // ... and per batch 64 x 2 landmark records {arena offset lo, hi, bytes, stage
                           // offset}, {k, row-3 offset in the stage, camera offset, 0}
    // deterministic mode (rba_options.deterministic): every contribution to a camera-space sum is
    // stored in its own slot of obuf; the slots of a camera are consecutive (camera-major) and are
    // added in a fixed order by k_det_reduce.  Family 1 = K1 camera norms (one slot per
    // observation), 4 = K4 block-Jacobi + b~, 5 = K5 product; a family's slots of observation `ob`
    // are slotF[ob] + part (the parts of one observation come from different work items: the
    // row-pair units of a small-k pack, the consumer runs a long track's tiles are split over, the
    // tile ranges of a huge track).  Scalar FP64 sums use per-CTA partials summed in CTA order.
    int det;
    int64_t arena_n;         // floats of the arena (bounds checks of the RBA_CHECKS build)
    int64_t n_slots[3];      // deterministic mode: slots of families 1, 4, 5
    float *obuf;
    int32_t *slot1, *slot4, *slot5;
    int64_t *camptr1, *camptr4, *camptr5;
    int32_t *run_part;     // large-pipe consumer runs (class offset + CTA * NSLOT + slot): the part index
                           // of the run's first landmark (its other landmarks start in it: part 0)
    double *det_part;      // DS_N x DET_PART per-CTA partials
    unsigned int *det_ctr; // DS_N last-CTA counters
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
    // auxiliary streams: independent per-class kernels fork off the context stream and join back
    static constexpr int NAUX = 5;
    cudaStream_t aux[NAUX] = {};
    cudaEvent_t ev_fork = nullptr, ev_join[NAUX] = {};
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
    std::vector<int32_t> h_pk, h_q;
    int64_t pack_lo[4] = {0, 0, 0, 0}, pack_hi[4] = {0, 0, 0, 0};  // G = 2, 4, 8, 16 pack ranges
    int64_t marg_lo[6] = {0, 0, 0, 0, 0, 0}, marg_hi[6] = {0, 0, 0, 0, 0, 0};  // K2 large items per class
    int64_t n_huge_y = 0, n_huge_out = 0, huge_max_k = 0;  // k > KLARGE (two-pass matvec)
    int64_t n_huge_fused = 0, n_huge_reg = 0;  // (items of k <= 1024 first: k_huge_fused<2, true>)
    int64_t fac_lo[5] = {0, 0, 0, 0, 0}, fac_hi[5] = {0, 0, 0, 0, 0};  // factored: G = 2..32 landmark ranges
    int64_t fac_big = 0;  // factored: first landmark with k > 32 (CTA-per-landmark matvec from here)
    int64_t s64_lo[5] = {0, 0, 0, 0, 0}, s64_hi[5] = {0, 0, 0, 0, 0}, s64_kmax[5] = {2, 2, 2, 2, 2};  // sqrt-BA-64 classes
    int64_t s64_ilo[5] = {0, 0, 0, 0, 0}, s64_ihi[5] = {0, 0, 0, 0, 0};  // their K2 items in marg_items
    int64_t s64_plo[5] = {0, 0, 0, 0, 0}, s64_phi[5] = {0, 0, 0, 0, 0};  // their product items
    int64_t s64_glo[4] = {0, 0, 0, 0}, s64_ghi[4] = {0, 0, 0, 0};  // k <= 32 items by group size 4..32
    int64_t s64_mlo[4] = {0, 0, 0, 0}, s64_mhi[4] = {0, 0, 0, 0};  // the same as landmark ranges
    int64_t s64_blo[3] = {0, 0, 0}, s64_bhi[3] = {0, 0, 0};  // k <= 4 / 8 / 16: their TMA batches
    int64_t cta_off[5] = {0, 0, 0, 0, 0}, cta_n[5] = {0, 0, 0, 0, 0};    // K4/K5 CTA ranges per class
    int64_t run_off[5] = {0, 0, 0, 0, 0};  // deterministic mode: per class offset into d.run_part
    int64_t n_chunks = 0, chunk_ctas = 0;
    int64_t n_packs = 0, max_large_k = 0;
    int64_t n_mid_packs = 0;  // landmarks marginalized by the warp-per-landmark K2 (17 <= k <= 32)
    int num_sms = 148;
    int64_t arena_floats = 0, logical_bytes = 0;
    double marg_bytes = 0, matvec_bytes = 0, backsub_bytes = 0;
    double bs_bytes[3] = {0, 0, 0};  // K7 regimes k <= 16 | 16 < k <= 256 | k > 256: bytes, end landmark
    int64_t bs_hi[3] = {0, 0, 0};  // algorithmic bytes per launch
    std::vector<void *> allocations;
    // pinned host scratch
    double *h_scal = nullptr;
    rba::PcgState *h_pcg = nullptr;
    // solver state of the step-by-step API (call ordering; the LM schedule itself lives on the
    // device, rba::LmDev)
    bool linearized = false, marginalized = false, solved = false, backsubbed = false;
    double lambda_blocks = 0.0;
    double cost = 0.0;
    bool lm_dirty = true;  // a step-by-step call changed the blocks / state: the next LM step relinearizes
    int64_t launches = 0;
    int64_t device_bytes = 0;
    // device-side LM loop (rba_lm.cu): one CUDA graph = while (LM) { if (relinearize) {K1, K2} else
    // {K3}; K4; while (PCG) {K5, K6}; K7, K8, control }, and the kernel-node counts of its parts
    struct LmGraph {
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        bool failed = false, built = false;
        int64_t n_head = 0, n_lin = 0, n_redamp = 0, n_mid = 0, n_pcg = 0, n_tail = 0;
    } lmg;
    rba_lm_report *h_reps = nullptr;  // pinned host copy of the device reports
    static constexpr int REP_CAP = 1024;
    // profiling
    // PCG as a CUDA graph with a device-side while loop (single GPU; NCCL path uses host batches)
    cudaGraph_t pcg_graph = nullptr;
    cudaGraphExec_t pcg_exec = nullptr;
    bool pcg_graph_failed = false;
    int64_t graph_body_kernels = 0;  // kernels per PCG-graph iteration (launch accounting)
    bool pcg_fused = false;          // the last PCG product left its sum in the per-SM slices
    bool nofork = false;             // launch the per-class kernels on the context stream only
    bool emulate_comm = false;       // RBA_EMULATE_COMM: the multi-GPU PCG path (host loop, product
                                     // reduced before the update) on one GPU, all-reduces skipped
    bool no_graph = false;           // RBA_NO_GRAPH (read at rba_create): eager LM / host-polled PCG
    bool host_reduce_path() const { return have_comm || emulate_comm; }
    bool profiling = false;
    int64_t prof_real_matvecs = 0;  // matvecs that did work (PCG iterations + hook calls) since rba_profile
    std::vector<rba::Launch> prof;
    std::vector<cudaEvent_t> ev_pool;
};

namespace rba {
// shared host helpers (rba_api.cu)
rba_status set_error(rba_status s, const std::string &msg);
rba_status allreduce(rba_ctx *c, void *buf, size_t count, ncclDataType_t t);
// device-side LM (rba_lm.cu)
cudaError_t launch_set_lambda(rba_ctx *c, double lambda);
cudaError_t launch_set_pcg_limits(rba_ctx *c, double tol, int max_iters);
cudaError_t launch_lm_init(rba_ctx *c, double lambda, double nu, int reset_iter);
cudaError_t launch_lm_need_lin(rba_ctx *c);
rba_status build_pcg_graph(rba_ctx *c);
// kernel launchers (rba_kernels.cu); each returns cudaGetLastError()
cudaError_t launch_check_depth(rba_ctx *c, int *d_bad);
cudaError_t launch_cam_prep(rba_ctx *c, int trial);
cudaError_t launch_reduce_cam_norms(rba_ctx *c);
void launch_reduce_slices64(rba_ctx *c, double *out);
cudaError_t launch_pts_permute(rba_ctx *c, int to_internal);
cudaError_t query_nsmid(rba_ctx *c, int *d_scratch, int *out);
cudaError_t launch_linearize(rba_ctx *c);
cudaError_t launch_cam_scale(rba_ctx *c);
cudaError_t launch_marginalize(rba_ctx *c);
cudaError_t launch_redamp(rba_ctx *c);
cudaError_t launch_precond_rhs(rba_ctx *c);
cudaError_t launch_precond_finalize(rba_ctx *c);
cudaError_t launch_matvec(rba_ctx *c, const float *v, float *out);
cudaError_t launch_matvec_pcg(rba_ctx *c);
cudaError_t launch_pcg_init(rba_ctx *c, cudaGraphConditionalHandle h = 0, int use_h = 0);
cudaError_t launch_pcg_step(rba_ctx *c, cudaGraphConditionalHandle h = 0, int use_h = 0);
cudaError_t launch_backsub(rba_ctx *c);
cudaError_t launch_trial_cost(rba_ctx *c);
cudaError_t launch_cost(rba_ctx *c, int at_trial, int slot);
cudaError_t launch_commit(rba_ctx *c);
cudaError_t launch_add_damping(rba_ctx *c, const float *v, float *out);
// explicit Schur complement (rba_sc.cu)
cudaError_t launch_sc_build(rba_ctx *c);
cudaError_t launch_sc_precond(rba_ctx *c);
void launch_sc_spmv(rba_ctx *c, const PcgState *st, const float *v32);
// factored storage (rba_factored.cu)
void launch_fac_matvec(rba_ctx *c, const float *v, const PcgState *st);
void launch_fac_precond(rba_ctx *c);
cudaError_t launch_fac_backsub(rba_ctx *c);
cudaError_t launch_fac_redamp(rba_ctx *c);
// sqrt-BA-64 (rba_sqrtba64.cu)
cudaError_t launch_marg64(rba_ctx *c);
cudaError_t launch_redamp64(rba_ctx *c);
void launch_rcs64(rba_ctx *c, const double *v, const PcgState *st);
void launch_pre64(rba_ctx *c);
cudaError_t launch_backsub64(rba_ctx *c);
void launch_f2d64(rba_ctx *c, const float *a, double *b, int64_t n);
cudaError_t launch_sc_backsub(rba_ctx *c);
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
