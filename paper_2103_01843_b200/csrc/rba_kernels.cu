// rba_kernels.cu -- sm_100a kernels of the FP32 sqrt-BA hot path (product path; no oracle code).
//
//  K0 k_check_depth       validation: every observation in front of its camera
//     k_cam_prep          per camera R(w), J_left(w), t, f, k1, k2 once per state
//  K1 k_linearize         residuals, E, camera Jacobian column norms into per-SM slices
//  K1b k_cam_scale        s = 1/(1+|c|), D^2 = clamp(|c|^2 s^2) (C7, C8)
//  K2 k_marg_small<G>     k <= 16: G-lane group per landmark: Jacobians, 3 Householder reflectors,
//                         compact-WY emission, side regions written by one TMA bulk store
//     k_marg_large<NT>    k > 16: CTA per (landmark, ~4 MB of tiles); compact-WY emission of
//                         Q^T [J_p | J_l | r] with the 6 damping Givens rotations folded in
//
//  K3 k_redamp            undo / re-apply the 6 damping rotations in place (Fig. 3)
//  K4 k_small_pipe<1>,    block-Jacobi blocks + b~ = sum A^T q
//     k_large_pipe<..,1>
//     k_precond_finalize  + lambda D_p^2, Cholesky inverse per camera (C12)
//  K5 k_small_pipe<0>,    H~ v = sum_j A_j^T (A_j v_j) (Eq. cg_mult), one HBM pass:
//     k_large_pipe<..,0>  TMA (cp.async.bulk) + mbarrier pipelines, persistent CTAs;
//     k_huge_*            k > 512: fused two-read product with TMA L2 prefetch
//     k_reduce_slices     FP64 sum of the per-SM FP32 slices (C24)
//  K6 k_pcg_init, k_pcg_a/b/c   one PCG iteration as three multi-CTA kernels (fixed-order dots);
//                         the loop is a CUDA graph with a device-side while node
//  K7 k_backsub           dl = -R^_1^-1 (Q^_1^T r^ + Q^_1^T J_p dp), trial point
//  K8 k_cost              E at the current or trial state (Eq. ba_energy; C14, C17)
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>

#include "rba_internal.cuh"
#include "rba_model.cuh"

#ifndef RBA_K2_EXP
#define RBA_K2_EXP 0  // K2 measurement experiments (tools/): 1 = no R2 emission, 2 = no camera model
#endif

namespace rba {

// ============================================================================ deterministic mode
// (rba_options.deterministic).  A camera-space contribution goes to its own slot
// (plain stores, no atomics); k_det_reduce adds the slots of a camera in a fixed order.
__device__ __forceinline__ void det_store12(const DevProblem &d, int64_t slot, const float *acc) {
    RBA_CHECK(slot >= 0 && 12 * slot + 12 <= 56 * d.n_slots[1] + 12 * (d.n_slots[2] + d.n_slots[0]));
    float4 *o4 = reinterpret_cast<float4 *>(d.obuf + 12 * slot);
    o4[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
    o4[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
    o4[2] = make_float4(acc[8], 0.f, 0.f, 0.f);
}
__device__ __forceinline__ void det_store54(const DevProblem &d, int64_t slot, const float *P, const float *b) {
    RBA_CHECK(slot >= 0 && slot < d.n_slots[1]);
    float4 *a4 = reinterpret_cast<float4 *>(d.obuf + (int64_t)PACC_STRIDE * slot);
#pragma unroll
    for (int i = 0; i < 11; i++) a4[i] = make_float4(P[4 * i], P[4 * i + 1], P[4 * i + 2], P[4 * i + 3]);
    a4[11] = make_float4(P[44], b[0], b[1], b[2]);
    a4[12] = make_float4(b[3], b[4], b[5], b[6]);
    a4[13] = make_float4(b[7], b[8], 0.f, 0.f);
}

// out[NV cam + e] = sum over the camera's slots m (ascending) of obuf[stride m + e], FP64: thread t
// takes slots t, t + 256, ... in order, then a fixed warp butterfly and a fixed order over warps.
template <int NV>
__global__ void __launch_bounds__(256) k_det_reduce(const float *__restrict__ obuf, const int64_t *__restrict__ camptr,
                                                    int stride, double *__restrict__ out,
                                                    const PcgState *__restrict__ st) {
    if (st && st->done) return;  // PCG graph: no product ran
    __shared__ double part[8][NV];
    const int64_t cam = blockIdx.x;
    const int64_t a = camptr[cam], b = camptr[cam + 1];
    double acc[NV];
#pragma unroll
    for (int e = 0; e < NV; e++) acc[e] = 0.0;
    for (int64_t m = a + threadIdx.x; m < b; m += 256) {
        const float4 *row = reinterpret_cast<const float4 *>(obuf + (int64_t)stride * m);
#pragma unroll
        for (int q = 0; q < (NV + 3) / 4; q++) {
            const float4 x = __ldcs(row + q);
            const float v[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int u = 0; u < 4; u++)
                if (4 * q + u < NV) acc[4 * q + u] += (double)v[u];
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int e = 0; e < NV; e++) {
        double v = acc[e];
#pragma unroll
        for (int m = 16; m; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
        if (lane == 0) part[warp][e] = v;
    }
    __syncthreads();
    if (threadIdx.x < NV) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < 8; w++) t += part[w][threadIdx.x];
        out[NV * cam + threadIdx.x] = t;
    }
}

// Grid-wide FP64 sum in a fixed order: the block total v (valid in every thread) goes to
// parts[blockIdx.x]; the last CTA to finish adds the parts in CTA order into *out.
__device__ void det_grid_sum(double v, double *parts, unsigned int *ctr, double *out) {
    __shared__ bool last;
    if (threadIdx.x == 0) parts[blockIdx.x] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(ctr, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (unsigned int b = 0; b < gridDim.x; b++) t += __ldcg(parts + b);
        *out = t;
        *ctr = 0;
    }
}

// ============================================================================ K0 / K1
__global__ void k_check_depth(DevProblem d, int *bad) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= d.n_obs) return;
    double c[CAMPRE], r[2];
    load_pre(d.campre, d.obs_cam[i], c);
    const double *X = d.pts + 3 * (int64_t)d.obs_lm[i];
    const double2 uv = d.obs_uv[i];
    const double Pz = cam_model_pre<float>(c, X[0], X[1], X[2], uv.x, uv.y, r, nullptr, nullptr);
    if (!(Pz < -1e-8) || !isfinite(r[0]) || !isfinite(r[1])) atomicAdd(bad, 1);
}

// K1: residuals, E and camera column norms^2 (sum over the camera's observations).
// Grid-stride (a few CTAs per SM): the per-CTA FP64 sums of E go to one address, so fewer CTAs
// means fewer serialized same-address atomics.
__global__ void __launch_bounds__(256) k_linearize(DevProblem d) {
    __shared__ double red[32];
    double e = 0.0, bad = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int cam_n = i < d.n_obs ? __ldg(d.obs_cam + i) : 0, lm_n = i < d.n_obs ? __ldg(d.obs_lm + i) : 0;
    for (; i < d.n_obs; i += stride) {
        double c[CAMPRE], r[2];
        float Jc[18], Jl[6];
        const int cam = cam_n, lm = lm_n;  // indices of the next observation are loaded one ahead
        if (i + stride < d.n_obs) cam_n = __ldg(d.obs_cam + i + stride), lm_n = __ldg(d.obs_lm + i + stride);
        load_pre(d.campre, cam, c);
        const double *X = d.pts + 3 * (int64_t)lm;
        const double2 uv = d.obs_uv[i];
        if (d.s64) {  // sqrt-BA-64: FP64 Jacobians and FP64 norm sums
            double Jcd[18], Jld[6];
            const double Pz = cam_model_pre<double>(c, X[0], X[1], X[2], uv.x, uv.y, r, Jcd, Jld);
            if (!(Pz < 0.0)) bad += 1.0;
            e += robust_rho(r[0] * r[0] + r[1] * r[1], d.huber);
            apply_irls<double>(r, Jcd, Jld, d.huber);
            double *sl = d.wsl64 + ((int64_t)smid() * d.n_p + cam) * 9;  // this SM's FP64 slice
#pragma unroll
            for (int q = 0; q < 9; q++) atomicAdd(sl + q, Jcd[q] * Jcd[q] + Jcd[9 + q] * Jcd[9 + q]);
        } else {
            const double Pz = cam_model_pre(c, X[0], X[1], X[2], uv.x, uv.y, r, Jc, Jl);
            if (!(Pz < 0.0)) bad += 1.0;
            e += robust_rho(r[0] * r[0] + r[1] * r[1], d.huber);
            apply_irls(r, Jc, Jl, d.huber);
            float n2[9];
#pragma unroll
            for (int q = 0; q < 9; q++) n2[q] = Jc[q] * Jc[q] + Jc[9 + q] * Jc[9 + q];
            if (d.det) det_store12(d, d.slot1[i], n2);  // own slot (k_det_reduce)
            else flush_cam12(wslice(d), cam, n2);     // per-SM slice (k_reduce_slices sums them in FP64)
        }
    }
    e = block_sum_d(e, red);
    bad = block_sum_d(bad, red);
    if (threadIdx.x == 0 && bad > 0) atomicAdd(d.scal + SC_BAD, bad);  // an integer count: exact
    if (d.det) det_grid_sum(e, d.det_part + DS_E * DET_PART, d.det_ctr + DS_E, d.scal + SC_E);
    else if (threadIdx.x == 0) atomicAdd(d.scal + SC_E, e);
}

__global__ void k_cam_scale(DevProblem d, float dmin, float dmax) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 9 * d.n_p) return;
    if (d.s64) {
        const double n2 = d.cam_n2d[i];
        const double s = 1.0 / (1.0 + sqrt(n2));
        const double D2 = fmin(fmax(n2 * s * s, (double)dmin), (double)dmax);
        d.sp64[i] = s, d.Dp264[i] = D2;
        d.sp[i] = (float)s, d.Dp2[i] = (float)D2;
        return;
    }
    float n2 = (float)d.cam_n2d[i];
    float s = 1.f / (1.f + sqrtf(n2));
    d.sp[i] = s;
    d.Dp2[i] = fminf(fmaxf(n2 * s * s, dmin), dmax);
    d.sp64[i] = s;
    d.Dp264[i] = d.Dp2[i];
}

__device__ __forceinline__ void named_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ============================================================================ K2 emission
// Compact-WY form of the marginalized block (Householder): Q^T = I - V T^T V^T, so every
// output row L of the pose columns of camera block o is
//     out[L, 9o+q] = Jterm(L, o, q) - V[L] . M[:, 9o+q],    M = T^T V^T J_p (3 x 9k),
// and J_p is block diagonal (observation o owns rows 2o, 2o+1).  The thread (lane) that owns
// camera block o keeps M[:, 9o..9o+8] and its two scaled J_p rows in registers, so each output
// float costs 3 FMA and is stored coalesced in the matvec layout.  The 6 damped rows (logical
// 0..2 and 2k..2k+2) use V_eff = Gm V and mix J_p rows 0..2 with the damping rotations Gm.
struct BlockWY {
    float m[3][9];   // M[:, 9o + q]
    float jp[2][9];  // scaled J_p rows 2o, 2o+1
};

// 9 values of logical row L for camera block o.  VR = V rows (specials already V_eff), GM = Gm.
__device__ __forceinline__ void wy_row(const BlockWY &B, const float4 *VR, const float *GM, int k, int L, int o,
                                       float *out9) {
    const float4 V = VR[L];
    float c0 = 0.f, c1 = 0.f;
    if (L >= 3 && L < 2 * k) {
        if (o == (L >> 1)) {
            c0 = (L & 1) ? 0.f : 1.f;
            c1 = (L & 1) ? 1.f : 0.f;
        }
    } else {
        const int s = L < 3 ? L : L - 2 * k + 3;
        if (o == 0) c0 = GM[3 * s], c1 = GM[3 * s + 1];
        else if (o == 1) c0 = GM[3 * s + 2];
    }
#pragma unroll
    for (int q = 0; q < 9; q++)
        out9[q] = c0 * B.jp[0][q] + c1 * B.jp[1][q] - (V.x * B.m[0][q] + V.y * B.m[1][q] + V.z * B.m[2][q]);
}

// Fast path for the plain rows L in [3, 2k) (no damping rotation involved): the J_p term is
// nonzero only in the 2 rows of the lane's own observation, so every other lane spends 3 FMA per
// output (same rounding as wy_row: -(V.M) then + the J_p entry).
__device__ __forceinline__ void wy_row_plain(const BlockWY &B, const float4 V, int L, int o, float *out9) {
#pragma unroll
    for (int q = 0; q < 9; q++) out9[q] = fmaf(-V.z, B.m[2][q], fmaf(-V.y, B.m[1][q], -V.x * B.m[0][q]));
    if (o == (L >> 1)) {
        const bool odd = L & 1;
#pragma unroll
        for (int q = 0; q < 9; q++) out9[q] += odd ? B.jp[1][q] : B.jp[0][q];
    }
}

// Packed forms of wy_row_plain / wy_row for the small-k pack layout (rba_internal.cuh): a row's 9
// values as 4 (q, q+1) pairs + q = 8, each pair one FFMA2 (sm_100 packed FP32 FMA) per term, in
// the same operation order (so the same rounding) as the scalar plain row.
struct Row9 {
    float2 p[4];
    float e;
};
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ Row9 wy_negvm(const BlockWY &B, const float4 V) {  // -(V . M[:, q])
    const float nx = -V.x, ny = -V.y, nz = -V.z;
    Row9 r;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const int q = 2 * i;
        float2 t = __fmul2_rn(f2(nx, nx), f2(B.m[0][q], B.m[0][q + 1]));
        t = __ffma2_rn(f2(ny, ny), f2(B.m[1][q], B.m[1][q + 1]), t);
        r.p[i] = __ffma2_rn(f2(nz, nz), f2(B.m[2][q], B.m[2][q + 1]), t);
    }
    r.e = fmaf(nz, B.m[2][8], fmaf(ny, B.m[1][8], nx * B.m[0][8]));
    return r;
}
__device__ __forceinline__ void row9_add_jp(Row9 &r, const BlockWY &B, int i) {  // += J_p row i
#pragma unroll
    for (int j = 0; j < 4; j++) r.p[j] = __fadd2_rn(r.p[j], f2(B.jp[i][2 * j], B.jp[i][2 * j + 1]));
    r.e += B.jp[i][8];
}
__device__ __forceinline__ Row9 wy_row_plain2(const BlockWY &B, const float4 V, int L, int o) {
    Row9 r = wy_negvm(B, V);
    if (o == (L >> 1)) row9_add_jp(r, B, L & 1);
    return r;
}
// damped rows (L < 3 or L >= 2k): V_eff from VR, J_p rows 0..2 mixed by Gm (blocks 0 and 1 only)
__device__ __forceinline__ Row9 wy_row2(const BlockWY &B, const float4 *VR, const float *GM, int k, int L, int o) {
    Row9 r = wy_negvm(B, VR[L]);
    if (L >= 3 && L < 2 * k) {
        if (o == (L >> 1)) row9_add_jp(r, B, L & 1);
    } else if (o < 2) {
        const int s = L < 3 ? L : L - 2 * k + 3;
        const float c0 = o == 0 ? GM[3 * s] : GM[3 * s + 2], c1 = o == 0 ? GM[3 * s + 1] : 0.f;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const float2 u = __ffma2_rn(f2(c1, c1), f2(B.jp[1][2 * j], B.jp[1][2 * j + 1]),
                                        __fmul2_rn(f2(c0, c0), f2(B.jp[0][2 * j], B.jp[0][2 * j + 1])));
            r.p[j] = __fadd2_rn(r.p[j], u);
        }
        r.e += fmaf(c1, B.jp[1][8], c0 * B.jp[0][8]);
    }
    return r;
}

// M column block from V rows 2o, 2o+1 and T (upper 3x3, entries T00..T22)
__device__ __forceinline__ void wy_m(BlockWY &B, float4 v0, float4 v1, float T00, float T01, float T02, float T11,
                                     float T12, float T22) {
#pragma unroll
    for (int q = 0; q < 9; q++) {
        const float j0 = B.jp[0][q], j1 = B.jp[1][q];
        const float W0 = v0.x * j0 + v1.x * j1, W1 = v0.y * j0 + v1.y * j1, W2 = v0.z * j0 + v1.z * j1;
        B.m[0][q] = T00 * W0;
        B.m[1][q] = T01 * W0 + T11 * W1;
        B.m[2][q] = T02 * W0 + T12 * W1 + T22 * W2;
    }
}

// V_eff rows of the 6 damped rows, written to VR[0..2] and VR[2k..2k+2]
__device__ __forceinline__ float4 veff(const float *Gm, const float *V3, int s) {
    float4 ve;
    ve.x = Gm[s * 3] * V3[0] + Gm[s * 3 + 1] * V3[3] + Gm[s * 3 + 2] * V3[6];
    ve.y = Gm[s * 3] * V3[1] + Gm[s * 3 + 1] * V3[4] + Gm[s * 3 + 2] * V3[7];
    ve.z = Gm[s * 3] * V3[2] + Gm[s * 3 + 1] * V3[5] + Gm[s * 3 + 2] * V3[8];
    ve.w = 0.f;
    return ve;
}

// factored storage (f4): one observation's record (28 floats: scaled J_p rows 2o,
// 2o+1 | V rows 2o, 2o+1 | (Q^T r^) rows 2o, 2o+1 | pad) and the landmark header (44 floats: R,
// T, Givens, damped R^1, damped special residual entries)
__device__ __forceinline__ void fac_write_obs(float *rec, const BlockWY &B, const float *v0, const float *v1, float q0,
                                              float q1) {
    float4 *r4 = reinterpret_cast<float4 *>(rec);
    r4[0] = make_float4(B.jp[0][0], B.jp[0][1], B.jp[0][2], B.jp[0][3]);
    r4[1] = make_float4(B.jp[0][4], B.jp[0][5], B.jp[0][6], B.jp[0][7]);
    r4[2] = make_float4(B.jp[0][8], B.jp[1][0], B.jp[1][1], B.jp[1][2]);
    r4[3] = make_float4(B.jp[1][3], B.jp[1][4], B.jp[1][5], B.jp[1][6]);
    r4[4] = make_float4(B.jp[1][7], B.jp[1][8], v0[0], v0[1]);
    r4[5] = make_float4(v0[2], v1[0], v1[1], v1[2]);
    r4[6] = make_float4(q0, q1, 0.f, 0.f);
}
__device__ __forceinline__ void fac_write_hdr(float *h, const float *R, float T00, float T01, float T02, float T11,
                                              float T12, float T22, const float *g, const float *L6, const float *rr6) {
#pragma unroll
    for (int i = 0; i < 9; i++) h[i] = R[i];
    h[9] = T00, h[10] = T01, h[11] = T02, h[12] = T11, h[13] = T12, h[14] = T22;
#pragma unroll
    for (int i = 0; i < 12; i++) h[15 + i] = g[i];
#pragma unroll
    for (int i = 0; i < 9; i++) h[27 + i] = L6[i];
#pragma unroll
    for (int i = 0; i < 6; i++) h[36 + i] = rr6[i];
    h[42] = 0.f, h[43] = 0.f;
}

// ============================================================================ K2 small (k <= 32)
// Warp <-> pack of np same-k landmarks; group of G lanes <-> landmark; lane o <-> observation o
// and camera block o.  Per-group shared memory: VR (2G+3 float4) + GM (18, padded to 20).
template <int G>
struct SmallTab {
    static constexpr int VR = 4 * (2 * G + 3);
    static constexpr int FLOATS = VR + 20;
    // the pack's side regions (R1 | TL | G of its <= 32/G landmarks, consecutive in the arena) are
    // assembled in shared memory and written with one bulk store (k <= G; k = 2 for G = 2)
    static constexpr int SIDE = (32 / G) * (int)side_floats(G);
};

template <int G>
#ifndef RBA_MARG_SMALL_MINB
#define RBA_MARG_SMALL_MINB 4  // 128 registers: 4 CTAs per SM (measured 3.35 -> 3.22 ms K2 on cfg4)
#endif
__global__ void __launch_bounds__(128, RBA_MARG_SMALL_MINB) k_marg_small(DevProblem d, const Pack *__restrict__ packs, int64_t pk_lo, int64_t pk_hi, float dmin,
                                                    float dmax) {
    constexpr int NG = 32 / G;
    using TB = SmallTab<G>;
    extern __shared__ float4 smem4[];
    float *smem = reinterpret_cast<float *>(smem4);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int grp = lane / G, gl = lane % G;
    const int64_t pi = pk_lo + (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    if (pi >= pk_hi) return;  // warp-uniform
    const Pack pack = packs[pi];  // (G = 32: one landmark of 17..32 observations, tile layout)
    const bool valid = grp < pack.np;
    const int64_t j = pack.lm0 + (valid ? grp : 0);
    const int k = pack.k;  // (the pack's observations are contiguous: no per-landmark index loads)
    // the pack's side-region offset, loaded now so the bulk store after the prologue does not wait on it
    int64_t side_off = 0;
    if (lane == 0) side_off = __ldg(d.lm_side + pack.lm0);
    const bool act = valid && gl < k;
    float *tab = smem + (warp * NG + grp) * TB::FLOATS;
    float *sside = smem + 4 * NG * TB::FLOATS + warp * TB::SIDE;  // this warp's pack side regions
    float4 *VR = reinterpret_cast<float4 *>(tab);
    float *GM = tab + TB::VR;

    // ---- per-observation Jacobians (lane gl <-> observation gl; rows 2gl, 2gl+1)
    float r[2] = {0.f, 0.f}, Jc[18], Jl[6];
#pragma unroll
    for (int i = 0; i < 18; i++) Jc[i] = 0.f;
#pragma unroll
    for (int i = 0; i < 6; i++) Jl[i] = 0.f;
    int cam = 0;
    float spc[9];
    if (act) {
        const int64_t o = (int64_t)pack.obs0 + grp * k + gl;
#if RBA_K2_EXP == 5  // measurement experiment: no dependent camera-index load
        cam = (int)(o % d.n_p);
#else
        cam = __ldg(d.obs_cam + o);
#endif
#pragma unroll
        for (int q = 0; q < 9; q++) spc[q] = __ldg(d.sp + 9 * cam + q);  // issued with the camera loads
        double c[CAMPRE], rd[2];
        load_pre(d.campre, cam, c);
        const double *X = d.pts + 3 * j;
        const double2 uv = d.obs_uv[o];
#if RBA_K2_EXP == 2  // measurement experiment: skip the camera model (emission-bound time)
        for (int q = 0; q < 18; q++) Jc[q] = (float)c[q] + q;
        for (int q = 0; q < 6; q++) Jl[q] = (float)c[q + 9] + q * gl;
        rd[0] = uv.x, rd[1] = uv.y;
#else
        cam_model_pre(c, X[0], X[1], X[2], uv.x, uv.y, rd, Jc, Jl);
#endif
        apply_irls(rd, Jc, Jl, d.huber);
        r[0] = (float)rd[0];
        r[1] = (float)rd[1];
    }
    // ---- landmark column scaling (C7, C8) over the landmark's own observations
    float sl[3], Dl[3];
#pragma unroll
    for (int q = 0; q < 3; q++) {
        float n2 = group_sum<G>(Jl[q] * Jl[q] + Jl[3 + q] * Jl[3 + q]);
        sl[q] = 1.f / (1.f + sqrtf(n2));
        Dl[q] = sqrtf(fminf(fmaxf(n2 * sl[q] * sl[q], dmin), dmax));
    }
    BlockWY B;
    float X[2][3], rv[2] = {r[0], r[1]};
#pragma unroll
    for (int q = 0; q < 9; q++) {
        const float s = act ? spc[q] : 0.f;
        B.jp[0][q] = Jc[q] * s;
        B.jp[1][q] = Jc[9 + q] * s;
    }
#pragma unroll
    for (int q = 0; q < 3; q++) {
        X[0][q] = Jl[q] * sl[q];
        X[1][q] = Jl[3 + q] * sl[q];
    }
    // ---- Householder QR of the 2k x 3 landmark Jacobian, reading C4 for the sign
    float V[2][3], tau[3];
#if RBA_K2_EXP == 3  // measurement experiment: no Householder reductions (trivial reflectors)
    for (int c = 0; c < 3; c++) {
        tau[c] = 1.f;
        for (int rr = 0; rr < 2; rr++) V[rr][c] = X[rr][c];
    }
#else
#pragma unroll
    for (int c = 0; c < 3; c++) {
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
        for (int rr = 0; rr < 2; rr++) {
            const int a = 2 * gl + rr;
            const float x = (act && a >= c) ? X[rr][c] : 0.f;
            s0 += x * x;
            s1 += (c + 1 < 3) ? x * X[rr][(c + 1) % 3] : 0.f;
            s2 += (c + 2 < 3) ? x * X[rr][(c + 2) % 3] : 0.f;
            s3 += x * rv[rr];
        }
        s0 = group_sum<G>(s0);
        s1 = group_sum<G>(s1);
        s2 = group_sum<G>(s2);
        s3 = group_sum<G>(s3);
        const int pl = c >> 1, pr = c & 1;  // pivot row c lives in lane c>>1, local row c&1
        const float x0 = __shfl_sync(0xffffffffu, X[pr][c], pl, G);
        const float y1 = __shfl_sync(0xffffffffu, X[pr][(c + 1) % 3], pl, G);
        const float y2 = __shfl_sync(0xffffffffu, X[pr][(c + 2) % 3], pl, G);
        const float yr = __shfl_sync(0xffffffffu, rv[pr], pl, G);
        const float sig = sqrtf(s0);
        const float alpha = x0 >= 0.f ? -sig : sig;
        const float vtv = 2.f * sig * (sig + fabsf(x0));
        const float tc = vtv > 0.f ? 2.f / vtv : 0.f;
        tau[c] = tc;
        const float d1 = s1 - alpha * y1, d2 = s2 - alpha * y2, dr = s3 - alpha * yr;
#pragma unroll
        for (int rr = 0; rr < 2; rr++) {
            const int a = 2 * gl + rr;
            float vv = 0.f;
            if (act && a >= c) vv = (a == c) ? x0 - alpha : X[rr][c];
            V[rr][c] = vv;
            if (c + 1 < 3) X[rr][(c + 1) % 3] -= tc * vv * d1;
            if (c + 2 < 3) X[rr][(c + 2) % 3] -= tc * vv * d2;
            rv[rr] -= tc * vv * dr;
            if (a == c) X[rr][c] = alpha;
            else if (a > c) X[rr][c] = 0.f;
        }
    }
#endif
    // ---- compact WY: T upper 3x3 (Q = I - V T V^T, Q^T = I - V T^T V^T)
    float p01 = 0.f, p02 = 0.f, p12 = 0.f;
#pragma unroll
    for (int rr = 0; rr < 2; rr++) {
        p01 += V[rr][0] * V[rr][1];
        p02 += V[rr][0] * V[rr][2];
        p12 += V[rr][1] * V[rr][2];
    }
    p01 = group_sum<G>(p01);
    p02 = group_sum<G>(p02);
    p12 = group_sum<G>(p12);
    const float T00 = tau[0], T11 = tau[1], T22 = tau[2];
    const float T01 = -tau[1] * T00 * p01;
    const float T02 = -tau[2] * (T00 * p02 + T01 * p12);
    const float T12 = -tau[2] * T11 * p12;
    if (act) {
#pragma unroll
        for (int rr = 0; rr < 2; rr++) {
            const int a = 2 * gl + rr;
            if (a >= 3) VR[a] = make_float4(V[rr][0], V[rr][1], V[rr][2], 0.f);
        }
    }
    // ---- damping (fused): R1 rows 0..2 and V rows 0..2 from lanes 0, 1
    float R[9], rr3[3], V3[9];
#pragma unroll
    for (int q = 0; q < 3; q++) {
        R[q] = __shfl_sync(0xffffffffu, X[0][q], 0, G);
        R[3 + q] = __shfl_sync(0xffffffffu, X[1][q], 0, G);
        R[6 + q] = __shfl_sync(0xffffffffu, X[0][q], 1, G);
        V3[q] = __shfl_sync(0xffffffffu, V[0][q], 0, G);
        V3[3 + q] = __shfl_sync(0xffffffffu, V[1][q], 0, G);
        V3[6 + q] = __shfl_sync(0xffffffffu, V[0][q], 1, G);
    }
    rr3[0] = __shfl_sync(0xffffffffu, rv[0], 0, G);
    rr3[1] = __shfl_sync(0xffffffffu, rv[1], 0, G);
    rr3[2] = __shfl_sync(0xffffffffu, rv[0], 1, G);
    const float sq = sqrtf((float)d.scal[SC_LAM]);  // lambda of this attempt (device-side LM control)
    const float sD[3] = {sq * Dl[0], sq * Dl[1], sq * Dl[2]};
    float L6[18], Gm[18], rr6[6], g[12];
    damp_rotations(R, rr3, sD, L6, Gm, rr6, g);
    if (valid && gl == 0) {
#pragma unroll
        for (int s = 0; s < 6; s++) VR[s < 3 ? s : 2 * k + s - 3] = veff(Gm, V3, s);
#pragma unroll
        for (int i = 0; i < 18; i++) GM[i] = Gm[i];
    }
    __syncwarp();
    if (d.fac) {  // factored storage: the factors instead of the dense block
        if (!act) return;
        float *base = d.arena + d.lm_r2[j];
        fac_write_obs(base + 44 + 28 * gl, B, V[0], V[1], rv[0], rv[1]);
        if (gl == 0) {
            fac_write_hdr(base, R, T00, T01, T02, T11, T12, T22, g, L6, rr6);
#pragma unroll
            for (int q = 0; q < 3; q++) {
                d.lm_s[3 * j + q] = sl[q];
                d.lm_D[3 * j + q] = Dl[q];
            }
        }
        return;
    }
    // M = T^T V^T J_p only now: through the damping its 27 values would be live next to the
    // rotations' (the kernel's register peak)
    wy_m(B, make_float4(V[0][0], V[0][1], V[0][2], 0.f), make_float4(V[1][0], V[1][1], V[1][2], 0.f), T00, T01,
         T02, T11, T12, T22);
    // ---- side regions first (R1 rows, TL, q copy, Givens, scaling: the damping values die here,
    // which frees their registers for the emission), assembled in shared memory and written by one
    // bulk store that overlaps the emission; then the emission (write-only stream, Fig. 2c)
    // in the pack layout
    float *blk_side = sside + grp * (int)side_floats(k);
    if (act) {
#pragma unroll
        for (int s = 0; s < 3; s++) {
            const Row9 v = wy_row2(B, VR, GM, k, s, gl);
            float *dst = blk_side + s * 9 * k + 9 * gl;
#pragma unroll
            for (int j = 0; j < 4; j++) dst[2 * j] = v.p[j].x, dst[2 * j + 1] = v.p[j].y;
            dst[8] = v.e;
        }
        float4 *TL = reinterpret_cast<float4 *>(blk_side + side_tl(k));
        // q copy of the small-k preconditioner pass, row a at qc[a] (a >= 3); G = 32 (tile layout):
        // the large pipe reads q from TL
        float *qc = G < 32 ? d.qpk + pack.q0 + 2 * k * grp - 3 : nullptr;
#pragma unroll
        for (int rr = 0; rr < 2; rr++) {
            const int a = 2 * gl + rr;
            if (a >= 3) {
                TL[a] = make_float4(0.f, 0.f, 0.f, rv[rr]);
                if (G < 32) qc[a] = rv[rr];
            }
        }
        if (gl == 0) {
#pragma unroll
            for (int s = 0; s < 3; s++) {
                TL[s] = make_float4(L6[s * 3], L6[s * 3 + 1], L6[s * 3 + 2], rr6[s]);
                TL[2 * k + s] = make_float4(0.f, 0.f, 0.f, rr6[3 + s]);
                if (G < 32) qc[2 * k + s] = rr6[3 + s];
            }
            float *gp = blk_side + side_g(k);
#pragma unroll
            for (int i = 0; i < 12; i++) gp[i] = g[i];
#pragma unroll
            for (int q = 0; q < 3; q++) {
                d.lm_s[3 * j + q] = sl[q];
                d.lm_D[3 * j + q] = Dl[q];
            }
        }
    }
    fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the bulk copy
    __syncwarp();
    if (lane == 0 && RBA_K2_EXP != 4) {  // (EXP 4: measurement experiment, no side-region store)
        bulk_s2g(d.arena + side_off, sside, 4u * (uint32_t)(pack.np * side_floats(k)));
        bulk_commit();
    }
    if (G == 32 && act) {  // 17 <= k <= 32: the 4-row tile layout of the large pipes (g = 0, n_g = k)
        float *R2 = d.arena + pack.base;
        RBA_CHECK(pack.base >= 0 && pack.base + large_r2_floats(k) <= d.arena_n);
        const int T = large_tiles(k);
        for (int t = 0; t < (RBA_K2_EXP == 1 ? 0 : T); t++) {
            float4 *S = reinterpret_cast<float4 *>(R2 + (int64_t)36 * k * t) + gl;
            float v36[36];
            Row9 rw[4];
            if (4 * t + 6 < 2 * k) {  // logical rows 4t+3 .. 4t+6 are plain rows (< 2k)
#pragma unroll
                for (int rr = 0; rr < 4; rr++) rw[rr] = wy_row_plain2(B, VR[4 * t + rr + 3], 4 * t + rr + 3, gl);
            } else {
#pragma unroll
                for (int rr = 0; rr < 4; rr++) {
                    const int a = 4 * t + rr;
                    if (a < 2 * k) {
                        rw[rr] = wy_row2(B, VR, GM, k, a + 3, gl);
                    } else {
#pragma unroll
                        for (int j = 0; j < 4; j++) rw[rr].p[j] = make_float2(0.f, 0.f);
                        rw[rr].e = 0.f;
                    }
                }
            }
#pragma unroll
            for (int rr = 0; rr < 4; rr++) {
#pragma unroll
                for (int j = 0; j < 4; j++) v36[9 * rr + 2 * j] = rw[rr].p[j].x, v36[9 * rr + 2 * j + 1] = rw[rr].p[j].y;
                v36[9 * rr + 8] = rw[rr].e;
            }
#pragma unroll
            for (int c = 0; c < 9; c++)
                S[c * k] = make_float4(v36[4 * c], v36[4 * c + 1], v36[4 * c + 2], v36[4 * c + 3]);
        }
    } else if (G < 32 && act) {
        float2 *A = reinterpret_cast<float2 *>(d.arena + pack.base);
        RBA_CHECK(pack.base >= 0 && pack.base + small_pack_floats(k, pack.np) <= d.arena_n && d.lm_side[pack.lm0] +
                  pack.np * side_floats(k) <= d.arena_n);
        const int npk = pack.np * k, mo = grp * k + gl;
        float2 *Ap = A + mo;
        for (int p = 0; p < (RBA_K2_EXP == 1 ? 0 : k); p++, Ap += 9 * npk) {  // (EXP 1: no R2 emission)
            Row9 r0, r1;
            if (p < k - 2) {  // rows 2p+3, 2p+4 < 2k: no damping rows
                r0 = wy_row_plain2(B, VR[2 * p + 3], 2 * p + 3, gl);
                r1 = wy_row_plain2(B, VR[2 * p + 4], 2 * p + 4, gl);
            } else {
                r0 = wy_row2(B, VR, GM, k, 2 * p + 3, gl);
                r1 = wy_row2(B, VR, GM, k, 2 * p + 4, gl);
            }
            // chunk order of the pack layout: row 0 pairs, row 1 pairs, (row 0, row 1) q = 8
            // (32-bit chunk offsets: one IMAD.WIDE per store address instead of a 64-bit add)
            const unsigned S = (unsigned)npk;
#pragma unroll
            for (int c = 0; c < 4; c++) Ap[c * S] = r0.p[c];
#pragma unroll
            for (int c = 0; c < 4; c++) Ap[(4 + c) * S] = r1.p[c];
            Ap[8 * S] = make_float2(r0.e, r1.e);
        }
    }
    // the side regions must be in global memory before the kernel ends (K4's large pipe, K7 and the
    // re-damp read them): wait for the bulk store's completion, not only for its source reads
    if (lane == 0 && RBA_K2_EXP != 4) bulk_wait_all();
}

// ============================================================================ K2 large (k > 32)
// CTA of NT >= k threads per (landmark, tile range); thread o <-> observation o and camera
// block o.  The O(k) prologue (Jacobians, Householder, WY) is recomputed by every CTA of a
// landmark; the O(k^2) emission is split across CTAs (~1 MB each).
// MULTI (k > KLARGE, "huge"): thread o' owns camera blocks o = o', o' + NT, ...; its two scaled J_p
// rows are recomputed per block in the emission loop instead of being kept from the prologue.
__device__ __forceinline__ void block_jp(const DevProblem &d, int64_t obs0, int o, const double *Xp, BlockWY &B) {
    const int cam = d.obs_cam[obs0 + o];
    double c[CAMPRE], r[2];
    float Jc[18], Jl[6];
    load_pre(d.campre, cam, c);
    const double2 uv = d.obs_uv[obs0 + o];
    cam_model_pre(c, Xp[0], Xp[1], Xp[2], uv.x, uv.y, r, Jc, Jl);
    apply_irls(r, Jc, Jl, d.huber);
#pragma unroll
    for (int q = 0; q < 9; q++) {
        const float s = d.sp[9 * cam + q];
        B.jp[0][q] = Jc[q] * s;
        B.jp[1][q] = Jc[9 + q] * s;
    }
}

// LPC > 1: LPC items (landmarks) per CTA, each on its own NT-thread sub-block synchronized by a
// named barrier (mid k: more resident landmarks per SM than NT-thread CTAs allow, measured below).
template <int NT, bool MULTI, int LPC = 1>
__global__ void __launch_bounds__(NT *LPC, (NT * LPC < 512 ? 512 / (NT * LPC) : 1))
    k_marg_large(DevProblem d, const LargeItem *__restrict__ items, int64_t n_items, int64_t sub_floats, float dmin,
                 float dmax) {
    extern __shared__ float4 smem4[];
    __shared__ float red_all[LPC][2][32 * 4];
    __shared__ float piv_all[LPC][4];
    __shared__ float GM_all[LPC][20];
    const int sub = LPC > 1 ? (int)threadIdx.x / NT : 0;
    const int tid = LPC > 1 ? (int)threadIdx.x % NT : (int)threadIdx.x;
    const int64_t item = (int64_t)blockIdx.x * LPC + sub;
    if (item >= n_items) return;  // (a whole sub-block: its named barrier is its own)
    float *piv = piv_all[sub], *GM = GM_all[sub];
    int nred = 0;  // sub_sum calls (partials buffer parity)
    auto sync = [&]() {
        if (LPC > 1) named_sync(1 + sub, NT);
        else __syncthreads();
    };
    // block_sum over the sub-block (warp shuffles, then one value per warp through shared memory);
    // the partials alternate between two buffers, so one barrier per call suffices (a buffer is
    // rewritten two calls later, after the intervening call's barrier every thread has passed)
    auto sub_sum = [&](float *v, int nv) {
        const int lane = tid & 31, w = tid >> 5;
        float *red = red_all[sub][nred++ & 1];
        for (int i = 0; i < nv; i++) v[i] = warp_sum_f(v[i]);
        if (lane == 0)
            for (int i = 0; i < nv; i++) red[i * 32 + w] = v[i];
        sync();
        for (int i = 0; i < nv; i++) {
            float s_ = 0.f;
            for (int w2 = 0; w2 < NT / 32; w2++) s_ += red[i * 32 + w2];
            v[i] = s_;
        }
    };
    const LargeItem it = items[item];
    const int64_t j = it.lm;
    const int k = d.lm_k[j];
    const bool own = tid < k;
    float4 *VR = smem4 + (LPC > 1 ? sub * (sub_floats / 4) : 0);  // 2k+3
    float *SX = reinterpret_cast<float *>(VR + (2 * k + 3));    // 2k x 3 landmark Jacobian
    float *SR = SX + 6 * k;                                     // 2k residuals
    const int64_t obs0 = d.lm_obs0[j];
    const double *Xp = d.pts + 3 * j;
    BlockWY B;
    float n2[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int q = 0; q < 9; q++) B.jp[0][q] = B.jp[1][q] = 0.f;
    for (int o = tid; o < k; o += NT) {  // !MULTI: NT >= k, at most o == tid
        const int cam = d.obs_cam[obs0 + o];
        double c[CAMPRE], r[2];
        float Jc[18], Jl[6];
        load_pre(d.campre, cam, c);
        const double2 uv = d.obs_uv[obs0 + o];
#if RBA_K2_EXP == 2
        for (int q = 0; q < 18; q++) Jc[q] = (float)c[q] + q;
        for (int q = 0; q < 6; q++) Jl[q] = (float)c[q + 9] + q * o;
        r[0] = uv.x, r[1] = uv.y;
#else
        cam_model_pre(c, Xp[0], Xp[1], Xp[2], uv.x, uv.y, r, Jc, Jl);
#endif
        apply_irls(r, Jc, Jl, d.huber);
        if (!MULTI) {
#pragma unroll
            for (int q = 0; q < 9; q++) {
                const float s = d.sp[9 * cam + q];
                B.jp[0][q] = Jc[q] * s;
                B.jp[1][q] = Jc[9 + q] * s;
            }
        }
#pragma unroll
        for (int q = 0; q < 3; q++) {
            SX[(2 * o) * 3 + q] = Jl[q];
            SX[(2 * o + 1) * 3 + q] = Jl[3 + q];
            n2[q] += Jl[q] * Jl[q] + Jl[3 + q] * Jl[3 + q];
        }
        SR[2 * o] = (float)r[0];
        SR[2 * o + 1] = (float)r[1];
    }
    sub_sum(n2, 3);
    float sl[3], Dl[3];
#pragma unroll
    for (int q = 0; q < 3; q++) {
        sl[q] = 1.f / (1.f + sqrtf(n2[q]));
        Dl[q] = sqrtf(fminf(fmaxf(n2[q] * sl[q] * sl[q], dmin), dmax));
    }
    for (int a = tid; a < 2 * k; a += NT)
#pragma unroll
        for (int q = 0; q < 3; q++) SX[a * 3 + q] *= sl[q];
    sync();
    // Householder, 3 reflectors; V kept in VR rows (all rows 0..2k-1 during the prologue)
    float tau[3];
#pragma unroll
    for (int c = 0; c < 3; c++) {
        float s[4] = {0.f, 0.f, 0.f, 0.f};
        for (int a = c + tid; a < 2 * k; a += NT) {
            const float x = SX[a * 3 + c];
            s[0] += x * x;
            if (c + 1 < 3) s[1] += x * SX[a * 3 + c + 1];
            if (c + 2 < 3) s[2] += x * SX[a * 3 + c + 2];
            s[3] += x * SR[a];
        }
        if (tid == 0) {
            piv[0] = SX[c * 3 + c];
            piv[1] = (c + 1 < 3) ? SX[c * 3 + c + 1] : 0.f;
            piv[2] = (c + 2 < 3) ? SX[c * 3 + c + 2] : 0.f;
            piv[3] = SR[c];
        }
        sub_sum(s, 4);  // (synchronizes)
        const float x0 = piv[0], y1 = piv[1], y2 = piv[2], yr = piv[3];
        const float sig = sqrtf(s[0]);
        const float alpha = x0 >= 0.f ? -sig : sig;
        const float vtv = 2.f * sig * (sig + fabsf(x0));
        const float tc = vtv > 0.f ? 2.f / vtv : 0.f;
        tau[c] = tc;
        const float d1 = s[1] - alpha * y1, d2 = s[2] - alpha * y2, dr = s[3] - alpha * yr;
        for (int a = tid; a < 2 * k; a += NT) {
            float vv = 0.f;
            if (a >= c) vv = (a == c) ? x0 - alpha : SX[a * 3 + c];
            float *vr = reinterpret_cast<float *>(VR + a);
            vr[c] = vv;
            if (c == 0) vr[3] = 0.f;
            if (c + 1 < 3) SX[a * 3 + c + 1] -= tc * vv * d1;
            if (c + 2 < 3) SX[a * 3 + c + 2] -= tc * vv * d2;
            SR[a] -= tc * vv * dr;
            if (a == c) SX[a * 3 + c] = alpha;
            else if (a > c) SX[a * 3 + c] = 0.f;
        }
        sync();
    }
    float p[3] = {0.f, 0.f, 0.f};
    for (int a = tid; a < 2 * k; a += NT) {
        const float4 v = VR[a];
        p[0] += v.x * v.y;
        p[1] += v.x * v.z;
        p[2] += v.y * v.z;
    }
    sub_sum(p, 3);
    const float T00 = tau[0], T11 = tau[1], T22 = tau[2];
    const float T01 = -tau[1] * T00 * p[0];
    const float T02 = -tau[2] * (T00 * p[1] + T01 * p[2]);
    const float T12 = -tau[2] * T11 * p[2];
    // (M = T^T V^T J_p is formed after the damping, below: its 27 values would be live through it)
    // damping (every thread computes the 6 rotations redundantly from smem values)
    float R[9], rr3[3], V3[9];
#pragma unroll
    for (int i = 0; i < 3; i++) {
#pragma unroll
        for (int q = 0; q < 3; q++) R[i * 3 + q] = SX[i * 3 + q];
        rr3[i] = SR[i];
        const float4 v = VR[i];
        V3[i * 3] = v.x, V3[i * 3 + 1] = v.y, V3[i * 3 + 2] = v.z;
    }
    const float sq = sqrtf((float)d.scal[SC_LAM]);
    const float sD[3] = {sq * Dl[0], sq * Dl[1], sq * Dl[2]};
    float L6[18], Gm[18], rr6[6], g[12];
    damp_rotations(R, rr3, sD, L6, Gm, rr6, g);
    sync();  // all reads of VR rows 0..2 done
    // (compile-time indices only: a thread-indexed access would put Gm / L6 / g / sl / Dl in local
    // memory -- round 1 had a 288-byte stack frame here)
    if (tid == 0) {
#pragma unroll
        for (int s6 = 0; s6 < 6; s6++) VR[s6 < 3 ? s6 : 2 * k + s6 - 3] = veff(Gm, V3, s6);
#pragma unroll
        for (int i = 0; i < 18; i++) GM[i] = Gm[i];
    }
    sync();
    if (d.fac) {  // factored storage: the factors instead of the dense block (one item per landmark)
        float *base = d.arena + d.lm_r2[j];
        for (int o = tid; o < k; o += NT) {
            if (MULTI) block_jp(d, obs0, o, Xp, B);
            float v0[3], v1[3];
#pragma unroll
            for (int q = 0; q < 3; q++) {
                v0[q] = 2 * o < 3 ? V3[3 * (2 * o) + q] : reinterpret_cast<const float *>(VR + 2 * o)[q];
                v1[q] = 2 * o + 1 < 3 ? V3[3 * (2 * o + 1) + q] : reinterpret_cast<const float *>(VR + 2 * o + 1)[q];
            }
            fac_write_obs(base + 44 + 28 * o, B, v0, v1, SR[2 * o], SR[2 * o + 1]);
        }
        if (tid == 0) fac_write_hdr(base, R, T00, T01, T02, T11, T12, T22, g, L6, rr6);
        if (tid == 0)
#pragma unroll
            for (int q = 0; q < 3; q++) d.lm_s[3 * j + q] = sl[q], d.lm_D[3 * j + q] = Dl[q];
        return;
    }
    // the landmark and residual columns, the Givens and the scaling first: the damping values die
    // here, freeing their registers for the emission
    if (it.t0 == 0) {
        float *side = d.arena + d.lm_side[j];
        float4 *TL = reinterpret_cast<float4 *>(side + side_tl(k));
        for (int a = 3 + tid; a < 2 * k; a += NT) TL[a] = make_float4(0.f, 0.f, 0.f, SR[a]);
        if (tid == 0) {
#pragma unroll
            for (int s = 0; s < 3; s++) {
                TL[s] = make_float4(L6[s * 3], L6[s * 3 + 1], L6[s * 3 + 2], rr6[s]);
                TL[2 * k + s] = make_float4(0.f, 0.f, 0.f, rr6[3 + s]);
                d.lm_s[3 * j + s] = sl[s];
                d.lm_D[3 * j + s] = Dl[s];
            }
#pragma unroll
            for (int i = 0; i < 12; i++) side[side_g(k) + i] = g[i];
        }
    }
    for (int o = tid; o < k; o += NT) {
        {  // raw V rows 2o, 2o+1 (VR rows 0..2 now hold V_eff of the damped rows)
            if (MULTI) block_jp(d, obs0, o, Xp, B);
            const float4 v0 = o == 0 ? make_float4(V3[0], V3[1], V3[2], 0.f)
                                     : (o == 1 ? make_float4(V3[6], V3[7], V3[8], 0.f) : VR[2 * o]);
            const float4 v1 = o == 0 ? make_float4(V3[3], V3[4], V3[5], 0.f) : VR[2 * o + 1];
            wy_m(B, v0, v1, T00, T01, T02, T11, T12, T22);
        }
        const int g_ = o >> 5, ng = min(32, k - 32 * g_);
        float *R2 = d.arena + d.lm_r2[j];
        for (int t = it.t0; t < (RBA_K2_EXP == 1 ? it.t0 : it.t1); t++) {
            float4 *S = reinterpret_cast<float4 *>(R2 + (int64_t)36 * k * t + 36 * 32 * g_) + (o & 31);
            float v36[36];
            Row9 rw[4];
            if (4 * t + 6 < 2 * k) {  // logical rows 4t+3 .. 4t+6 are plain rows (< 2k)
#pragma unroll
                for (int rr = 0; rr < 4; rr++) rw[rr] = wy_row_plain2(B, VR[4 * t + rr + 3], 4 * t + rr + 3, o);
            } else {
#pragma unroll
                for (int rr = 0; rr < 4; rr++) {
                    const int a = 4 * t + rr;
                    if (a < 2 * k) {
                        rw[rr] = wy_row2(B, VR, GM, k, a + 3, o);
                    } else {
#pragma unroll
                        for (int jj = 0; jj < 4; jj++) rw[rr].p[jj] = make_float2(0.f, 0.f);
                        rw[rr].e = 0.f;
                    }
                }
            }
#pragma unroll
            for (int rr = 0; rr < 4; rr++) {
#pragma unroll
                for (int jj = 0; jj < 4; jj++) v36[9 * rr + 2 * jj] = rw[rr].p[jj].x, v36[9 * rr + 2 * jj + 1] = rw[rr].p[jj].y;
                v36[9 * rr + 8] = rw[rr].e;
            }
#pragma unroll
            for (int c = 0; c < 9; c++)
                S[c * ng] = make_float4(v36[4 * c], v36[4 * c + 1], v36[4 * c + 2], v36[4 * c + 3]);
        }
        if (it.t0 == 0) {
            float *side = d.arena + d.lm_side[j];
#pragma unroll
            for (int s = 0; s < 3; s++) {
                const Row9 v = wy_row2(B, VR, GM, k, s, o);
                float *dst = side + s * 9 * k + 9 * o;
#pragma unroll
                for (int jj = 0; jj < 4; jj++) dst[2 * jj] = v.p[jj].x, dst[2 * jj + 1] = v.p[jj].y;
                dst[8] = v.e;
            }
        }
    }
}

// ============================================================================ K3 re-damping
// Warp per landmark.  Undo the stored rotations (transposed, reverse order, Fig. 3c), drop the
// damping rows, and fold sqrt(lam) D_l in again with freshly computed rotations.
__global__ void __launch_bounds__(256) k_redamp(DevProblem d) {
    const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (j >= d.n_l) return;
    const int k = d.lm_k[j];
    float *side = d.arena + d.lm_side[j];
    float *r2 = d.arena + d.lm_r2[j];
    const int32_t pk = d.lm_pk[j];
    float4 *TL = reinterpret_cast<float4 *>(side + side_tl(k));
    float *gp = side + side_g(k);
    float g[12];
#pragma unroll
    for (int i = 0; i < 12; i++) g[i] = gp[i];
    // landmark + residual columns of the 6 special rows
    float M6[6][4];
#pragma unroll
    for (int s = 0; s < 6; s++) {
        const float4 t = TL[s < 3 ? s : 2 * k + s - 3];
        M6[s][0] = t.x, M6[s][1] = t.y, M6[s][2] = t.z, M6[s][3] = t.w;
    }
#pragma unroll
    for (int m = 5; m >= 0; m--) {
        const int p = damp_p(m), t = damp_t(m);
        const float c = g[2 * m], s = g[2 * m + 1];
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const float a = M6[p][q], b = M6[t][q];
            M6[p][q] = c * a - s * b;
            M6[t][q] = s * a + c * b;
        }
    }
    float R[9], rr3[3];
#pragma unroll
    for (int i = 0; i < 3; i++) {
        R[i * 3] = M6[i][0], R[i * 3 + 1] = M6[i][1], R[i * 3 + 2] = M6[i][2];
        rr3[i] = M6[i][3];
    }
    // exact upper-triangular R1 after undo
    R[3] = 0.f, R[6] = 0.f, R[7] = 0.f;
    const float sq = sqrtf((float)d.scal[SC_LAM]);
    const float sD[3] = {sq * d.lm_D[3 * j], sq * d.lm_D[3 * j + 1], sq * d.lm_D[3 * j + 2]};
    float L6[18], Gm[18], rr6[6], gn[12];
    damp_rotations(R, rr3, sD, L6, Gm, rr6, gn);
    // pose columns: 3 rows of R1 (side) + last 3 rows of R2
    const int W = 9 * k;
    for (int c = lane; c < W; c += 32) {
        const int o = c / 9, q = c - 9 * o;
        float x[6];
        int64_t idx[3];
#pragma unroll
        for (int s = 0; s < 3; s++) {
            x[s] = side[s * W + c];
            idx[s] = r2_index(k, pk, 2 * k - 3 + s, o, q);
            x[3 + s] = r2[idx[s]];
        }
#pragma unroll
        for (int m = 5; m >= 0; m--) {
            const int p = damp_p(m), t = damp_t(m);
            const float cc = g[2 * m], ss = g[2 * m + 1];
            const float a = x[p], b = x[t];
            x[p] = cc * a - ss * b;
            x[t] = ss * a + cc * b;
        }
#pragma unroll
        for (int s = 0; s < 6; s++) {
            const float v = Gm[s * 3] * x[0] + Gm[s * 3 + 1] * x[1] + Gm[s * 3 + 2] * x[2];
            if (s < 3) side[s * W + c] = v;
            else r2[idx[s - 3]] = v;
        }
    }
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < 3; s++) {
            TL[s] = make_float4(L6[s * 3], L6[s * 3 + 1], L6[s * 3 + 2], rr6[s]);
            TL[2 * k + s] = make_float4(0.f, 0.f, 0.f, rr6[3 + s]);
        }
        const int32_t qo = d.lm_q[j];  // small landmarks: the q copy of the damping rows too
        if (qo >= 0)
#pragma unroll
            for (int s = 0; s < 3; s++) d.qpk[qo + 2 * k - 3 + s] = rr6[3 + s];
#pragma unroll
        for (int i = 0; i < 12; i++) gp[i] = gn[i];
    }
}

// ============================================================================ K4 preconditioner + rhs
// P_i = sum_j A_j[:,i]^T A_j[:,i] (45 upper entries) and b~_i = sum_j A_j[:,i]^T q_j (P:348,
// P:647-648): every thread owns one camera block of one landmark, streams its slabs (the same
// coalesced loads as the matvec), accumulates 54 values in registers and adds them to the
// camera's slot once.
__device__ __forceinline__ void acc_rows(float *P, float *b, const float *row, float qa) {
    int idx = 0;
#pragma unroll
    for (int q1 = 0; q1 < 9; q1++) {
        b[q1] += row[q1] * qa;
#pragma unroll
        for (int q2 = q1; q2 < 9; q2++) P[idx++] += row[q1] * row[q2];
    }
}
__device__ __forceinline__ void flush54(float *acc, const float *P, const float *b) {
    // acc: 56-float (16-byte aligned) camera slot: 45 upper-triangle entries of P, 9 of b, 2 pad
    float4 *a4 = reinterpret_cast<float4 *>(acc);
#pragma unroll
    for (int i = 0; i < 11; i++) atomicAdd(a4 + i, make_float4(P[4 * i], P[4 * i + 1], P[4 * i + 2], P[4 * i + 3]));
    atomicAdd(a4 + 11, make_float4(P[44], b[0], b[1], b[2]));
    atomicAdd(a4 + 12, make_float4(b[3], b[4], b[5], b[6]));
    atomicAdd(a4 + 13, make_float4(b[7], b[8], 0.f, 0.f));
}

// per camera (one warp): P_i + lambda D_p^2 -> Cholesky (FP64) -> inverse M^-1 (FP64, 81); b~
// copied out.  The block sits in shared memory; column b of L is formed by lanes b..8 (the same
// left-looking sums, in the same order, as a serial Cholesky), and column c of the inverse by lane c.
constexpr int FIN_WARPS = 8;
__global__ void __launch_bounds__(32 * FIN_WARPS) k_precond_finalize(DevProblem d, double *bad) {
    __shared__ double sP[FIN_WARPS][81];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t i = (int64_t)blockIdx.x * FIN_WARPS + w;
    if (i >= d.n_p) return;  // (warp-uniform)
    double *P = sP[w];
    const double lam = d.scal[SC_LAM];
    const double *acc = d.pd + 54 * i;
    for (int t = lane; t < 45; t += 32) {  // upper-triangle entry t = (a, b), b >= a, row-major
        int a = 0, r = t;
        while (r >= 9 - a) r -= 9 - a, a++;
        const int b = a + r;
        double v = acc[t];
        if (a == b) v += lam * d.Dp264[9 * i + a];
        P[a * 9 + b] = v;
        P[b * 9 + a] = v;
    }
    if (lane < 9) d.bt[9 * i + lane] = acc[45 + lane];  // FP64
    __syncwarp();
    bool ok = true;  // L overwrites the lower triangle of P
    for (int b = 0; b < 9; b++) {
        if (lane == b) {
            double s = P[b * 9 + b];
            for (int m = 0; m < b; m++) s -= P[b * 9 + m] * P[b * 9 + m];
            if (!(s > 0.0)) ok = false, s = 1.0;
            P[b * 9 + b] = sqrt(s);
        }
        __syncwarp();
        if (lane > b && lane < 9) {
            double s = P[lane * 9 + b];
            for (int m = 0; m < b; m++) s -= P[lane * 9 + m] * P[b * 9 + m];
            P[lane * 9 + b] = s / P[b * 9 + b];
        }
        __syncwarp();
    }
    if (__any_sync(0xffffffffu, !ok) && lane == 0) atomicAdd(bad, 1.0);
    if (lane < 9) {  // solve L L^T x = e_lane
        const int col = lane;
        double y[9], x[9];
#pragma unroll
        for (int a = 0; a < 9; a++) {
            double s = (a == col) ? 1.0 : 0.0;
#pragma unroll
            for (int m = 0; m < a; m++) s -= P[a * 9 + m] * y[m];
            y[a] = s / P[a * 9 + a];
        }
#pragma unroll
        for (int a = 8; a >= 0; a--) {
            double s = y[a];
#pragma unroll
            for (int m = a + 1; m < 9; m++) s -= P[m * 9 + a] * x[m];
            x[a] = s / P[a * 9 + a];
        }
#pragma unroll
        for (int a = 0; a < 9; a++) d.Minv[81 * i + a * 9 + col] = x[a];
    }
}

// ============================================================================ K5 matvec
// H~ v = sum_j A_j^T (A_j v_j) (Eq. cg_mult).  A_j is read from HBM exactly once: each
// thread holds the slab of one camera block o (2 or 4 rows x 9) in registers, forms its partial
// of y = A v for the slab rows, the partials of a row are summed over the landmark's blocks
// (warp shuffles for small k, a per-slot named barrier for large k), and out_o += slab^T y
// accumulates in registers; the 9 entries of out_o are added to the camera vector once per
// landmark (per CTA range for large k).

// Sum 4 values over the warp with 6 shuffles (transpose-style butterfly).  Returns the total of
// value r = (lane >> 3) & 3 in every lane; lanes 0, 8, 16, 24 hold rows 0, 1, 2, 3.
__device__ __forceinline__ float warp_sum4(float y0, float y1, float y2, float y3, int lane) {
    const bool hi16 = lane & 16;
    // step 16: keep rows {2,3} if hi16 else {0,1}
    float a = hi16 ? y2 : y0, b = hi16 ? y3 : y1;
    const float sa = hi16 ? y0 : y2, sb = hi16 ? y1 : y3;
    a += __shfl_xor_sync(0xffffffffu, sa, 16);
    b += __shfl_xor_sync(0xffffffffu, sb, 16);
    // step 8: keep one row
    const bool hi8 = lane & 8;
    float c = hi8 ? b : a;
    const float sc = hi8 ? a : b;
    c += __shfl_xor_sync(0xffffffffu, sc, 8);
    c += __shfl_xor_sync(0xffffffffu, c, 4);
    c += __shfl_xor_sync(0xffffffffu, c, 2);
    c += __shfl_xor_sync(0xffffffffu, c, 1);
    return c;  // row = 2 * (lane >> 4 & 1) + (lane >> 3 & 1)
}

__device__ __forceinline__ float group_sum_rt(float v, int G) {
    for (int m = G >> 1; m; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m, G);
    return v;
}
__device__ __forceinline__ int group_of(int k) { return k == 2 ? 2 : (k <= 4 ? 4 : (k <= 8 ? 8 : 16)); }


// ---- small k (<= KSMALL): TMA stages of consecutive packs (+ their camera indices, pack headers
// and a work-unit table); warp <-> unit (pack, <= 4 row pairs), lane <-> (landmark m = lane / G,
// camera block o = lane % G), slabs read from shared memory, row-pair partials reduced with G-lane
// shuffles, the unit's 9 outputs per lane added to the camera vector with float4 reductions.
#ifndef RBA_SP_WARPS
#define RBA_SP_WARPS 12
#endif
constexpr int SP_WARPS = RBA_SP_WARPS;              // consumer warps
constexpr int SP_CAMCAP = 320;                      // camera indices per stage (host guarantees)
constexpr int SP_PACKCAP = 64;                      // packs per stage (host guarantees)
constexpr int SP_UNITCAP = 4 * SP_PACKCAP;          // work units per stage
constexpr int SP_OFF_CAM = SMALL_STAGE_BYTES;
constexpr int SP_OFF_PACK = SP_OFF_CAM + 4 * SP_CAMCAP;
constexpr int SP_OFF_UNIT = SP_OFF_PACK + (int)sizeof(Pack) * SP_PACKCAP;
constexpr int SP_OFF_Q = SP_OFF_UNIT + 2 * SP_UNITCAP;     // K4: the packs' q (SP_QCAP floats)
constexpr int SP_OFF_HDR = SP_OFF_Q + 4 * SP_QCAP;         // stage descriptor (written by the producer)
constexpr int SP_SB = SP_OFF_HDR + 128;
#ifndef RBA_SP_STAGES
#define RBA_SP_STAGES 4  // 4 stages, v read through L1 (measured 2.47 -> 2.43 ms cfg4 matvec vs 3 stages + v in smem)
#endif
#ifndef RBA_SP_VCAP
#define RBA_SP_VCAP 0
#endif
#ifndef RBA_YRED_SHFL
#define RBA_YRED_SHFL 1  // y reduction by xor butterfly (measured 2.54 -> 2.47 ms cfg4 matvec)
#endif
#ifndef RBA_LP_AHEAD
#define RBA_LP_AHEAD 0  // 1: large pipe loads the next tile descriptor and the next landmark's camera / v ahead (measured neutral)
#endif
#ifndef RBA_SP_AGG
#define RBA_SP_AGG 1  // small pipe: add a pack's per-camera partials over its landmarks before the reductions
#endif
#ifndef RBA_STRIPE
#define RBA_STRIPE 0  // 1: large-pipe product, NSLOT > 1: one bulk copy of NSLOT consecutive tiles per stage (measured slower: cfg3 0.266 -> 0.298 ms)
#endif
#ifndef RBA_SP_EXP
#define RBA_SP_EXP 0  // small-pipe experiment: 1 = no staged camera / pack / unit tables
#endif
#ifndef RBA_MARG_LPC64
#define RBA_MARG_LPC64 1  // K2, 33 <= k <= 64: landmarks per CTA (64-thread sub-blocks, named barriers; measured 2: 74, 4: 83 vs 1: 69 us on cfg 3)
#endif
#ifndef RBA_LP_EARLY_RELEASE
// 1: a large-pipe consumer releases its stage right after issuing its shared-memory loads.  Measured
// WRONG on B200: the TMA refill of the stage (async proxy) can overwrite it before those loads have
// read it, although mbarrier.arrive is a release -- a warp's contribution then comes from the wrong
// tile now and then (tools/det_classes.py: k = 150 / 256 tracks, 7-8 of 15 repeated passes differ).
// 0 (default): release once the loaded values are in use.
#define RBA_LP_EARLY_RELEASE 0
#endif
#ifndef RBA_LP_LANES
// large pipes: one producer lane per slot, its tile descriptors loaded a batch ahead, lane 0 arms
// the stage's full barrier with the bytes of all slots (one arrival; an arrival per lane measured
// the same).  0: one producer thread for all slots (cfg3 K4 0.33 -> 0.28 ms, K5 0.263 -> 0.245 ms
// with 1)
#define RBA_LP_LANES 1
#endif
#ifndef RBA_PF_AHEAD
#define RBA_PF_AHEAD 0  // stages prefetched into L2 beyond the shared-memory ring (measured: slower, 0.29 -> 0.52 ms cfg3)
#endif
#ifndef RBA_PIPE_SMEM
#define RBA_PIPE_SMEM 225000  // 3 stages of 4 x 512 x 36-byte tiles (measured +2.3% over 200 KB)
#endif
constexpr int SP_STAGES = RBA_SP_STAGES;
constexpr int SP_VCAP = RBA_SP_VCAP;                // v (9 n_p floats) kept in shared memory if it fits
constexpr size_t SP_SMEM = (size_t)SP_STAGES * SP_SB + 4 * SP_VCAP + 2 * SP_STAGES * sizeof(uint64_t);

// one work unit: NRP row pairs starting at p0 of the lane's (landmark, camera block)
template <int NRP, bool PRECOND>
__device__ __forceinline__ void small_unit(const DevProblem &d, const float2 *A, int npk, int p0, int k, int G,
                                           bool valid, int cam, const float *vo, const float *qs,
                                           float *__restrict__ out12, int64_t slot) {
    // the slab chunks as stored (rba_internal.cuh): c = 0..3 row-0 (q, q+1) pairs, 4..7 row-1 pairs,
    // 8 = (row 0, row 1) at q = 8 -- so both products run on packed FP32 FMAs (FFMA2)
    float2 ch[NRP][9];
#pragma unroll
    for (int u = 0; u < NRP; u++)
#pragma unroll
        for (int c = 0; c < 9; c++) ch[u][c] = valid ? A[((p0 + u) * 9 + c) * npk] : make_float2(0.f, 0.f);
    static_assert(!PRECOND, "K4 accumulates whole landmarks in k_small_pipe");
    {
        float2 v2[4];
#pragma unroll
        for (int c = 0; c < 4; c++) v2[c] = make_float2(vo[2 * c], vo[2 * c + 1]);
        const float v8 = vo[8];
        float y[2 * NRP];
#pragma unroll
        for (int u = 0; u < NRP; u++) {  // y = A v on the unit's 2 rows
            float2 t0 = make_float2(0.f, 0.f), t1 = make_float2(0.f, 0.f);
#pragma unroll
            for (int c = 0; c < 4; c++) {
                t0 = __ffma2_rn(ch[u][c], v2[c], t0);
                t1 = __ffma2_rn(ch[u][4 + c], v2[c], t1);
            }
            const float2 t8 = __fmul2_rn(ch[u][8], make_float2(v8, v8));
            y[2 * u] = (t0.x + t0.y) + t8.x;
            y[2 * u + 1] = (t1.x + t1.y) + t8.y;
        }
        for (int mm = G >> 1; mm; mm >>= 1) {
#pragma unroll
            for (int i = 0; i < 2 * NRP; i++) y[i] += __shfl_xor_sync(0xffffffffu, y[i], mm, G);
        }
        float2 a2[4];
        float a8 = 0.f;
#pragma unroll
        for (int c = 0; c < 4; c++) a2[c] = make_float2(0.f, 0.f);
#pragma unroll
        for (int u = 0; u < NRP; u++) {  // out += A^T y
            const float2 y0 = make_float2(y[2 * u], y[2 * u]), y1 = make_float2(y[2 * u + 1], y[2 * u + 1]);
#pragma unroll
            for (int c = 0; c < 4; c++) a2[c] = __ffma2_rn(ch[u][4 + c], y1, __ffma2_rn(ch[u][c], y0, a2[c]));
            a8 = fmaf(ch[u][8].y, y[2 * u + 1], fmaf(ch[u][8].x, y[2 * u], a8));
        }
        float acc[9];  // (0 on invalid lanes: their slab is 0)
#pragma unroll
        for (int c = 0; c < 4; c++) acc[2 * c] = a2[c].x, acc[2 * c + 1] = a2[c].y;
        acc[8] = a8;
        if (d.det) {
            if (valid) det_store12(d, slot, acc);
            return;
        }
        if (RBA_SP_AGG && G < 32) {
            // the pack's landmarks are sorted by first camera and observe windows of cameras, so
            // usually every landmark of the pack has the same camera in block o: add their partials
            // over m with shuffles and issue one set of reductions per o instead of one per lane
            const int lane = threadIdx.x & 31, o = lane % G;
            const int cam0 = __shfl_sync(0xffffffffu, cam, o);
            if (__all_sync(0xffffffffu, !valid || cam == cam0)) {
                for (int mm = G; mm < 32; mm <<= 1)
#pragma unroll
                    for (int q = 0; q < 9; q++) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], mm);
                if (lane < G && o < k) flush_cam12(wslice(d), cam0, acc);
                return;
            }
        }
        if (valid) flush_cam12(wslice(d), cam, acc);
    }
}

template <bool PRECOND>
__global__ void __launch_bounds__(SP_WARPS * 32 + 32, 1)
    k_small_pipe(DevProblem d, const float *__restrict__ v, float *__restrict__ out12,
                 const PcgState *__restrict__ st, int dbg) {
    if (!PRECOND && st && st->done) return;
    extern __shared__ __align__(128) unsigned char sm[];
    float *sv = reinterpret_cast<float *>(sm + (size_t)SP_STAGES * SP_SB);
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + (size_t)SP_STAGES * SP_SB + 4 * SP_VCAP);
    uint64_t *empty = full + SP_STAGES;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t lo = d.chunk_lo[blockIdx.x], hi = d.chunk_lo[blockIdx.x + 1];
    const bool vsm = !PRECOND && 9 * d.n_p <= SP_VCAP;
    if (vsm)
        for (int64_t i = tid; i < 9 * d.n_p; i += blockDim.x) sv[i] = __ldg(v + i);
    const float *vv = vsm ? sv : v;
    if (tid == 0) {
        for (int s = 0; s < SP_STAGES; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], SP_WARPS);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == SP_WARPS) {  // producer
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            SmallChunk nxc{};
            if (lo < hi) nxc = d.chunks[lo];
            // the consumers wait on the TMA data (ncu: the full-barrier wait is the top stall): keep
            // RBA_PF_AHEAD more stages in flight as L2 prefetches beyond the shared-memory ring
            int64_t pf_base = 0;
            int pf_bytes = 0;
            if (RBA_PF_AHEAD && lo + RBA_PF_AHEAD < hi) pf_base = d.chunks[lo + RBA_PF_AHEAD].base, pf_bytes = d.chunks[lo + RBA_PF_AHEAD].bytes;
            for (int64_t i = lo; i < hi; i++) {
                const int s = (int)((i - lo) % SP_STAGES);
                const uint32_t ph = (uint32_t)(((i - lo) / SP_STAGES) & 1);
                const SmallChunk ch = nxc;
                if (i + 1 < hi) nxc = d.chunks[i + 1];  // prefetch the next stage's descriptor
                RBA_CHECK(ch.bytes <= SMALL_STAGE_BYTES && ch.ncam <= SP_CAMCAP && ch.np <= SP_PACKCAP &&
                          ch.nunit <= SP_UNITCAP && (!PRECOND || ch.nq <= SP_QCAP) && ch.base >= 0 &&
                          ch.base + ch.bytes / 4 <= d.arena_n && ch.cam0 >= 0 && ch.cam0 + ch.ncam <= d.n_obs + 8);
                if (RBA_PF_AHEAD && pf_bytes) {
                    bulk_prefetch_l2(d.arena + pf_base, (uint32_t)pf_bytes);
                    pf_bytes = 0;
                    if (i + 1 + RBA_PF_AHEAD < hi) {
                        const SmallChunk &pc = d.chunks[i + 1 + RBA_PF_AHEAD];
                        pf_base = pc.base, pf_bytes = pc.bytes;
                    }
                }
                mbar_wait(&empty[s], ph ^ 1);
                *reinterpret_cast<SmallChunk *>(sm + (size_t)s * SP_SB + SP_OFF_HDR) = ch;
                mbar_arrive_expect_tx(&full[s], (uint32_t)ch.bytes + (RBA_SP_EXP ? 0u : 4u * (uint32_t)ch.ncam +
                                                    (uint32_t)sizeof(Pack) * (uint32_t)ch.np + 2u * (uint32_t)ch.nunit) +
                                                    (PRECOND ? 4u * (uint32_t)ch.nq : 0u));
                unsigned char *dst = sm + (size_t)s * SP_SB;
                bulk_g2s_stream(dst, d.arena + ch.base, (uint32_t)ch.bytes, &full[s], pol);
                if (!RBA_SP_EXP) {
                    bulk_g2s(dst + SP_OFF_CAM, d.obs_cam + ch.cam0, 4u * (uint32_t)ch.ncam, &full[s]);
                    bulk_g2s(dst + SP_OFF_PACK, d.packs + ch.p0, (uint32_t)sizeof(Pack) * ch.np, &full[s]);
                    bulk_g2s(dst + SP_OFF_UNIT, d.units + ch.unit0, 2u * (uint32_t)ch.nunit, &full[s]);
                }
                if (PRECOND) bulk_g2s_stream(dst + SP_OFF_Q, d.qpk + ch.q0, 4u * (uint32_t)ch.nq, &full[s], pol);
            }
        }
        return;
    }
    // Work items (K5: the units of a stage; K4: its packs) are dealt to the consumer warps round
    // robin over the concatenation of all stages (item n of the sequence -> warp n mod SP_WARPS), so
    // every warp has work although a stage holds only a few items (1-8 for k >= 8); warps run up
    // to SP_STAGES stages apart.
    int base = 0;  // items of the previous stages, mod SP_WARPS
    for (int64_t i = lo; i < hi; i++) {
        const int s = (int)((i - lo) % SP_STAGES);
        const uint32_t ph = (uint32_t)(((i - lo) / SP_STAGES) & 1);
        const unsigned char *stg = sm + (size_t)s * SP_SB;
        mbar_wait(&full[s], ph);
        const SmallChunk ch = *reinterpret_cast<const SmallChunk *>(stg + SP_OFF_HDR);
#if RBA_SP_EXP  // experiment: the stage tables read from global (L1 / L2) instead of staged copies
        const int *scam = d.obs_cam + ch.cam0;
        const Pack *spk = d.packs + ch.p0;
        const uint16_t *sun = d.units + ch.unit0;
#else
        const int *scam = reinterpret_cast<const int *>(stg + SP_OFF_CAM);
        const Pack *spk = reinterpret_cast<const Pack *>(stg + SP_OFF_PACK);
        const uint16_t *sun = reinterpret_cast<const uint16_t *>(stg + SP_OFF_UNIT);
#endif
        const int nitems = dbg == 1 ? 0 : (PRECOND ? ch.np : ch.nreal);
        int first = warp - base;
        if (first < 0) first += SP_WARPS;
        base = (base + nitems) % SP_WARPS;
        for (int wi = first; wi < nitems; wi += SP_WARPS) {
            const int code = PRECOND ? wi : sun[wi];
            const Pack pack = spk[code & 255];
            const int p0 = PRECOND ? 0 : 4 * (code >> 8);
            const int k = pack.k;
            const int G = group_of(k);
            const int m = lane / G, o = lane % G;
            const bool valid = m < pack.np && o < k;
            const int npk = pack.np * k, mo = m * k + o;
            const float2 *A = reinterpret_cast<const float2 *>(stg + 4 * (pack.base - ch.base)) + mo;
            RBA_CHECK(pack.base >= ch.base && 4 * (pack.base - ch.base + small_pack_floats(k, pack.np)) <= ch.bytes);
            RBA_CHECK(!valid || (pack.obs0 - ch.cam0 + mo >= 0 && pack.obs0 - ch.cam0 + mo < ch.ncam));
            RBA_CHECK(!PRECOND || !valid || (pack.q0 - ch.q0 + 2 * k * m >= 0 && pack.q0 - ch.q0 + 2 * k * (m + 1) <= ch.nq));
            const int cam = valid ? scam[pack.obs0 - ch.cam0 + mo] : 0;
            float vo[9];
#pragma unroll
            for (int q = 0; q < 9; q++) vo[q] = (valid && !PRECOND) ? vv[9 * cam + q] : 0.f;
            // K4: the landmark's q from the staged copy, row a at qs[a - 3]
            const float *qs = reinterpret_cast<const float *>(stg + SP_OFF_Q) + (pack.q0 - ch.q0) + 2 * k * m;
            if (PRECOND) {  // a warp takes all row pairs of a pack: one flush per (landmark, camera)
                float P[45], b[9];
#pragma unroll
                for (int q = 0; q < 45; q++) P[q] = 0.f;
#pragma unroll
                for (int q = 0; q < 9; q++) b[q] = 0.f;
                for (int pp = 0; pp < (valid ? k : 0); pp++) {
                    float sl[18];
#pragma unroll
                    for (int c = 0; c < 9; c++) {
                        const float2 x = A[(pp * 9 + c) * npk];
                        sl[slab_elem(c, 0)] = x.x, sl[slab_elem(c, 1)] = x.y;
                    }
                    acc_rows(P, b, sl, qs[2 * pp]);
                    acc_rows(P, b, sl + 9, qs[2 * pp + 1]);
                }
                if (d.det) {
                    if (valid) det_store54(d, d.slot4[pack.obs0 + mo], P, b);
                    continue;
                }
                if (RBA_SP_AGG && G < 32) {  // same camera across the pack's landmarks: see small_unit
                    const int cam0 = __shfl_sync(0xffffffffu, cam, o);
                    if (__all_sync(0xffffffffu, !valid || cam == cam0)) {
                        for (int mm = G; mm < 32; mm <<= 1) {
#pragma unroll
                            for (int q = 0; q < 45; q++) P[q] += __shfl_xor_sync(0xffffffffu, P[q], mm);
#pragma unroll
                            for (int q = 0; q < 9; q++) b[q] += __shfl_xor_sync(0xffffffffu, b[q], mm);
                        }
                        if (lane < G && o < k) flush54(pslice(d) + PACC_STRIDE * (int64_t)cam0, P, b);
                        continue;
                    }
                }
                if (valid) flush54(pslice(d) + PACC_STRIDE * (int64_t)cam, P, b);
                continue;
            }
            if constexpr (!PRECOND) {
                // deterministic mode: the unit's own slot (part = its row-pair group)
                const int64_t slot = (d.det && valid) ? (int64_t)d.slot5[pack.obs0 + mo] + (code >> 8) : 0;
                switch (min(4, k - p0)) {
                    case 1: small_unit<1, false>(d, A, npk, p0, k, G, valid, cam, vo, qs, out12, slot); break;
                    case 2: small_unit<2, false>(d, A, npk, p0, k, G, valid, cam, vo, qs, out12, slot); break;
                    case 3: small_unit<3, false>(d, A, npk, p0, k, G, valid, cam, vo, qs, out12, slot); break;
                    default: small_unit<4, false>(d, A, npk, p0, k, G, valid, cam, vo, qs, out12, slot); break;
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
}

template <int NS, int NSLOT>
struct PipeCfg {
    static constexpr int NC = NS * NSLOT;           // consumer threads
    static constexpr int TB = 144 * NS;             // bytes of the largest tile (k <= NS)
    static constexpr int SB = TB * NSLOT;           // stage bytes
    static constexpr int STAGES = RBA_PIPE_SMEM / SB > 8 ? 8 : RBA_PIPE_SMEM / SB;
    // K4 only: the 4 TL rows (residual entries q) of each staged tile, 64 B per slot and stage
    static constexpr size_t QOFF = (size_t)STAGES * SB;
    static constexpr size_t SMEM = QOFF + (size_t)STAGES * NSLOT * 64 + 2 * STAGES * sizeof(uint64_t);
};

// Consumer slot s of NSLOT processes tiles lo + i*NSLOT + s; NS threads per slot <-> camera blocks.
// PRECOND = false: matvec (K5); true: block-Jacobi blocks + rhs (K4).
template <int NS, int NSLOT, bool PRECOND>
__global__ void __launch_bounds__(NS *NSLOT + 32, 1)
    k_large_pipe(DevProblem d, const TileRef *__restrict__ tiles, const int64_t *__restrict__ cta_lo,
                 const float *__restrict__ v, float *__restrict__ out, const PcgState *__restrict__ st,
                 const int32_t *__restrict__ run_part) {
    using C = PipeCfg<NS, NSLOT>;
    if (!PRECOND && st && st->done) return;
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + C::QOFF + (size_t)C::STAGES * NSLOT * 64);
    uint64_t *empty = full + C::STAGES;
    __shared__ __align__(16) float red[2][C::NC / 32][4];
    const int tid = threadIdx.x;
    const int64_t lo = cta_lo[blockIdx.x], hi = cta_lo[blockIdx.x + 1];
    // Run mode: slot s streams the contiguous tile run [lo + s nst, lo + (s + 1) nst): consecutive
    // tiles of a landmark stay in one slot, so its camera / v / flush work is paid once per
    // landmark; a stage is NSLOT separate bulk copies of one tile each.
    // Stripe mode (the product with NSLOT > 1, not deterministic): stage i = the NSLOT consecutive
    // tiles lo + i NSLOT .. (one contiguous range of the arena: ONE bulk copy of NSLOT tiles, so the
    // copies are as large as the big-k classes'), slot s takes tile lo + i NSLOT + s; a landmark's
    // partial sums are flushed once per slot that saw it.
    const bool stripe = RBA_STRIPE && !PRECOND && NSLOT > 1 && !d.det;
    constexpr bool LANES = RBA_LP_LANES != 0;
    const int64_t nst = (hi - lo + NSLOT - 1) / NSLOT;
    if (tid == 0) {
        for (int s = 0; s < C::STAGES; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], C::NC / 32);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (tid >= C::NC) {  // ---------------- producer warp: one elected lane streams the tiles
        if (tid == C::NC && stripe) {
            const uint64_t pol = policy_evict_first();
            int64_t n_off = 0, n_bytes = 0;  // the next stage's source range (loaded one ahead)
            auto range = [&](int64_t i, int64_t &off, int64_t &bytes) {
                const int64_t first = lo + i * NSLOT, last = min(hi, first + NSLOT) - 1;
                const TileRef a = tiles[first], z = tiles[last];
                off = a.off;
                bytes = 4 * (z.off - a.off + 36 * (int64_t)z.k);
            };
            if (nst > 0) range(0, n_off, n_bytes);
            for (int64_t i = 0; i < nst; i++) {
                const int s = (int)(i % C::STAGES);
                const uint32_t ph = (uint32_t)((i / C::STAGES) & 1);
                const int64_t c_off = n_off, c_bytes = n_bytes;
                if (i + 1 < nst) range(i + 1, n_off, n_bytes);
                mbar_wait(&empty[s], ph ^ 1);
                RBA_CHECK(c_bytes > 0 && c_bytes <= C::SB && c_off >= 0 && c_off + c_bytes / 4 <= d.arena_n);
                mbar_arrive_expect_tx(&full[s], (uint32_t)c_bytes);
                bulk_g2s_stream(sm + (size_t)s * C::SB, d.arena + c_off, (uint32_t)c_bytes, &full[s], pol);
            }
        } else if (LANES && !stripe && tid < C::NC + NSLOT) {
            // run mode: producer lane sl streams slot sl's tile run [r0, r1) (one arrival per lane
            // on the full barrier); its tile descriptors (arena offset, k, TL offset) are loaded in
            // batches of PD, one batch ahead, so no copy waits on a descriptor load
            const int sl = tid - C::NC;
            const uint64_t pol = policy_evict_first();
            const int64_t r0 = lo + sl * nst, r1 = min(hi, r0 + nst);
            constexpr int PD = 4;
            int64_t coff[PD], ctl[PD], noff[PD], ntl[PD];
            int ck[PD], nk[PD];
            auto load = [&](int64_t i0) {
#pragma unroll
                for (int u = 0; u < PD; u++) {
                    const int64_t ti = r0 + i0 + u;
                    nk[u] = 0, noff[u] = 0, ntl[u] = 0;
                    if (ti < r1) {
                        const TileRef tr = tiles[ti];
                        nk[u] = tr.k, noff[u] = tr.off, ntl[u] = PRECOND ? tr.tl : 0;
                    }
                }
            };
            load(0);
            for (int64_t i0 = 0; i0 < nst; i0 += PD) {
#pragma unroll
                for (int u = 0; u < PD; u++) coff[u] = noff[u], ctl[u] = ntl[u], ck[u] = nk[u];
                load(i0 + PD);
#pragma unroll
                for (int u = 0; u < PD; u++) {
                    const int64_t i = i0 + u;
                    if (i >= nst) break;
                    const int s = (int)(i % C::STAGES);
                    const uint32_t ph = (uint32_t)((i / C::STAGES) & 1);
                    mbar_wait(&empty[s], ph ^ 1);
                    RBA_CHECK(ck[u] <= NS && coff[u] >= 0 && coff[u] + 36 * ck[u] <= d.arena_n);
                    // one arrival per stage: lane 0 announces the bytes of all slots (a copy that
                    // lands first only drives the transaction count negative meanwhile)
                    uint32_t nb = ck[u] ? 144u * (uint32_t)ck[u] + (PRECOND ? 64u : 0u) : 0u;
#pragma unroll
                    for (int m = 1; m < NSLOT; m <<= 1) nb += __shfl_xor_sync((1u << NSLOT) - 1u, nb, m);
                    if (sl == 0) mbar_arrive_expect_tx(&full[s], nb);
                    if (ck[u]) {
                        bulk_g2s_stream(sm + (size_t)s * C::SB + (size_t)sl * C::TB, d.arena + coff[u],
                                        144u * (uint32_t)ck[u], &full[s], pol);
                        if (PRECOND) bulk_g2s(sm + C::QOFF + ((size_t)s * NSLOT + sl) * 64, d.arena + ctl[u], 64u, &full[s]);
                    }
                }
            }
        } else if (!LANES && tid == C::NC) {
            const uint64_t pol = policy_evict_first();
            // descriptors (arena offset, k) of the next stage are loaded one stage ahead, as
            // independent loads, so their latency overlaps the wait and the current copies
            int64_t noff[NSLOT], ntl[NSLOT];
            int nk[NSLOT];
            auto tl_off = [&](int64_t ti) -> int64_t {  // float offset of TL rows 3 + 4t .. 6 + 4t
                return (PRECOND && ti < hi) ? tiles[ti].tl : 0;
            };
            // tiles of stage i + RBA_PF_AHEAD (per slot), prefetched into L2 beyond the ring
            int64_t poff[NSLOT];
            int pk[NSLOT];
#pragma unroll
            for (int sl = 0; sl < NSLOT; sl++) {
                const int64_t ti = lo + sl * nst;
                nk[sl] = ti < hi ? tiles[ti].k : 0;
                noff[sl] = ti < hi ? tiles[ti].off : 0;
                ntl[sl] = tl_off(ti);
                const int64_t tp = ti + RBA_PF_AHEAD;
                pk[sl] = (RBA_PF_AHEAD && RBA_PF_AHEAD < nst && tp < hi) ? tiles[tp].k : 0;
                poff[sl] = pk[sl] ? tiles[tp].off : 0;
            }
            for (int64_t i = 0; i < nst; i++) {
                const int s = (int)(i % C::STAGES);
                const uint32_t ph = (uint32_t)((i / C::STAGES) & 1);
                if (RBA_PF_AHEAD) {
#pragma unroll
                    for (int sl = 0; sl < NSLOT; sl++) {
                        if (pk[sl]) bulk_prefetch_l2(d.arena + poff[sl], 144u * (uint32_t)pk[sl]);
                        const int64_t tp = lo + sl * nst + i + 1 + RBA_PF_AHEAD;
                        pk[sl] = (i + 1 + RBA_PF_AHEAD < nst && tp < hi) ? tiles[tp].k : 0;
                        poff[sl] = pk[sl] ? tiles[tp].off : 0;
                    }
                }
                int64_t coff[NSLOT], ctl[NSLOT];
                int ck[NSLOT];
                uint32_t total = 0;
#pragma unroll
                for (int sl = 0; sl < NSLOT; sl++) {
                    coff[sl] = noff[sl];
                    ctl[sl] = ntl[sl];
                    ck[sl] = nk[sl];
                    total += 144u * (uint32_t)ck[sl] + ((PRECOND && ck[sl]) ? 64u : 0u);
                    const int64_t tn = i + 1 < nst ? lo + sl * nst + (i + 1) : hi;
                    nk[sl] = tn < hi ? tiles[tn].k : 0;
                    noff[sl] = tn < hi ? tiles[tn].off : 0;
                    ntl[sl] = tl_off(tn);
                }
                mbar_wait(&empty[s], ph ^ 1);
#pragma unroll
                for (int sl = 0; sl < NSLOT; sl++) RBA_CHECK(ck[sl] <= NS && coff[sl] >= 0 && coff[sl] + 36 * ck[sl] <= d.arena_n);
                mbar_arrive_expect_tx(&full[s], total);
#pragma unroll
                for (int sl = 0; sl < NSLOT; sl++)
                    if (ck[sl])
                        bulk_g2s_stream(sm + (size_t)s * C::SB + (size_t)sl * C::TB, d.arena + coff[sl], 144u * (uint32_t)ck[sl],
                                 &full[s], pol);
                if (PRECOND)
#pragma unroll
                    for (int sl = 0; sl < NSLOT; sl++)
                        if (ck[sl]) bulk_g2s(sm + C::QOFF + ((size_t)s * NSLOT + sl) * 64, d.arena + ctl[sl], 64u, &full[s]);
            }
        }
        return;
    }
    // ---------------- consumers
    const int slot = tid / NS, o = tid % NS, lane = tid & 31, warp = tid >> 5;
    constexpr int NWS = NS / 32;
    int cur = -1, k = 0, cam = 0, ng = 1, g = 0, cur_obs0 = 0;
    bool valid = false;
    float vo[9], acc[9], P[PRECOND ? 45 : 1], b[PRECOND ? 9 : 1];
#pragma unroll
    for (int q = 0; q < 9; q++) vo[q] = 0.f, acc[q] = 0.f;
    // deterministic mode: the part index of this consumer run's first landmark (later ones: 0)
    int part = (d.det && run_part) ? run_part[(int)blockIdx.x * NSLOT + slot] : 0;
    auto flush = [&]() {
        if (cur < 0 || !valid) return;
        if (d.det) {
            if (PRECOND) det_store54(d, (int64_t)d.slot4[cur_obs0 + o] + part, P, b);
            else det_store12(d, (int64_t)d.slot5[cur_obs0 + o] + part, acc);
        } else if (PRECOND) {
            flush54(pslice(d) + PACC_STRIDE * (int64_t)cam, P, b);
        } else {
            flush_cam12(wslice(d), cam, acc);
        }
    };
    int buf = 0;
    // The next stage's tile descriptor and the next landmark's camera / v block are loaded ahead
    // (RBA_LP_AHEAD): at a landmark change the slot would otherwise wait on two dependent L2 round
    // trips (camera index, then v) -- for k <= 64 that stall was longer than the landmark's tiles.
    constexpr bool LPA = RBA_LP_AHEAD && NS <= 128;  // (NS >= 256: landmark changes are rare, registers tight)
    auto tile_of = [&](int64_t i) -> int64_t { return stripe ? lo + i * NSLOT + slot : lo + slot * nst + i; };
    TileRef tr_n{-1, 0, 0, 0, 0, 0};
    if (nst > 0 && tile_of(0) < hi) tr_n = tiles[tile_of(0)];
    int pf_state = 0, pf_cam = 0;  // 0 none, 1 camera index loaded, 2 camera and v loaded
    int64_t pf_obs0 = -1;
    float pf_v[9];
#pragma unroll
    for (int q = 0; q < 9; q++) pf_v[q] = 0.f;
    for (int64_t i = 0; i < nst; i++) {
        const int s = (int)(i % C::STAGES);
        const uint32_t ph = (uint32_t)((i / C::STAGES) & 1);
        const int64_t ti = tile_of(i);
        const bool have = ti < hi;  // uniform over the slot
        TileRef tr = have ? tr_n : TileRef{-1, 0, 0, 0, 0, 0};
        if (LPA && i + 1 < nst && tile_of(i + 1) < hi) tr_n = tiles[tile_of(i + 1)];
        else if (!LPA && have) tr = tiles[ti];
        int64_t stage_off = 0;  // stripe mode: arena offset of the stage's first tile
        if (stripe) stage_off = tiles[lo + i * NSLOT].off;
        if (have) {
            if (tr.lm != cur) {
                flush();
                if (cur >= 0) part = 0;  // a landmark that starts in this run
                cur = tr.lm;
                cur_obs0 = tr.obs0;
                k = tr.k;
                valid = o < k;
                g = o >> 5;
                ng = valid ? min(32, k - 32 * g) : 1;
                if (LPA && pf_state > 0 && pf_obs0 == tr.obs0) {
                    cam = pf_cam;
#pragma unroll
                    for (int q = 0; q < 9; q++)
                        vo[q] = (PRECOND || !valid) ? 0.f : (pf_state == 2 ? pf_v[q] : __ldg(v + 9 * cam + q));
                } else {
                    if (valid) cam = __ldg(d.obs_cam + tr.obs0 + o);  // (first observation carried by the tile)
#pragma unroll
                    for (int q = 0; q < 9; q++) vo[q] = (PRECOND || !valid) ? 0.f : __ldg(v + 9 * cam + q);
                }
                // the following landmark of the class starts at observation obs0 + k
                pf_state = 0;
                pf_obs0 = tr.obs0 + k;
                if (LPA && pf_obs0 + o < d.n_obs) pf_cam = __ldg(d.obs_cam + pf_obs0 + o), pf_state = 1;
                if (PRECOND) {
#pragma unroll
                    for (int q = 0; q < 45; q++) P[q] = 0.f;
#pragma unroll
                    for (int q = 0; q < 9; q++) b[q] = 0.f;
                } else {
#pragma unroll
                    for (int q = 0; q < 9; q++) acc[q] = 0.f;
                }
            } else if (LPA && !PRECOND && pf_state == 1) {  // second step of the prefetch: v of that camera
#pragma unroll
                for (int q = 0; q < 9; q++) pf_v[q] = __ldg(v + 9 * pf_cam + q);
                pf_state = 2;
            }
        }
        mbar_wait(&full[s], ph);
        if (PRECOND && NS == 512) {  // 544 threads: <= 120 registers; one row at a time (no spills)
            if (have && valid) {
                const float4 *Q = reinterpret_cast<const float4 *>(sm + C::QOFF + ((size_t)s * NSLOT + slot) * 64);
                const float *S1 = reinterpret_cast<const float *>(
                    reinterpret_cast<const float4 *>(sm + (size_t)s * C::SB + (size_t)slot * C::TB) + 288 * g + (o & 31));
#pragma unroll
                for (int r = 0; r < 4; r++) {
                    float row[9];
#pragma unroll
                    for (int q = 0; q < 9; q++) {
                        const int f = 9 * r + q;  // float f of the thread's 36: float4 f / 4, lane f % 4
                        row[q] = S1[4 * (f >> 2) * ng + (f & 3)];
                    }
                    const float qa = Q[r].w;
                    if (4 * tr.t + r < 2 * k) acc_rows(P, b, row, qa);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            continue;
        }
        float sl[36], qv[4] = {0.f, 0.f, 0.f, 0.f};
        if (PRECOND && have && valid) {
            const float4 *Q = reinterpret_cast<const float4 *>(sm + C::QOFF + ((size_t)s * NSLOT + slot) * 64);
#pragma unroll
            for (int r = 0; r < 4; r++) qv[r] = Q[r].w;
        }
        if (have && valid) {
            const float4 *S4 =
                reinterpret_cast<const float4 *>(sm + (size_t)s * C::SB +
                                                 (stripe ? (size_t)4 * (tr.off - stage_off) : (size_t)slot * C::TB)) +
                288 * g + (o & 31);
#pragma unroll
            for (int c = 0; c < 9; c++) {
                const float4 x = S4[c * ng];
                sl[4 * c] = x.x, sl[4 * c + 1] = x.y, sl[4 * c + 2] = x.z, sl[4 * c + 3] = x.w;
            }
        } else {
#pragma unroll
            for (int c = 0; c < 36; c++) sl[c] = 0.f;
        }
        // the stage is released once the values read from it are in use (RBA_LP_EARLY_RELEASE = 1:
        // right after the loads were issued)
        auto release = [&]() {
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        };
        if (RBA_LP_EARLY_RELEASE || !have) release();
        if (!have) continue;
        if (PRECOND) {
            if (valid) {
#pragma unroll
                for (int r = 0; r < 4; r++) {
                    const int a = 4 * tr.t + r;
                    if (a < 2 * k) acc_rows(P, b, sl + 9 * r, qv[r]);
                }
            }
            if (!RBA_LP_EARLY_RELEASE) release();
        } else {
            float y[4];
#pragma unroll
            for (int r = 0; r < 4; r++) {
                float sacc = 0.f;
#pragma unroll
                for (int q = 0; q < 9; q++) sacc += sl[9 * r + q] * vo[q];
                y[r] = sacc;
            }
            if (!RBA_LP_EARLY_RELEASE) release();
            const float yr = warp_sum4(y[0], y[1], y[2], y[3], lane);
            if ((lane & 7) == 0) red[buf][warp][lane >> 3] = yr;
            if (NS == 32) {
                __syncwarp();
#pragma unroll
                for (int r = 0; r < 4; r++) y[r] = red[buf][warp][r];
            } else {
                named_sync(1 + slot, NS);
#if RBA_YRED_SHFL
                // lane l reads warp (l mod NWS)'s 4 partials (one LDS.128), then an xor butterfly over
                // NWS lanes leaves the totals in every lane (instead of NWS LDS.128 + 4 NWS FADD)
                float4 pv = *reinterpret_cast<const float4 *>(&red[buf][slot * NWS + (lane & (NWS - 1))][0]);
#pragma unroll
                for (int m = NWS / 2; m; m >>= 1) {
                    pv.x += __shfl_xor_sync(0xffffffffu, pv.x, m);
                    pv.y += __shfl_xor_sync(0xffffffffu, pv.y, m);
                    pv.z += __shfl_xor_sync(0xffffffffu, pv.z, m);
                    pv.w += __shfl_xor_sync(0xffffffffu, pv.w, m);
                }
                y[0] = pv.x, y[1] = pv.y, y[2] = pv.z, y[3] = pv.w;
#else
#pragma unroll
                for (int r = 0; r < 4; r++) {
                    float sacc = 0.f;
#pragma unroll
                    for (int w = 0; w < NWS; w++) sacc += red[buf][slot * NWS + w][r];
                    y[r] = sacc;
                }
#endif
            }
#pragma unroll
            for (int q = 0; q < 9; q++)
                acc[q] += sl[q] * y[0] + sl[9 + q] * y[1] + sl[18 + q] * y[2] + sl[27 + q] * y[3];
            buf ^= 1;
        }
    }
    flush();
}

// ---- huge k (> KLARGE): a 4 x 9k tile no longer fits on chip twice (k = 1748: 252 KB), so the
// product takes two passes over the same 4-row tiles: y = A v per tile (CTA-wide reduction), then
// out_o += sum_t slab_{o,t}^T y_t with thread <-> camera block.  The preconditioner needs no y and
// uses the second pass alone.  (2x the algorithmic bytes on these landmarks.)
__device__ __forceinline__ void huge_slab(const float *__restrict__ R2, int k, int t, int o, float *sl) {
    const int g = o >> 5, ng = min(32, k - 32 * g);
    const float4 *S4 = reinterpret_cast<const float4 *>(R2 + (int64_t)36 * k * t + 36 * 32 * g) + (o & 31);
#pragma unroll
    for (int c = 0; c < 9; c++) {
        const float4 x = __ldcs(S4 + c * ng);
        sl[4 * c] = x.x, sl[4 * c + 1] = x.y, sl[4 * c + 2] = x.z, sl[4 * c + 3] = x.w;
    }
}

__global__ void __launch_bounds__(HUGE_NT) k_huge_y(DevProblem d, const float *__restrict__ v,
                                                    const PcgState *__restrict__ st) {
    if (st && st->done) return;
    __shared__ float red[32 * 4];
    const HugeItem it = d.huge_y[blockIdx.x];
    const int64_t j = it.lm;
    const int k = d.lm_k[j], t = it.t0;
    const float *R2 = d.arena + d.lm_r2[j];
    const int32_t *oc = d.obs_cam + d.lm_obs0[j];
    float y[4] = {0.f, 0.f, 0.f, 0.f};
    for (int o = threadIdx.x; o < k; o += HUGE_NT) {
        float sl[36];
        huge_slab(R2, k, t, o, sl);
        const float *vv = v + 9 * (int64_t)oc[o];
#pragma unroll
        for (int q = 0; q < 9; q++) {
            const float x = __ldg(vv + q);
#pragma unroll
            for (int r = 0; r < 4; r++) y[r] += sl[9 * r + q] * x;
        }
    }
    block_sum<4>(y, red);
    if (threadIdx.x == 0) reinterpret_cast<float4 *>(d.ybuf + it.yoff)[t] = make_float4(y[0], y[1], y[2], y[3]);
}

// Fused variant of the two passes: CTA per (landmark, tile range), thread <-> camera blocks
// o = tid + m HUGE_FNT (m < HUGE_NB); per tile the y partials from the tile's slabs (HBM), a CTA
// reduction, then out_o += slab^T y from a second read of the same tile, which L2 still holds (a
// tile is <= 144 KMAX = 442 KB), so HBM sees each tile once.
#ifndef RBA_HUGE_PF_DEFAULT
#define RBA_HUGE_PF_DEFAULT 0  // 0: two tiles ahead (round-2 measured default)
#endif
constexpr int HUGE_FNT = 512, HUGE_NB = (KMAX + HUGE_FNT - 1) / HUGE_FNT;
constexpr int HUGE_REG_K = 2 * HUGE_FNT;  // k <= this: the tile stays in registers (NB = 2)
// Persistent: CTA b takes items b, b + grid, ...; thread 0 keeps the tile two ahead in the CTA's
// tile sequence (across item boundaries) prefetching into L2.  REG (k <= HUGE_REG_K): the thread's
// two slabs stay in registers through the CTA reduction, so the second half of the product reads
// no memory; otherwise they are read again from L2.
template <int NB, bool REG>
__global__ void __launch_bounds__(HUGE_FNT, 1) k_huge_fused(DevProblem d, const HugeItem *__restrict__ items,
                                                            int64_t n_items, const float *__restrict__ v,
                                                            const PcgState *__restrict__ st, int pf_bytes) {
    if (st && st->done) return;
    // y partials of the 16 warps, double-buffered so one barrier per tile suffices (a warp can only
    // rewrite a buffer after the next tile's barrier, i.e. after every warp has read it)
    __shared__ __align__(16) float red[2][HUGE_FNT / 32][4];
    // the item's v blocks of this thread's camera blocks, [m][q][tid] (conflict-free), loaded once
    // per item instead of once per tile
    extern __shared__ float sv_dyn[];  // [NB][9][HUGE_FNT] (dynamic: NB = 6 exceeds 48 KB)
    float(*sv)[9][HUGE_FNT] = reinterpret_cast<float(*)[9][HUGE_FNT]>(sv_dyn);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int nt = 0;  // tiles processed (reduction buffer parity)
    // prefetch cursor (thread 0): item pi, tile pt of it
    int64_t pi = blockIdx.x;
    int pt = 0, pk = 0, pt1 = 0;
    const float *pr = nullptr;
    auto pf_load = [&]() {
        if (pi < n_items) {
            const HugeItem q = items[pi];
            pk = d.lm_k[q.lm], pr = d.arena + d.lm_r2[q.lm], pt = q.t0, pt1 = q.t1;
        }
    };
    auto pf_next = [&]() {  // prefetch the cursor's tile, then advance it
        if (pi >= n_items) return;
        bulk_prefetch_l2(pr + (int64_t)36 * pk * pt, 144u * (uint32_t)pk);
        if (++pt >= pt1) {
            pi += gridDim.x;
            pf_load();
        }
    };
    if (tid == 0) {  // keep ~pf_bytes of this CTA's tiles on their way into L2 (at least 2 tiles)
        pf_load();
        const int ahead = pk > 0 ? max(2, min(16, pf_bytes / (144 * pk))) : 2;
        for (int a = 0; a < ahead; a++) pf_next();
    }
    for (int64_t ii = blockIdx.x; ii < n_items; ii += gridDim.x) {
        const HugeItem it = items[ii];
        const int64_t j = it.lm;
        const int k = d.lm_k[j];
        const float *R2 = d.arena + d.lm_r2[j];
        const int32_t *oc = d.obs_cam + d.lm_obs0[j];
        float acc[NB][9];
#pragma unroll
        for (int m = 0; m < NB; m++) {
#pragma unroll
            for (int q = 0; q < 9; q++) acc[m][q] = 0.f;
            const int o = tid + m * HUGE_FNT;
            if (o < k) {
                const float *vv = v + 9 * (int64_t)oc[o];
#pragma unroll
                for (int q = 0; q < 9; q++) sv[m][q][tid] = __ldg(vv + q);
            }
        }
        for (int t = it.t0; t < it.t1; t++) {
            if (tid == 0) pf_next();
            float y[4] = {0.f, 0.f, 0.f, 0.f};
            float sl[REG ? NB : 1][36];
#pragma unroll
            for (int m = 0; m < NB; m++) {
                const int o = tid + m * HUGE_FNT;
                if (o < k) {
                    const int g = o >> 5, ng = min(32, k - 32 * g);
                    const float4 *S4 = reinterpret_cast<const float4 *>(R2 + (int64_t)36 * k * t + 36 * 32 * g) + (o & 31);
                    float *x36 = sl[REG ? m : 0];
#pragma unroll
                    for (int c = 0; c < 9; c++) {
                        const float4 x = S4[c * ng];
                        x36[4 * c] = x.x, x36[4 * c + 1] = x.y, x36[4 * c + 2] = x.z, x36[4 * c + 3] = x.w;
                    }
#pragma unroll
                    for (int q = 0; q < 9; q++) {
                        const float xq = sv[m][q][tid];
#pragma unroll
                        for (int r = 0; r < 4; r++) y[r] += x36[9 * r + q] * xq;
                    }
                }
            }
            {  // CTA sum of the 4 row dot products: warp transpose-reduce, one barrier, 16-lane butterfly
                const float yr = warp_sum4(y[0], y[1], y[2], y[3], lane);
                const int buf = nt++ & 1;
                if ((lane & 7) == 0) red[buf][warp][lane >> 3] = yr;
                __syncthreads();
                float4 pv = *reinterpret_cast<const float4 *>(&red[buf][lane & (HUGE_FNT / 32 - 1)][0]);
#pragma unroll
                for (int mm = HUGE_FNT / 64; mm; mm >>= 1) {
                    pv.x += __shfl_xor_sync(0xffffffffu, pv.x, mm);
                    pv.y += __shfl_xor_sync(0xffffffffu, pv.y, mm);
                    pv.z += __shfl_xor_sync(0xffffffffu, pv.z, mm);
                    pv.w += __shfl_xor_sync(0xffffffffu, pv.w, mm);
                }
                y[0] = pv.x, y[1] = pv.y, y[2] = pv.z, y[3] = pv.w;
            }
#pragma unroll
            for (int m = 0; m < NB; m++) {
                const int o = tid + m * HUGE_FNT;
                if (o < k) {
                    if (REG) {
#pragma unroll
                        for (int e = 0; e < 36; e++) acc[m][e % 9] += sl[REG ? m : 0][e] * y[e / 9];
                    } else {
                        const int g = o >> 5, ng = min(32, k - 32 * g);
                        const float4 *S4 =
                            reinterpret_cast<const float4 *>(R2 + (int64_t)36 * k * t + 36 * 32 * g) + (o & 31);
#pragma unroll
                        for (int c = 0; c < 9; c++) {
                            const float4 x = S4[c * ng];  // L2 hit: the tile was read just above
                            const float e4[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                            for (int u = 0; u < 4; u++) {
                                const int el = 4 * c + u, r = el / 9, q = el % 9;
                                acc[m][q] += e4[u] * y[r];
                            }
                        }
                    }
                }
            }
        }
        float *out = d.det ? nullptr : wslice(d);
        const int64_t ob0 = d.lm_obs0[j];
#pragma unroll
        for (int m = 0; m < NB; m++) {
            const int o = tid + m * HUGE_FNT;
            if (o < k) {
                if (d.det) det_store12(d, (int64_t)d.slot5[ob0 + o] + it.yoff, acc[m]);  // part = item within landmark
                else flush_cam12(out, oc[o], acc[m]);
            }
        }
    }
}

template <bool PRECOND>
__global__ void __launch_bounds__(HUGE_NT) k_huge_out(DevProblem d, float *__restrict__ out,
                                                      const PcgState *__restrict__ st) {
    if (!PRECOND && st && st->done) return;
    const HugeItem it = d.huge_out[blockIdx.x];
    const int64_t j = it.lm;
    const int k = d.lm_k[j], o = it.o0 + (int)threadIdx.x;
    if (o >= k) return;
    const float *R2 = d.arena + d.lm_r2[j];
    const int cam = d.obs_cam[d.lm_obs0[j] + o];
    float acc[9], P[PRECOND ? 45 : 1], b[PRECOND ? 9 : 1];
#pragma unroll
    for (int q = 0; q < 9; q++) acc[q] = 0.f;
    if (PRECOND) {
#pragma unroll
        for (int q = 0; q < 45; q++) P[q] = 0.f;
#pragma unroll
        for (int q = 0; q < 9; q++) b[q] = 0.f;
    }
    const float4 *TL = reinterpret_cast<const float4 *>(d.arena + d.lm_side[j] + side_tl(k));
    const float4 *Y = reinterpret_cast<const float4 *>(d.ybuf + it.yoff);
    // this CTA's camera blocks [o0, o0 + 256) are one contiguous range of each tile: TMA-prefetch
    // it into L2 two tiles ahead (thread 0; the threads are otherwise independent)
    const uint32_t span = 144u * (uint32_t)(min(it.o0 + HUGE_NT, k) - it.o0);
    const int64_t soff = (int64_t)36 * it.o0;
    if (threadIdx.x == 0)
        for (int t = it.t0; t < min(it.t1, it.t0 + 2); t++) bulk_prefetch_l2(R2 + (int64_t)36 * k * t + soff, span);
    for (int t = it.t0; t < it.t1; t++) {
        if (threadIdx.x == 0 && t + 2 < it.t1) bulk_prefetch_l2(R2 + (int64_t)36 * k * (t + 2) + soff, span);
        float sl[36];
        huge_slab(R2, k, t, o, sl);
        if (PRECOND) {
#pragma unroll
            for (int r = 0; r < 4; r++) {
                const int a = 4 * t + r;
                if (a < 2 * k) acc_rows(P, b, sl + 9 * r, TL[3 + a].w);
            }
        } else {
            const float4 y = Y[t];
#pragma unroll
            for (int q = 0; q < 9; q++) acc[q] += sl[q] * y.x + sl[9 + q] * y.y + sl[18 + q] * y.z + sl[27 + q] * y.w;
        }
    }
    if (PRECOND && d.det) det_store54(d, (int64_t)d.slot4[d.lm_obs0[j] + o] + it.t0 / HUGE_TPO, P, b);
    else if (PRECOND) flush54(pslice(d) + PACC_STRIDE * (int64_t)cam, P, b);
    else flush_cam12(wslice(d), cam, acc);  // (two-pass product: not used in deterministic mode)
}

// FP64 sum over the SM slices (stride `stride` floats per camera, `nv` values used), zeroing them
// for the next launch: out[nv * cam + e] = sum_s slice_s[stride * cam + e].  CTA = 32 outputs x 8
// slice phases (each thread sums every 8th slice, loads unrolled), then an 8-way smem reduction.
__global__ void __launch_bounds__(256) k_reduce_slices(float *__restrict__ sl, int64_t n_p, int stride, int nv,
                                                       int nslice, double *__restrict__ out,
                                                       const PcgState *__restrict__ st) {
    if (st && st->done) return;  // PCG graph: no matvec ran, the slices are still zero
    __shared__ double part[8][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int64_t i = (int64_t)blockIdx.x * 32 + tx;
    double s = 0.0;
    if (i < nv * n_p) {
        const int64_t cam = i / nv;
        const int64_t e = stride * cam + (i - nv * cam);
        const int64_t S = (int64_t)stride * n_p;
        float a[24];
#pragma unroll
        for (int u = 0; u < 24; u++) {  // all loads in flight first (nslice <= 192), then the zeroing
            const int k = ty + 8 * u;
            a[u] = k < nslice ? sl[k * S + e] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 24; u++) {
            const int k = ty + 8 * u;
            if (k < nslice) sl[k * S + e] = 0.f;
        }
        for (int k = ty + 8 * 24; k < nslice; k += 8) {  // (more than 192 SMs)
            s += (double)sl[k * S + e];
            sl[k * S + e] = 0.f;
        }
#pragma unroll
        for (int u = 0; u < 24; u += 4) s += ((double)a[u] + (double)a[u + 1]) + ((double)a[u + 2] + (double)a[u + 3]);
    }
    part[ty][tx] = s;
    __syncthreads();
    if (ty == 0 && i < nv * n_p) {
        double t = 0.0;
#pragma unroll
        for (int y = 0; y < 8; y++) t += part[y][tx];
        out[i] = t;
    }
}

// out = H~ v = wd + lambda D_p^2 v  (test hook, FP32 out)
__global__ void k_add_damping(DevProblem d, const float *v, float *out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 9 * d.n_p) return;
    out[i] = (float)(d.wd[i] + d.scal[SC_LAM] * d.Dp264[i] * v[i]);
}

// ============================================================================ K6 PCG (single CTA)
// Reading C11: stop when |rho| <= tol |rho_0| or it == max; p^T w <= 0 -> indefinite.
__device__ __forceinline__ void precond_apply(const DevProblem &d, const double *in, double *outv, int64_t N) {
    for (int64_t i = threadIdx.x; i < N; i += blockDim.x) {
        const int64_t cam = i / 9;
        const int a = (int)(i - 9 * cam);
        const double *M = d.Minv + 81 * cam + 9 * a;
        const double *x = in + 9 * cam;
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < 9; b++) s += M[b] * x[b];
        outv[i] = s;
    }
}

// ---- one PCG iteration as three multi-CTA kernels (the single-CTA k_pcg_step is latency-bound at
// ~60 us on config 4).  Dots are per-CTA partials summed in a fixed order by the last CTA to finish
// (threadfence + counter), so the result does not depend on CTA scheduling.
__device__ __forceinline__ bool last_cta(unsigned int *ctr) {
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(ctr, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) __threadfence();
    return last;
}
__device__ __forceinline__ double sum_parts(const double *part, int n, int stride, double *red) {
    double t = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) t += __ldcg(part + (int64_t)i * stride);  // (L2: other CTAs' writes)
    return block_sum_d(t, red);
}

// A: w = wd + lambda D_p^2 p, with wd = the sum of the per-SM slices (fused: 32 outputs x 8 slice
// phases per CTA, slices zeroed for the next product) or already in wd (all-reduced / other
// storage); then alpha = rho^T z / p^T w, or done with "indefinite" if p^T w <= 0.
__global__ void __launch_bounds__(256) k_pcg_a(DevProblem d, int fuse, cudaGraphConditionalHandle h, int use_h) {
    __shared__ double part[8][33];
    __shared__ double red[32];
    PcgState *st = d.pcg;
    if (st->done) {
        if (use_h && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(h, 0);
        return;
    }
    const double lam = d.scal[SC_LAM];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int64_t N = 9 * d.n_p, i = (int64_t)blockIdx.x * 32 + tx;
    double s = 0.0;
    if (i < N) {
        if (fuse) {
            const int64_t cam = i / 9, e = 12 * cam + (i - 9 * cam), S = 12 * d.n_p;
            float a[24];
#pragma unroll
            for (int u = 0; u < 24; u++) {  // all loads first (nslice <= 192 here), then the zeroing
                const int k = ty + 8 * u;
                a[u] = k < d.nslice ? d.wsl[k * S + e] : 0.f;
            }
#pragma unroll
            for (int u = 0; u < 24; u++) {
                const int k = ty + 8 * u;
                if (k < d.nslice) d.wsl[k * S + e] = 0.f;
            }
            for (int k = ty + 8 * 24; k < d.nslice; k += 8) {  // (more than 192 SMs)
                s += (double)d.wsl[k * S + e];
                d.wsl[k * S + e] = 0.f;
            }
#pragma unroll
            for (int u = 0; u < 24; u += 4) s += ((double)a[u] + (double)a[u + 1]) + ((double)a[u + 2] + (double)a[u + 3]);
        } else if (ty == 0) {
            s = d.wd[i];
        }
    }
    part[ty][tx] = s;
    __syncthreads();
    double pw = 0.0;
    if (ty == 0 && i < N) {
        double t = 0.0;
#pragma unroll
        for (int y = 0; y < 8; y++) t += part[y][tx];
        if (fuse) d.wd[i] = t;
        const double w = t + lam * d.Dp264[i] * d.p[i];
        d.w[i] = w;
        pw = d.p[i] * w;
    }
    pw = block_sum_d(pw, red);
    if (threadIdx.x == 0) d.pcg_part[blockIdx.x] = pw;
    if (!last_cta(&st->ctr_a)) return;
    pw = sum_parts(d.pcg_part, gridDim.x, 1, red);
    if (threadIdx.x == 0) {
        st->ctr_a = 0;
        if (!(pw > 0.0)) {
            st->done = 1, st->reason = 2;
            if (use_h) cudaGraphSetConditional(h, 0);
        } else {
            st->alpha = st->rz / pw;
        }
    }
}

// B: thread <-> one entry (32 cameras x 9 per CTA): x += alpha p, rho -= alpha w, then z = M^-1 rho
// with the camera's 9 updated rho entries exchanged through shared memory; |rho|, rho^T z.  The
// last CTA decides convergence (C11) / max iterations and forms beta.
__global__ void __launch_bounds__(288) k_pcg_b(DevProblem d, cudaGraphConditionalHandle h, int use_h) {
    __shared__ double red[32];
    __shared__ double rs[288];
    PcgState *st = d.pcg;
    if (st->done) return;  // (A already cleared the condition)
    const double alpha = st->alpha;
    const int tid = threadIdx.x, cl = tid / 9, a = tid - 9 * cl;
    const int64_t cam = (int64_t)blockIdx.x * 32 + cl, i = 9 * cam + a;
    const bool valid = cam < d.n_p;
    double r = 0.0;
    if (valid) {
        d.x[i] += alpha * d.p[i];
        r = d.r[i] - alpha * d.w[i];
        d.r[i] = r;
    }
    rs[tid] = r;
    __syncthreads();
    double rr = r * r, rz = 0.0;
    if (valid) {
        const double *M = d.Minv + 81 * cam + 9 * a;
        double z = 0.0;
#pragma unroll
        for (int q = 0; q < 9; q++) z += M[q] * rs[9 * cl + q];
        d.z[i] = z;
        rz = r * z;
    }
    rr = block_sum_d(rr, red);
    rz = block_sum_d(rz, red);
    if (threadIdx.x == 0) d.pcg_part[2 * blockIdx.x] = rr, d.pcg_part[2 * blockIdx.x + 1] = rz;
    if (!last_cta(&st->ctr_b)) return;
    rr = sum_parts(d.pcg_part, gridDim.x, 2, red);
    rz = sum_parts(d.pcg_part + 1, gridDim.x, 2, red);
    if (threadIdx.x == 0) {
        st->ctr_b = 0;
        const int it = st->it + 1;
        st->it = it;
        st->rn = sqrt(rr);
        int stop = 0;
        if (sqrt(rr) <= st->tol * st->r0) stop = 1, st->reason = 0;
        else if (it >= st->max_iters) stop = 1, st->reason = 1;
        if (stop) st->done = 1;
        if (use_h) cudaGraphSetConditional(h, stop ? 0 : 1);
        st->beta = rz / st->rz;
        st->rz = rz;
    }
}

// C: p = z + beta p (and its FP32 copy for the product)
__global__ void __launch_bounds__(256) k_pcg_c(DevProblem d) {
    const PcgState *st = d.pcg;
    if (st->done) return;
    const double beta = st->beta;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 9 * d.n_p) return;
    const double pn = d.z[i] + beta * d.p[i];
    d.p[i] = pn;
    d.p32[i] = (float)pn;
}

// PCG vectors (x, rho, z, p, w) are FP64 (9 n_p each, reading C24); the matvec reads p as FP32 (p32).
__global__ void __launch_bounds__(1024) k_pcg_init(DevProblem d, cudaGraphConditionalHandle h, int use_h) {
    __shared__ double red[32];
    const int64_t N = 9 * d.n_p;
    double rr = 0.0;
    for (int64_t i = threadIdx.x; i < N; i += blockDim.x) {
        const double r = -d.bt[i];
        d.r[i] = r;
        d.x[i] = 0.0;
        rr += r * r;
    }
    __syncthreads();
    precond_apply(d, d.r, d.z, N);
    __syncthreads();
    double rz = 0.0;
    for (int64_t i = threadIdx.x; i < N; i += blockDim.x) {
        d.p[i] = d.z[i];
        d.p32[i] = (float)d.z[i];
        rz += d.r[i] * d.z[i];
    }
    rr = block_sum_d(rr, red);
    rz = block_sum_d(rz, red);
    if (threadIdx.x == 0) {
        d.pcg->rz = rz;
        d.pcg->r0 = sqrt(rr);
        d.pcg->rn = sqrt(rr);
        d.pcg->it = 0;
        d.pcg->reason = 0;
        // a block found not SPD by k_precond_finalize makes the attempt indefinite
        const bool nspd = d.scal[SC_NSPD] > 0.0;
        d.pcg->done = (rr == 0.0 || d.pcg->max_iters <= 0 || nspd) ? 1 : 0;
        if (nspd) d.pcg->reason = 2;
        d.pcg->ctr_a = 0;
        d.pcg->ctr_b = 0;
        if (use_h) cudaGraphSetConditional(h, d.pcg->done ? 0 : 1);
    }
}

// lam < 0: read lambda from d.scal[SC_LAM] (graph launches).  use_h: also drive the graph's
// while-loop condition (0 once the solve is done).
__global__ void __launch_bounds__(1024) k_pcg_step(DevProblem d, cudaGraphConditionalHandle h, int use_h) {
    __shared__ double red[32];
    __shared__ int stop;
    PcgState *st = d.pcg;
    const double lam = d.scal[SC_LAM];
    const double tol = st->tol;
    const int max_iters = st->max_iters;
    if (st->done) {
        if (use_h && threadIdx.x == 0) cudaGraphSetConditional(h, 0);
        return;
    }
    const int64_t N = 9 * d.n_p;
    double pw = 0.0;
    for (int64_t i = threadIdx.x; i < N; i += blockDim.x) {
        const double w = d.wd[i] + lam * d.Dp264[i] * d.p[i];
        d.w[i] = w;
        pw += d.p[i] * w;
    }
    pw = block_sum_d(pw, red);
    if (!(pw > 0.0)) {
        if (threadIdx.x == 0) {
            st->done = 1, st->reason = 2;
            if (use_h) cudaGraphSetConditional(h, 0);
        }
        return;
    }
    const double alpha = st->rz / pw;
    double rr = 0.0;
    for (int64_t i = threadIdx.x; i < N; i += blockDim.x) {
        d.x[i] += alpha * d.p[i];
        const double r = d.r[i] - alpha * d.w[i];
        d.r[i] = r;
        rr += r * r;
    }
    rr = block_sum_d(rr, red);
    if (threadIdx.x == 0) {
        const int it = st->it + 1;
        st->it = it;
        st->rn = sqrt(rr);
        stop = 0;
        if (sqrt(rr) <= tol * st->r0) stop = 1, st->reason = 0;
        else if (it >= max_iters) stop = 1, st->reason = 1;
        if (stop) st->done = 1;
        if (use_h) cudaGraphSetConditional(h, stop ? 0 : 1);
    }
    __syncthreads();
    if (stop) return;
    precond_apply(d, d.r, d.z, N);
    __syncthreads();
    double rz = 0.0;
    for (int64_t i = threadIdx.x; i < N; i += blockDim.x) rz += d.r[i] * d.z[i];
    rz = block_sum_d(rz, red);
    const double beta = rz / st->rz;
    for (int64_t i = threadIdx.x; i < N; i += blockDim.x) {
        const double pn = d.z[i] + beta * d.p[i];
        d.p[i] = pn;
        d.p32[i] = (float)pn;
    }
    __syncthreads();
    if (threadIdx.x == 0) st->rz = rz;
}

// ============================================================================ K7 back-substitution
// Landmarks are stored sorted by k, so K7 splits them into three regimes by lanes per landmark,
// each a block-uniform role of one grid (one wave; blocks per regime in proportion to its bytes):
// L = 4 for k <= 16 (8 landmarks per warp and sweep), a warp (L = 32) for 16 < k <= 256, a CTA
// (L = 256) for k > 256.  Lane gl <-> observations o = gl, gl + L, ...: one camera-index load, then
// the observation's 9 FP64 dp entries and its 3 x 9 R^1 | Q^1^T J_p entries (the lanes of a group
// read contiguous 36-byte row segments) are independent loads in flight; the three row sums are
// reduced with shuffles (+ shared memory for L = 256); every lane of the group solves the 3x3
// upper-triangular system, lanes 0..2 write one component each (their point / scaling entries
// and the TL rows are loaded with the R^1 rows; the next sweep's header one sweep ahead).  (Round
// 1: 8 lanes over the flattened 9k columns of every landmark, a division and a dependent
// camera-index load per element, the longest tracks last on 8 lanes: 0.16 ms on config 3.)  The
// model-decrease sums go out once per CTA (same-address FP64 atomics serialize).
#ifndef RBA_BACKSUB_MINB
#define RBA_BACKSUB_MINB 3
#endif
#ifndef RBA_BS_L0
#define RBA_BS_L0 4  // lanes per landmark for k <= 16 (mean k ~4.2-4.6 on configs 3-4)
#endif
struct BsRange {
    int64_t lo, hi;  // landmarks of the regime
    int nb;          // its blocks
};
template <int L>
__device__ __forceinline__ void bs_regime(const DevProblem &d, const BsRange R, int b0, double &q1, double &dd,
                                          double (*sw)[3]) {
    constexpr int PB = 256 / L;  // landmarks per block and sweep
    const int gl = threadIdx.x % L;
    const int64_t step = (int64_t)R.nb * PB;
    int64_t j = R.lo + (int64_t)(blockIdx.x - b0) * PB + threadIdx.x / L;
    int k = 0;
    int64_t soff = 0, obs0 = 0;
    if (j < R.hi) k = __ldg(d.lm_k + j), soff = __ldg(d.lm_side + j), obs0 = __ldg(d.lm_obs0 + j);
    // the loop test is on the warp's first landmark (L = 8) / j itself (L >= 32): warp- resp. block-uniform
    for (; j - (int64_t)((threadIdx.x & 31) / L) < R.hi; j += step) {
        const bool valid = j < R.hi;
        const int qc = gl < 3 ? gl : 0;
        double pt = 0.0;
        float lsq = 0.f, lDq = 0.f;
        if (valid && gl < 3) pt = d.pts[3 * j + qc], lsq = __ldg(d.lm_s + 3 * j + qc), lDq = __ldg(d.lm_D + 3 * j + qc);
        const float *side = d.arena + soff;
        const int W = 9 * k;
        const int32_t *oc = d.obs_cam + obs0;
        const int kc = valid ? k : 0;
        {  // next sweep's header
            const int64_t jn = j + step;
            k = 0, soff = 0, obs0 = 0;
            if (jn < R.hi) k = __ldg(d.lm_k + jn), soff = __ldg(d.lm_side + jn), obs0 = __ldg(d.lm_obs0 + jn);
        }
        float4 t0 = make_float4(1.f, 0.f, 0.f, 0.f), t1 = make_float4(0.f, 1.f, 0.f, 0.f), t2 = make_float4(0.f, 0.f, 1.f, 0.f);
        if (valid && gl < 3) {
            const float4 *TL = reinterpret_cast<const float4 *>(side + side_tl(kc));
            t0 = __ldg(TL), t1 = __ldg(TL + 1), t2 = __ldg(TL + 2);
        }
        // FP64 arithmetic on the stored FP32 R^1 | Q^1^T J_p rows (the 3x3 solve amplifies errors by
        // cond(R^1), large for far / short-baseline landmarks)
        double s0 = 0.0, s1 = 0.0, s2 = 0.0;
        for (int o = gl; o < kc; o += L) {
            const double *x = d.x + 9 * (int64_t)__ldg(oc + o);
            const float *r0 = side + 9 * o;
            float a0[9], a1[9], a2[9];
            double xv[9];
#pragma unroll
            for (int q = 0; q < 9; q++) {
                xv[q] = x[q];
                a0[q] = __ldg(r0 + q);
                a1[q] = __ldg(r0 + W + q);
                a2[q] = __ldg(r0 + 2 * W + q);
            }
#pragma unroll
            for (int q = 0; q < 9; q++) {
                s0 += (double)a0[q] * xv[q];
                s1 += (double)a1[q] * xv[q];
                s2 += (double)a2[q] * xv[q];
            }
        }
        constexpr int WL = L < 32 ? L : 32;
#pragma unroll
        for (int m = WL / 2; m; m >>= 1) {
            s0 += __shfl_xor_sync(0xffffffffu, s0, m, WL);
            s1 += __shfl_xor_sync(0xffffffffu, s1, m, WL);
            s2 += __shfl_xor_sync(0xffffffffu, s2, m, WL);
        }
        if (L == 256) {  // the 8 warp sums, added in warp order by threads 0..2
            if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5][0] = s0, sw[threadIdx.x >> 5][1] = s1, sw[threadIdx.x >> 5][2] = s2;
            __syncthreads();
            if (threadIdx.x < 3) {
                s0 = s1 = s2 = 0.0;
#pragma unroll
                for (int w = 0; w < 8; w++) s0 += sw[w][0], s1 += sw[w][1], s2 += sw[w][2];
            }
            __syncthreads();
        }
        if (valid && gl < 3) {  // lanes 0..2 solve and write one component each
            const double b0 = t0.w + s0, b1 = t1.w + s1, b2 = t2.w + s2;
            const double x2 = b2 / t2.z;
            const double x1 = (b1 - t1.z * x2) / t1.y;
            const double x0 = (b0 - t0.y * x1 - (double)t0.z * x2) / t0.x;
            const float dlq = (float)-(qc == 0 ? x0 : qc == 1 ? x1 : x2);
            if (gl == 0) q1 += (double)t0.w * t0.w + (double)t1.w * t1.w + (double)t2.w * t2.w;
            d.dl[3 * j + qc] = dlq;
            d.pts_trial[3 * j + qc] = pt + (double)(lsq * dlq);
            const double Dd = (double)lDq * dlq;
            dd += Dd * Dd;
        }
    }
}

__global__ void __launch_bounds__(256, RBA_BACKSUB_MINB) k_backsub(DevProblem d, BsRange r8, BsRange r32, BsRange r256) {
    __shared__ double red[32];
    __shared__ double sw[8][3];
    if (d.pcg->reason == 2) return;  // indefinite attempt: no step (the LM control rejects it)
    const double lam = d.scal[SC_LAM];
    double q1 = 0.0, dd = 0.0;
    const int b = blockIdx.x;
    if (b < r8.nb) bs_regime<RBA_BS_L0>(d, r8, 0, q1, dd, sw);
    else if (b < r8.nb + r32.nb) bs_regime<32>(d, r32, r8.nb, q1, dd, sw);
    else bs_regime<256>(d, r256, r8.nb + r32.nb, q1, dd, sw);
    q1 = block_sum_d(q1, red);
    dd = block_sum_d(dd, red);
    if (d.det) {
        det_grid_sum(q1, d.det_part + DS_Q1R2 * DET_PART, d.det_ctr + DS_Q1R2, d.scal + SC_Q1R2);
        det_grid_sum(lam * dd, d.det_part + DS_DAMPL * DET_PART, d.det_ctr + DS_DAMPL, d.scal + SC_DAMPL);
    } else if (threadIdx.x == 0) {
        atomicAdd(d.scal + SC_Q1R2, q1);
        atomicAdd(d.scal + SC_DAMPL, lam * dd);
    }
}

// trial cameras x_p + S_p dp and the (replicated) camera part of the model decrease (C10):
// sum_i (-b~_i dp_i + rho_i dp_i + lam D_p,i^2 dp_i^2)
__global__ void __launch_bounds__(1024) k_trial_cams(DevProblem d, int with_model) {
    __shared__ double red[32];
    if (d.pcg->reason == 2) return;
    const double lam = d.scal[SC_LAM];
    const int64_t N = 9 * d.n_p;
    double m = 0.0;
    for (int64_t i = threadIdx.x; i < N; i += blockDim.x) {
        const double dp = d.x[i];
        d.cams_trial[i] = d.cams[i] + d.sp64[i] * dp;
        m += -d.bt[i] * dp + d.r[i] * dp + lam * d.Dp264[i] * dp * dp;
    }
    m = block_sum_d(m, red);
    if (threadIdx.x == 0) d.scal[SC_MODELP] = with_model ? m : 0.0;
}

// ============================================================================ K8 cost
__global__ void __launch_bounds__(256) k_cost(DevProblem d, const double *__restrict__ campre,
                                              const double *__restrict__ pts, int slot, int bad_slot) {
    __shared__ double red[32];
    if (slot == SC_ET && d.pcg->reason == 2) return;  // indefinite attempt: no trial point
    double e = 0.0, bad = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d.n_obs;
         i += (int64_t)gridDim.x * blockDim.x) {  // grid-stride (see k_linearize)
        double c[CAMPRE], r[2];
        load_pre(campre, d.obs_cam[i], c);
        const double *X = pts + 3 * (int64_t)d.obs_lm[i];
        const double2 uv = d.obs_uv[i];
        const double Pz = cam_model_pre<float>(c, X[0], X[1], X[2], uv.x, uv.y, r, nullptr, nullptr);
        if (!(Pz < 0.0) || !isfinite(r[0]) || !isfinite(r[1])) bad += 1.0;
        else e += robust_rho(r[0] * r[0] + r[1] * r[1], d.huber);
    }
    e = block_sum_d(e, red);
    bad = block_sum_d(bad, red);
    if (threadIdx.x == 0 && bad > 0) atomicAdd(d.scal + bad_slot, bad);
    if (d.det) det_grid_sum(e, d.det_part + DS_ET * DET_PART, d.det_ctr + DS_ET, d.scal + slot);
    else if (threadIdx.x == 0) atomicAdd(d.scal + slot, e);
}

// ============================================================================ launchers
static inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }


__global__ void k_nsmid(int *out) {
    unsigned r;
    asm volatile("mov.u32 %0, %%nsmid;" : "=r"(r));
    *out = (int)r;
}
// number of SM-id slots (%nsmid >= any %smid; SM ids need not be dense)
cudaError_t query_nsmid(rba_ctx *c, int *d_scratch, int *out) {
    k_nsmid<<<1, 1, 0, c->stream>>>(d_scratch);
    cudaError_t e = cudaMemcpyAsync(out, d_scratch, sizeof(int), cudaMemcpyDeviceToHost, c->stream);
    if (e) return e;
    return cudaStreamSynchronize(c->stream);
}

__global__ void k_cam_prep(const double *__restrict__ cams, double *__restrict__ pre, int64_t n_p) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n_p) cam_prep(cams + 9 * i, pre + CAMPRE * i);
}
// per-camera R / J_left of the current (trial = 0) or trial (1) cameras
cudaError_t launch_cam_prep(rba_ctx *c, int trial) {
    k_cam_prep<<<nblk(c->d.n_p, 128), 128, 0, c->stream>>>(trial ? c->d.cams_trial : c->d.cams,
                                                            trial ? c->d.campre_trial : c->d.campre, c->d.n_p);
    c->launches++;
    return cudaGetLastError();
}

// landmark state between the caller's order (pts_io, 3 n_l global) and the internal order
__global__ void k_pts_permute(DevProblem d, int to_internal) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= d.n_l) return;
    const int64_t g = d.lm_orig[i];
#pragma unroll
    for (int q = 0; q < 3; q++) {
        if (to_internal) d.pts[3 * i + q] = d.pts_io[3 * g + q];
        else d.pts_io[3 * g + q] = d.pts[3 * i + q];
    }
}
cudaError_t launch_pts_permute(rba_ctx *c, int to_internal) {
    if (c->d.n_l == 0) return cudaSuccess;
    k_pts_permute<<<nblk(c->d.n_l, 256), 256, 0, c->stream>>>(c->d, to_internal);
    c->launches++;
    return cudaGetLastError();
}

cudaError_t launch_check_depth(rba_ctx *c, int *d_bad) {
    if (c->d.n_obs == 0) return cudaSuccess;
    launch_cam_prep(c, 0);
    k_check_depth<<<nblk(c->d.n_obs, 256), 256, 0, c->stream>>>(c->d, d_bad);
    c->launches++;
    return cudaGetLastError();
}

cudaError_t launch_linearize(rba_ctx *c) {
    launch_cam_prep(c, 0);
    if (c->d.n_obs == 0) return cudaSuccess;
    Prof P(c, KID_LIN, 24.0 * c->d.n_obs);
    k_linearize<<<(unsigned)std::min<int64_t>(nblk(c->d.n_obs, 256), 8 * (int64_t)c->num_sms), 256, 0, c->stream>>>(c->d);
    P.end();
    c->launches++;
    return cudaGetLastError();
}

cudaError_t launch_cam_scale(rba_ctx *c) {
    k_cam_scale<<<nblk(9 * c->d.n_p, 256), 256, 0, c->stream>>>(c->d, (float)c->opt.diag_min,
                                                                  (float)c->opt.diag_max);
    c->launches++;
    return cudaGetLastError();
}

extern double plan_marg_bytes(rba_ctx *c);
extern double plan_backsub_bytes(rba_ctx *c);
extern double plan_matvec_bytes(rba_ctx *c);

// fork the context stream into the auxiliary streams (independent class kernels) and join back
// (RBA_NOFORK: everything on the context stream, a diagnostic switch)
static bool nofork_env() {
    static const bool v = getenv("RBA_NOFORK") != nullptr;
    return v;
}
struct ForkJoin {
    rba_ctx *c;
    int next = 0;
    bool on;
    explicit ForkJoin(rba_ctx *c_) : c(c_), on(!c_->nofork && !nofork_env()) {
        if (!on) return;
        cudaEventRecord(c->ev_fork, c->stream);
        for (int i = 0; i < rba_ctx::NAUX; i++) cudaStreamWaitEvent(c->aux[i], c->ev_fork, 0);
    }
    cudaStream_t s() {  // round robin: context stream, aux 0, aux 1, ...
        if (!on) return c->stream;
        const int i = next++ % (rba_ctx::NAUX + 1);
        return i == 0 ? c->stream : c->aux[i - 1];
    }
    void join() {
        if (!on) return;
        for (int i = 0; i < rba_ctx::NAUX; i++) {
            cudaEventRecord(c->ev_join[i], c->aux[i]);
            cudaStreamWaitEvent(c->stream, c->ev_join[i], 0);
        }
    }
};

template <int G>
static cudaError_t marg_small_cls(rba_ctx *c, int cls, cudaStream_t st) {
    const int64_t lo = G == 32 ? 0 : c->pack_lo[cls], hi = G == 32 ? c->n_mid_packs : c->pack_hi[cls];
    if (hi <= lo) return cudaSuccess;
    const size_t sm = (size_t)4 * ((32 / G) * SmallTab<G>::FLOATS + SmallTab<G>::SIDE) * sizeof(float);
    k_marg_small<G><<<nblk(hi - lo, 4), 128, sm, st>>>(c->d, G == 32 ? c->d.mid_packs : c->d.packs, lo, hi,
                                                              (float)c->opt.diag_min, (float)c->opt.diag_max);
    c->launches++;
    return cudaGetLastError();
}

template <int NT, bool MULTI = false, int LPC = 1>
static cudaError_t marg_large_cls(rba_ctx *c, int cls, cudaStream_t st) {
    const int64_t lo = c->marg_lo[cls], hi = c->marg_hi[cls];
    if (hi <= lo) return cudaSuccess;
    const int64_t K = MULTI ? (cls == 5 ? c->huge_max_k : KLARGE) : NT;
    const int64_t sub_floats = pad4(4 * (2 * K + 3) + 8 * K);  // per item (sub-block)
    const size_t sm = (size_t)LPC * sub_floats * sizeof(float);
    cudaFuncSetAttribute(k_marg_large<NT, MULTI, LPC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_marg_large<NT, MULTI, LPC><<<(unsigned)((hi - lo + LPC - 1) / LPC), NT * LPC, sm, st>>>(
        c->d, c->d.marg_items + lo, hi - lo, sub_floats, (float)c->opt.diag_min, (float)c->opt.diag_max);
    c->launches++;
    return cudaGetLastError();
}

cudaError_t launch_marginalize(rba_ctx *c) {
    Prof P(c, KID_MARG, plan_marg_bytes(c));
    cudaError_t e;
    ForkJoin F(c);
    static const bool m512 = getenv("RBA_MARG512_MULTI") && atoi(getenv("RBA_MARG512_MULTI"));  // tuning knob
    static const bool small_first = getenv("RBA_MARG_ORDER") && atoi(getenv("RBA_MARG_ORDER"));  // tuning knob
    auto smalls = [&]() -> cudaError_t {
        cudaError_t x;
        if ((x = marg_small_cls<16>(c, 3, F.s()))) return x;
        if ((x = marg_small_cls<8>(c, 2, F.s()))) return x;
        if ((x = marg_small_cls<4>(c, 1, F.s()))) return x;
        return marg_small_cls<2>(c, 0, F.s());
    };
    if (small_first && (e = smalls())) return e;
    if ((e = marg_large_cls<512, true>(c, 5, F.s()))) return e;
    if (m512) {
        if ((e = marg_large_cls<256, true>(c, 4, F.s()))) return e;
    } else if ((e = marg_large_cls<512>(c, 4, F.s()))) {
        return e;
    }
    if ((e = marg_large_cls<256>(c, 3, F.s()))) return e;
    if ((e = marg_large_cls<128>(c, 2, F.s()))) return e;
    if ((e = marg_large_cls<64, false, RBA_MARG_LPC64>(c, 1, F.s()))) return e;
    // 17 <= k <= 32: warp per landmark (shuffle reductions, 4 landmarks per CTA) when dense FP32
    if (c->n_mid_packs > 0) {
        if ((e = marg_small_cls<32>(c, 0, F.s()))) return e;
    } else if ((e = marg_large_cls<32>(c, 0, F.s()))) {
        return e;
    }
    if (!small_first && (e = smalls())) return e;
    F.join();
    P.end();
    return cudaSuccess;
}

cudaError_t launch_redamp(rba_ctx *c) {
    if (c->d.n_l == 0) return cudaSuccess;
    if (c->d.fac) return launch_fac_redamp(c);
    Prof P(c, KID_DAMP, 0.0);
    k_redamp<<<nblk(32 * c->d.n_l, 256), 256, 0, c->stream>>>(c->d);
    P.end();
    c->launches++;
    return cudaGetLastError();
}

template <int NS, int NSLOT, bool PRE>
static void large_pipe_cls(rba_ctx *c, int cls, const float *v, float *out, const PcgState *st, cudaStream_t ss) {
    const int64_t n = c->cta_n[cls];
    if (n <= 0) return;
    using Cf = PipeCfg<NS, NSLOT>;
    cudaFuncSetAttribute(k_large_pipe<NS, NSLOT, PRE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cf::SMEM);
    k_large_pipe<NS, NSLOT, PRE><<<(unsigned)n, Cf::NC + 32, Cf::SMEM, ss>>>(
        c->d, c->d.tiles, c->d.cta_lo + c->cta_off[cls], v, out, st, c->d.det ? c->d.run_part + c->run_off[cls] : nullptr);
    c->launches++;
}

template <bool PRE>
static void pipes_all(rba_ctx *c, const float *v, float *out12, const PcgState *st) {
    ForkJoin F(c);
    static const bool fused_env = !getenv("RBA_HUGE_TWOPASS");
    const bool fused = fused_env || c->d.det;  // (the two-pass product has no deterministic slots)
    if (c->n_huge_fused > 0 && !PRE && fused) {  // k > KLARGE: fused passes (second read from L2)
        // items of k <= HUGE_REG_K first; RBA_HUGE_PERSIST: one CTA per SM looping over the items
        // (default: CTA per item, the block scheduler balances)
        static const bool persist = getenv("RBA_HUGE_PERSIST") != nullptr;
        static const bool noreg = getenv("RBA_HUGE_NOREG") != nullptr;
        // L2 prefetch distance of the fused kernel in bytes per CTA (tuning knob RBA_HUGE_PF)
        static const int huge_pf = getenv("RBA_HUGE_PF") ? atoi(getenv("RBA_HUGE_PF")) : RBA_HUGE_PF_DEFAULT;
        const int64_t nr = noreg ? 0 : c->n_huge_reg, ng = c->n_huge_fused - nr;
        auto grid = [&](int64_t n) { return (unsigned)(persist ? std::min<int64_t>(n, c->num_sms) : n); };
        if (nr > 0) {
            constexpr size_t sm2 = (size_t)2 * 9 * HUGE_FNT * sizeof(float);
            cudaFuncSetAttribute(k_huge_fused<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
            k_huge_fused<2, true><<<grid(nr), HUGE_FNT, sm2, F.s()>>>(c->d, c->d.huge_fused, nr, v, st, huge_pf);
            c->launches++;
        }
        if (ng > 0) {
            constexpr size_t smn = (size_t)HUGE_NB * 9 * HUGE_FNT * sizeof(float);
            cudaFuncSetAttribute(k_huge_fused<HUGE_NB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smn);
            k_huge_fused<HUGE_NB, false><<<grid(ng), HUGE_FNT, smn, F.s()>>>(c->d, c->d.huge_fused + nr, ng, v, st, huge_pf);
            c->launches++;
        }
    } else if (c->n_huge_out > 0) {  // k > KLARGE: two passes, same stream
        cudaStream_t hs = F.s();
        if (!PRE) {
            k_huge_y<<<(unsigned)c->n_huge_y, HUGE_NT, 0, hs>>>(c->d, v, st);
            c->launches++;
        }
        if (PRE) k_huge_out<true><<<(unsigned)c->n_huge_out, HUGE_NT, 0, hs>>>(c->d, out12, st);
        else k_huge_out<false><<<(unsigned)c->n_huge_out, HUGE_NT, 0, hs>>>(c->d, out12, st);
        c->launches++;
    }
    // longest first so the short classes fill the long ones' tails
    large_pipe_cls<512, 1, PRE>(c, 4, v, out12, st, F.s());
    if (c->chunk_ctas > 0) {
        cudaFuncSetAttribute(k_small_pipe<PRE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SP_SMEM);
        static const int dbg = getenv("RBA_DEBUG_SMALLPIPE") ? atoi(getenv("RBA_DEBUG_SMALLPIPE")) : 0;
        k_small_pipe<PRE><<<(unsigned)c->chunk_ctas, SP_WARPS * 32 + 32, SP_SMEM, F.s()>>>(c->d, v, out12, st,
                                                                                           PRE ? 0 : dbg);
        c->launches++;
    }
    large_pipe_cls<256, 1, PRE>(c, 3, v, out12, st, F.s());
    large_pipe_cls<128, 2, PRE>(c, 2, v, out12, st, F.s());
    large_pipe_cls<64, 4, PRE>(c, 1, v, out12, st, F.s());
    large_pipe_cls<32, 8, PRE>(c, 0, v, out12, st, F.s());
    F.join();
}

static void reduce_slices(rba_ctx *c, float *sl, int stride, int nv, double *out, const PcgState *st) {
    if (c->d.det) {  // deterministic mode: the camera-major slots, fixed order (family by stride / nv)
        if (c->d.n_p == 0) return;
        if (nv == 54) k_det_reduce<54><<<(unsigned)c->d.n_p, 256, 0, c->stream>>>(c->d.obuf, c->d.camptr4, PACC_STRIDE, out, st);
        else k_det_reduce<9><<<(unsigned)c->d.n_p, 256, 0, c->stream>>>(c->d.obuf, sl == nullptr ? c->d.camptr1 : c->d.camptr5,
                                                                          12, out, st);
        c->launches++;
        return;
    }
    k_reduce_slices<<<nblk(nv * c->d.n_p, 32), 256, 0, c->stream>>>(sl, c->d.n_p, stride, nv, c->d.nslice, out, st);
    c->launches++;
}

// K1 camera column norms^2: the per-SM slices into cam_n2d (FP32 path; sqrt-BA-64 adds FP64 directly)
cudaError_t launch_reduce_cam_norms(rba_ctx *c) {
    if (c->d.s64) launch_reduce_slices64(c, c->d.cam_n2d);
    else reduce_slices(c, c->d.det ? nullptr : c->d.wsl, 12, 9, c->d.cam_n2d, nullptr);  // (det: family 1)
    return cudaGetLastError();
}

cudaError_t launch_precond_rhs(rba_ctx *c) {
    Prof P(c, KID_PRE, plan_matvec_bytes(c));
    if (c->d.s64) {
        launch_pre64(c);
        P.end();
        return cudaGetLastError();
    }
    if (c->d.fac) launch_fac_precond(c);
    else pipes_all<true>(c, nullptr, c->d.psl, nullptr);
    reduce_slices(c, c->d.psl, PACC_STRIDE, 54, c->d.pd, nullptr);
    P.end();
    return cudaGetLastError();
}

cudaError_t launch_precond_finalize(rba_ctx *c) {
    k_precond_finalize<<<nblk(c->d.n_p, FIN_WARPS), 32 * FIN_WARPS, 0, c->stream>>>(c->d, c->d.scal + SC_NSPD);
    c->launches++;
    return cudaGetLastError();
}

// wd = (H~ - lambda D_p^2) v: sqrt-BA product (Eq. cg_mult) or, in explicit-SC mode, the BSR SpMV.
// reduce = false: leave the sum in the per-SM slices (k_pcg_a reduces them); returns whether the
// product went to the slices.
static bool matvec_body(rba_ctx *c, const float *v, const PcgState *st, bool reduce = true) {
    if (c->d.sc) {
        launch_sc_spmv(c, st, st ? nullptr : v);
        return false;
    }
    if (c->d.s64) {  // sqrt-BA-64: FP64 product straight into wd
        const double *v64 = c->d.p;
        if (!st) {  // test hook: FP32 input
            launch_f2d64(c, v, c->d.z, 9 * c->d.n_p);
            v64 = c->d.z;
        }
        launch_rcs64(c, v64, st);
        return false;
    }
    if (c->d.fac) launch_fac_matvec(c, v, st);
    else pipes_all<false>(c, v, c->d.wsl, st);
    if (c->d.det) {  // the slots are always reduced here (k_pcg_a then reads wd)
        reduce_slices(c, c->d.wsl, 12, 9, c->d.wd, st);
        return false;
    }
    if (reduce) reduce_slices(c, c->d.wsl, 12, 9, c->d.wd, st);
    return true;
}

static cudaError_t matvec_impl(rba_ctx *c, const float *v, const PcgState *st) {
    Prof P(c, KID_MATVEC, plan_matvec_bytes(c));
    matvec_body(c, v, st);
    P.end();
    return cudaGetLastError();
}

// wd = sum_j A_j^T (A_j v_j) in FP64 (callers all-reduce it afterwards)
cudaError_t launch_matvec(rba_ctx *c, const float *v, float *) { return matvec_impl(c, v, nullptr); }
// PCG iteration product: the slices are reduced by k_pcg_a unless the result is all-reduced first
cudaError_t launch_matvec_pcg(rba_ctx *c) {
    Prof P(c, KID_MATVEC, plan_matvec_bytes(c));
    // with an all-reduce between product and update (multi-GPU), reduce the slices into wd here
    // and let the update kernels read wd; otherwise the first update kernel sums the slices
    const bool reduce_now = c->host_reduce_path();
    c->pcg_fused = matvec_body(c, c->d.p32, c->d.pcg, reduce_now) && !reduce_now;
    P.end();
    return cudaGetLastError();
}

cudaError_t launch_add_damping(rba_ctx *c, const float *v, float *out) {
    k_add_damping<<<nblk(9 * c->d.n_p, 256), 256, 0, c->stream>>>(c->d, v, out);
    c->launches++;
    return cudaGetLastError();
}

cudaError_t launch_pcg_init(rba_ctx *c, cudaGraphConditionalHandle h, int use_h) {
    k_pcg_init<<<1, 1024, 0, c->stream>>>(c->d, h, use_h);
    c->launches++;
    return cudaGetLastError();
}

static void pcg_update(rba_ctx *c, cudaStream_t s, bool fuse, cudaGraphConditionalHandle h, int use_h) {
    const int64_t N = 9 * c->d.n_p;
    k_pcg_a<<<(unsigned)((N + 31) / 32), 256, 0, s>>>(c->d, fuse ? 1 : 0, h, use_h);
    k_pcg_b<<<nblk(c->d.n_p, 32), 288, 0, s>>>(c->d, h, use_h);
    k_pcg_c<<<nblk(N, 256), 256, 0, s>>>(c->d);
    c->launches += 3;
}

// The PCG update after a product (launch_matvec_pcg + the all-reduce of wd when sharded); h / use_h:
// the conditional handle of the device-side PCG `while` loop the update kernels drive.
cudaError_t launch_pcg_step(rba_ctx *c, cudaGraphConditionalHandle h, int use_h) {
    Prof P(c, KID_PCG, 0.0);
    static const bool single = getenv("RBA_PCG_SINGLE_CTA") != nullptr;  // the single-CTA step (A/B)
    if (single) {
        if (c->pcg_fused) reduce_slices(c, c->d.wsl, 12, 9, c->d.wd, c->d.pcg);
        k_pcg_step<<<1, 1024, 0, c->stream>>>(c->d, h, use_h);
        c->launches++;
    } else {
        pcg_update(c, c->stream, c->pcg_fused, h, use_h);
    }
    c->pcg_fused = false;
    P.end();
    return cudaGetLastError();
}

cudaError_t launch_backsub(rba_ctx *c) {
    Prof P(c, KID_BACKSUB, c->d.sc || c->d.fac || c->d.s64 ? 0.0 : plan_backsub_bytes(c));
    if (c->d.sc) {
        cudaError_t e = launch_sc_backsub(c);
        if (e) return e;
    } else if (c->d.fac) {
        cudaError_t e = launch_fac_backsub(c);
        if (e) return e;
    } else if (c->d.s64) {
        cudaError_t e = launch_backsub64(c);
        if (e) return e;
    } else if (c->d.n_l) {
        // one wave; blocks per regime in proportion to its bytes, capped by its landmark count
        static int per_sm = 0;
        if (!per_sm && (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_backsub, 256, 0) || per_sm < 1)) per_sm = 3;
        const int64_t G = std::min<int64_t>((int64_t)c->num_sms * per_sm, DET_PART);
        BsRange r[3];
        int64_t lo = 0;
        // per-regime weights on the byte shares (tuning knob RBA_BS_W="w0,w1,w2"; measured on cfg 3 /
        // cfg 4: 1,1,1 0.095 / 0.286 ms, 1,1.5,1.5 0.086 / 0.252, 1,2,2 0.088 / 0.266, 2,1,1 0.125 / 0.406)
        static double w[3] = {1.0, 1.5, 1.5};
        static const bool wset = [] {
            if (const char *e = getenv("RBA_BS_W")) sscanf(e, "%lf,%lf,%lf", &w[0], &w[1], &w[2]);
            return true;
        }();
        (void)wset;
        const double tot = w[0] * c->bs_bytes[0] + w[1] * c->bs_bytes[1] + w[2] * c->bs_bytes[2];
        constexpr int per_block[3] = {256 / RBA_BS_L0, 8, 1};  // landmarks per block and sweep
        for (int i = 0; i < 3; i++) {
            const int64_t hi = std::max(lo, c->bs_hi[i]), n = hi - lo;
            int64_t nb = n ? std::max<int64_t>(1, (int64_t)(G * w[i] * c->bs_bytes[i] / tot)) : 0;
            nb = std::min<int64_t>(nb, (n + per_block[i] - 1) / per_block[i]);
            r[i] = BsRange{lo, hi, (int)nb};
            lo = hi;
        }
        const unsigned g = (unsigned)(r[0].nb + r[1].nb + r[2].nb);
        k_backsub<<<g, 256, 0, c->stream>>>(c->d, r[0], r[1], r[2]);
        c->launches++;
    }
    k_trial_cams<<<1, 1024, 0, c->stream>>>(c->d, c->d.sc ? 0 : 1);
    c->launches++;
    P.end();
    return cudaGetLastError();
}

cudaError_t launch_cost(rba_ctx *c, int at_trial, int slot) {
    if (c->d.n_obs == 0) return cudaSuccess;
    Prof P(c, KID_COST, 20.0 * c->d.n_obs);
    const int bad_slot = at_trial ? SC_BADT : SC_BAD;
    launch_cam_prep(c, at_trial);
    k_cost<<<(unsigned)std::min<int64_t>(nblk(c->d.n_obs, 256), 8 * (int64_t)c->num_sms), 256, 0, c->stream>>>(c->d, at_trial ? c->d.campre_trial : c->d.campre,
                                                          at_trial ? c->d.pts_trial : c->d.pts, slot, bad_slot);
    P.end();
    c->launches++;
    return cudaGetLastError();
}

cudaError_t launch_trial_cost(rba_ctx *c) { return launch_cost(c, 1, SC_ET); }
cudaError_t launch_commit(rba_ctx *) { return cudaSuccess; }

}  // namespace rba
