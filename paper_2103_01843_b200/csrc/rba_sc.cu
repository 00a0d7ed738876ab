// rba_sc.cu -- explicit Schur-complement baseline (the paper's "explicit-32" /
// "explicit-64" solvers, Table 1).  Same linearization, scaling, damping,
// PCG and LM control as the sqrt-BA path; only the landmark elimination differs:
//   H_ll,j = J_l,j^T J_l,j + lambda D_l^2                      (3 x 3, per landmark)
//   H~_pp  = H_pp + lambda D_p^2 - sum_j H_pl,j H_ll,j^-1 H_lp,j  (block-sparse, camera pairs)
//   b~_p   = b_p - sum_j H_pl,j H_ll,j^-1 b_l,j                 (Eq. P:197-198 with P:277)
//   dl_j   = -H_ll,j^-1 (b_l,j + H_lp,j dp)
// stored explicitly as 9 x 9 blocks on the covisibility graph (BSR, both triangles), in FP32
// (explicit-32) or FP64 (explicit-64), T below.  Arithmetic of the reduction is in T too: that is
// what the paper compares (the FP32 Schur complement loses definiteness).
// Product path only (no oracle code).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "rba_internal.cuh"
#include "rba_model.cuh"

namespace rba {

// per-observation scaled, IRLS-weighted Jacobians of landmark j's observation a
template <typename T>
struct ObsJ {
    T jp[2][9], jl[2][3], r[2];
    int cam;
};

template <typename T>
__device__ __forceinline__ void sc_obs(const DevProblem &d, int64_t j, int a, ObsJ<T> &o) {
    const int64_t oi = d.lm_obs0[j] + a;
    o.cam = d.obs_cam[oi];
    double c[CAMPRE], r[2];
    T Jc[18], Jl[6];
    load_pre(d.campre, o.cam, c);
    const double *X = d.pts + 3 * j;
    const double2 uv = d.obs_uv[oi];
    cam_model_pre<T>(c, X[0], X[1], X[2], uv.x, uv.y, r, Jc, Jl);
    apply_irls<T>(r, Jc, Jl, d.huber);
#pragma unroll
    for (int q = 0; q < 9; q++) {
        const T s = (T)d.sp[9 * o.cam + q];
        o.jp[0][q] = Jc[q] * s;
        o.jp[1][q] = Jc[9 + q] * s;
    }
#pragma unroll
    for (int q = 0; q < 3; q++) o.jl[0][q] = Jl[q], o.jl[1][q] = Jl[3 + q];
    o.r[0] = (T)r[0];
    o.r[1] = (T)r[1];
}

template <typename T>
__device__ __forceinline__ T warp_sum_t(T v) {
#pragma unroll
    for (int m = 16; m; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
    return v;
}

// landmark scaling (C7, C8) and the 3x3 system of landmark j, reduced over the warp
template <typename T>
struct LmSys {
    T sl[3], Dl[3];
    T Hinv[9];  // (H_ll + lambda D_l^2)^-1, symmetric
    T bl[3];
};

template <typename T>
__device__ void sc_landmark_system(const DevProblem &d, int64_t j, int k, T lam, float dmin, float dmax, LmSys<T> &S) {
    const int lane = threadIdx.x & 31;
    T n2[3] = {0, 0, 0};
    for (int a = lane; a < k; a += 32) {
        ObsJ<T> o;
        sc_obs<T>(d, j, a, o);
#pragma unroll
        for (int q = 0; q < 3; q++) n2[q] += o.jl[0][q] * o.jl[0][q] + o.jl[1][q] * o.jl[1][q];
    }
#pragma unroll
    for (int q = 0; q < 3; q++) {
        n2[q] = warp_sum_t(n2[q]);
        S.sl[q] = T(1) / (T(1) + sqrt(n2[q]));
        T D2 = n2[q] * S.sl[q] * S.sl[q];
        D2 = D2 < (T)dmin ? (T)dmin : (D2 > (T)dmax ? (T)dmax : D2);
        S.Dl[q] = sqrt(D2);
    }
    T H[6] = {0, 0, 0, 0, 0, 0}, b[3] = {0, 0, 0};  // H00 H01 H02 H11 H12 H22
    for (int a = lane; a < k; a += 32) {
        ObsJ<T> o;
        sc_obs<T>(d, j, a, o);
        for (int rr = 0; rr < 2; rr++) {
            const T x0 = o.jl[rr][0] * S.sl[0], x1 = o.jl[rr][1] * S.sl[1], x2 = o.jl[rr][2] * S.sl[2];
            H[0] += x0 * x0, H[1] += x0 * x1, H[2] += x0 * x2, H[3] += x1 * x1, H[4] += x1 * x2, H[5] += x2 * x2;
            b[0] += x0 * o.r[rr], b[1] += x1 * o.r[rr], b[2] += x2 * o.r[rr];
        }
    }
#pragma unroll
    for (int i = 0; i < 6; i++) H[i] = warp_sum_t(H[i]);
#pragma unroll
    for (int i = 0; i < 3; i++) S.bl[i] = warp_sum_t(b[i]);
    H[0] += lam * S.Dl[0] * S.Dl[0];
    H[3] += lam * S.Dl[1] * S.Dl[1];
    H[5] += lam * S.Dl[2] * S.Dl[2];
    // symmetric 3x3 inverse by cofactors
    const T c00 = H[3] * H[5] - H[4] * H[4], c01 = H[2] * H[4] - H[1] * H[5], c02 = H[1] * H[4] - H[2] * H[3];
    const T c11 = H[0] * H[5] - H[2] * H[2], c12 = H[1] * H[2] - H[0] * H[4], c22 = H[0] * H[3] - H[1] * H[1];
    const T det = H[0] * c00 + H[1] * c01 + H[2] * c02;
    const T id = T(1) / det;
    S.Hinv[0] = c00 * id, S.Hinv[1] = c01 * id, S.Hinv[2] = c02 * id;
    S.Hinv[3] = c01 * id, S.Hinv[4] = c11 * id, S.Hinv[5] = c12 * id;
    S.Hinv[6] = c02 * id, S.Hinv[7] = c12 * id, S.Hinv[8] = c22 * id;
}

__device__ __forceinline__ int64_t bsr_find(const DevProblem &d, int r, int c) {
    int lo = d.bsr_ptr[r], hi = d.bsr_ptr[r + 1] - 1;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (d.bsr_col[mid] < c) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ void atomic_add_t(float *p, float v) { atomicAdd(p, v); }
__device__ __forceinline__ void atomic_add_t(double *p, double v) { atomicAdd(p, v); }

// one (a, b) contribution -L_a^T G_b (+ J_a^T J_a on the diagonal) to a stored 9 x 9 block:
// FP32 as 21 float4 reductions over the 84-element block, FP64 as 81 scalar ones
template <typename O>
__device__ __forceinline__ void sc_block_add(float *B, const float *L, const float *gv, const O &o, bool diag) {
    float v[SC_BS];
#pragma unroll
    for (int q1 = 0; q1 < 9; q1++)
#pragma unroll
        for (int q2 = 0; q2 < 9; q2++) {
            float x = -(L[3 * q1] * gv[3 * q2] + L[3 * q1 + 1] * gv[3 * q2 + 1] + L[3 * q1 + 2] * gv[3 * q2 + 2]);
            if (diag) x += o.jp[0][q1] * o.jp[0][q2] + o.jp[1][q1] * o.jp[1][q2];
            v[9 * q1 + q2] = x;
        }
#pragma unroll
    for (int i = 81; i < SC_BS; i++) v[i] = 0.f;
    float4 *B4 = reinterpret_cast<float4 *>(B);
#pragma unroll
    for (int i = 0; i < SC_BS / 4; i++) atomicAdd(B4 + i, make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]));
}
template <typename O>
__device__ __forceinline__ void sc_block_add(double *B, const double *L, const double *gv, const O &o, bool diag) {
#pragma unroll 1
    for (int q1 = 0; q1 < 9; q1++)
#pragma unroll
        for (int q2 = 0; q2 < 9; q2++) {
            double x = -(L[3 * q1] * gv[3 * q2] + L[3 * q1 + 1] * gv[3 * q2 + 1] + L[3 * q1 + 2] * gv[3 * q2 + 2]);
            if (diag) x += o.jp[0][q1] * o.jp[0][q2] + o.jp[1][q1] * o.jp[1][q2];
            atomicAdd(B + 9 * q1 + q2, x);
        }
}

// lower blocks of H~ from the upper ones: block (r, c), c < r, = block (c, r)^T.  Warp per block row.
template <typename T>
__global__ void __launch_bounds__(256) k_sc_mirror(DevProblem d) {
    T *val = reinterpret_cast<T *>(d.bsr_val);
    const int lane = threadIdx.x & 31;
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (r >= d.n_p) return;
    for (int e = d.bsr_ptr[r] + lane; e < d.bsr_ptr[r + 1]; e += 32) {
        const int c = d.bsr_col[e];
        if (c >= r) continue;
        const T *U = val + SC_BS * bsr_find(d, c, (int)r);
        T *B = val + SC_BS * (int64_t)e;
#pragma unroll
        for (int q1 = 0; q1 < 9; q1++)
#pragma unroll
            for (int q2 = 0; q2 < 9; q2++) B[9 * q1 + q2] = U[9 * q2 + q1];
    }
}

// ---- build: warp per landmark (grid-stride).  Phase 1: per observation a, G_a = J_p,a^T J_l,a
// (9x3, the H_pl block) and L_a = G_a H_ll^-1 go to a per-observation scratch; b~ contributions
// J_p,a^T r_a - L_a b_l are added.  Phase 2: lane a adds block (a, b), b >= a:
//   delta_ab J_p,a^T J_p,a - L_a G_b^T   to H~(c_a, c_b) (and its transpose to H~(c_b, c_a)).
template <typename T>
__global__ void __launch_bounds__(256) k_sc_build(DevProblem d, float dmin, float dmax) {
    const T lam = (T)d.scal[SC_LAM];  // lambda of this attempt (explicit-32: rounded to FP32)
    T *val = reinterpret_cast<T *>(d.bsr_val);
    T *bsc = reinterpret_cast<T *>(d.sc_b);
    T *scr = reinterpret_cast<T *>(d.sc_scratch);
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < d.n_l; j += nwarps) {
        const int k = d.lm_k[j];
        LmSys<T> S;
        sc_landmark_system<T>(d, j, k, lam, dmin, dmax, S);
        if (lane < 3) {
            d.lm_s[3 * j + lane] = (float)S.sl[lane];
            d.lm_D[3 * j + lane] = (float)S.Dl[lane];
        }
        const int64_t obs0 = d.lm_obs0[j];
        for (int a = lane; a < k; a += 32) {
            ObsJ<T> o;
            sc_obs<T>(d, j, a, o);
            T *g = scr + 54 * (obs0 + a), *l = g + 27;
            T bt[9];
#pragma unroll
            for (int q = 0; q < 9; q++) {
                T G[3];
#pragma unroll
                for (int m = 0; m < 3; m++) G[m] = (o.jp[0][q] * o.jl[0][m] + o.jp[1][q] * o.jl[1][m]) * S.sl[m];
#pragma unroll
                for (int m = 0; m < 3; m++) {
                    g[3 * q + m] = G[m];
                    l[3 * q + m] = G[0] * S.Hinv[m] + G[1] * S.Hinv[3 + m] + G[2] * S.Hinv[6 + m];
                }
                bt[q] = o.jp[0][q] * o.r[0] + o.jp[1][q] * o.r[1] -
                        (l[3 * q] * S.bl[0] + l[3 * q + 1] * S.bl[1] + l[3 * q + 2] * S.bl[2]);
            }
#pragma unroll
            for (int q = 0; q < 9; q++) atomic_add_t(bsc + 9 * (int64_t)o.cam + q, bt[q]);
        }
        __syncwarp();
        for (int a = lane; a < k; a += 32) {
            ObsJ<T> o;
            sc_obs<T>(d, j, a, o);
            const T *la = scr + 54 * (obs0 + a) + 27;
            T L[27];
#pragma unroll
            for (int i = 0; i < 27; i++) L[i] = la[i];
            // upper triangle only (observations are camera-sorted, so cam_a <= cam_b); the lower
            // blocks are filled by k_sc_mirror
            for (int b = a; b < k; b++) {
                const int cb = d.obs_cam[obs0 + b];
                const T *gb = scr + 54 * (obs0 + b);
                T *B = val + SC_BS * bsr_find(d, o.cam, cb);
                T gv[27];
#pragma unroll
                for (int i = 0; i < 27; i++) gv[i] = gb[i];
                sc_block_add(B, L, gv, o, b == a);
            }
        }
        __syncwarp();
    }
}

// ---- SpMV on the explicit H~ (without lambda D_p^2, added by the PCG update); out in FP64.
// SpMV, CTA per camera row: threads stride over the row's blocks (each block read once, as 16-byte
// vectors), 9 partial sums per thread reduced across the CTA (warp shuffles + shared memory).
template <typename T>
__global__ void __launch_bounds__(128) k_sc_spmv_row(DevProblem d, const T *__restrict__ v, double *__restrict__ out,
                                                     const PcgState *__restrict__ st) {
    if (st && st->done) return;
    __shared__ double red[4][9];
    const int c = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const T *val = reinterpret_cast<const T *>(d.bsr_val);
    T acc[9];
#pragma unroll
    for (int i = 0; i < 9; i++) acc[i] = 0;
    for (int e = d.bsr_ptr[c] + tid; e < d.bsr_ptr[c + 1]; e += 128) {
        const T *x = v + 9 * (int64_t)__ldg(d.bsr_col + e);
        T xv[9];
#pragma unroll
        for (int q = 0; q < 9; q++) xv[q] = __ldg(x + q);
        T b[SC_BS];
        if constexpr (sizeof(T) == 4) {
            const float4 *B4 = reinterpret_cast<const float4 *>(val + SC_BS * (int64_t)e);
#pragma unroll
            for (int u = 0; u < SC_BS / 4; u++) {
                const float4 w = __ldcs(B4 + u);
                b[4 * u] = w.x, b[4 * u + 1] = w.y, b[4 * u + 2] = w.z, b[4 * u + 3] = w.w;
            }
        } else {
            const double2 *B2 = reinterpret_cast<const double2 *>(val + SC_BS * (int64_t)e);
#pragma unroll
            for (int u = 0; u < SC_BS / 2; u++) {
                const double2 w = __ldcs(B2 + u);
                b[2 * u] = w.x, b[2 * u + 1] = w.y;
            }
        }
#pragma unroll
        for (int i = 0; i < 9; i++)
#pragma unroll
            for (int q = 0; q < 9; q++) acc[i] += b[9 * i + q] * xv[q];
    }
#pragma unroll
    for (int i = 0; i < 9; i++) {
        double t = (double)acc[i];
#pragma unroll
        for (int m = 16; m; m >>= 1) t += __shfl_xor_sync(0xffffffffu, t, m);
        if (lane == 0) red[warp][i] = t;
    }
    __syncthreads();
    if (tid < 9) out[9 * (int64_t)c + tid] = red[0][tid] + red[1][tid] + red[2][tid] + red[3][tid];
}

// preconditioner blocks (the diagonal blocks of H~, 45 upper entries) and b~ into pd (FP64)
template <typename T>
__global__ void k_sc_precond(DevProblem d) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= d.n_p) return;
    const T *B = reinterpret_cast<const T *>(d.bsr_val) + SC_BS * bsr_find(d, (int)c, (int)c);
    const T *bsc = reinterpret_cast<const T *>(d.sc_b);
    double *o = d.pd + 54 * c;
    int idx = 0;
    for (int a = 0; a < 9; a++)
        for (int b = a; b < 9; b++) o[idx++] = (double)B[9 * a + b];
    for (int a = 0; a < 9; a++) o[45 + a] = (double)bsc[9 * c + a];
}

// ---- back-substitution dl_j = -H_ll^-1 (b_l + sum_a G_a^T dp_a) and the model decrease
// L(0) - L(dx) = -sum_a (2 r_a^T J_a dx_a + |J_a dx_a|^2) (C10, undamped), summed per CTA.
template <typename T>
__global__ void __launch_bounds__(256) k_sc_backsub(DevProblem d, float dmin, float dmax) {
    __shared__ double red[32];
    if (d.pcg->reason == 2) return;  // indefinite attempt: no step
    const T lam = (T)d.scal[SC_LAM];
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double md = 0.0;
    for (int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < d.n_l; j += nwarps) {
        const int k = d.lm_k[j];
        LmSys<T> S;
        sc_landmark_system<T>(d, j, k, lam, dmin, dmax, S);
        T g[3] = {0, 0, 0};
        for (int a = lane; a < k; a += 32) {
            ObsJ<T> o;
            sc_obs<T>(d, j, a, o);
            const double *dp = d.x + 9 * (int64_t)o.cam;
            for (int rr = 0; rr < 2; rr++) {
                T u = 0;
#pragma unroll
                for (int q = 0; q < 9; q++) u += o.jp[rr][q] * (T)dp[q];
#pragma unroll
                for (int m = 0; m < 3; m++) g[m] += o.jl[rr][m] * S.sl[m] * u;
            }
        }
        T dl[3];
#pragma unroll
        for (int m = 0; m < 3; m++) g[m] = warp_sum_t(g[m]) + S.bl[m];
#pragma unroll
        for (int m = 0; m < 3; m++) dl[m] = -(S.Hinv[3 * m] * g[0] + S.Hinv[3 * m + 1] * g[1] + S.Hinv[3 * m + 2] * g[2]);
        for (int a = lane; a < k; a += 32) {
            ObsJ<T> o;
            sc_obs<T>(d, j, a, o);
            const double *dp = d.x + 9 * (int64_t)o.cam;
            for (int rr = 0; rr < 2; rr++) {
                double u = 0.0;
#pragma unroll
                for (int q = 0; q < 9; q++) u += (double)o.jp[rr][q] * dp[q];
#pragma unroll
                for (int m = 0; m < 3; m++) u += (double)(o.jl[rr][m] * S.sl[m]) * (double)dl[m];
                md -= 2.0 * (double)o.r[rr] * u + u * u;
            }
        }
        if (lane < 3) {
            d.dl[3 * j + lane] = (float)dl[lane];
            d.pts_trial[3 * j + lane] = d.pts[3 * j + lane] + (double)S.sl[lane] * (double)dl[lane];
        }
    }
    md = block_sum_d(md, red);
    if (threadIdx.x == 0) atomicAdd(d.scal + SC_Q1R2, md);
}

__global__ void k_f2d(const float *__restrict__ a, double *__restrict__ b, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) b[i] = a[i];
}

// ============================================================================ launchers
static inline unsigned nb(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

template <typename T>
static cudaError_t sc_build_t(rba_ctx *c) {
    DevProblem &d = c->d;
    cudaMemsetAsync(d.bsr_val, 0, sizeof(T) * SC_BS * (size_t)d.nnzb, c->stream);
    cudaMemsetAsync(d.sc_b, 0, sizeof(T) * 9 * (size_t)d.n_p, c->stream);
    if (d.n_l) {
        const unsigned g = (unsigned)std::min<int64_t>(nb(32 * d.n_l, 256), (int64_t)c->num_sms * 16);
        k_sc_build<T><<<g, 256, 0, c->stream>>>(d, (float)c->opt.diag_min, (float)c->opt.diag_max);
        k_sc_mirror<T><<<nb(32 * d.n_p, 256), 256, 0, c->stream>>>(d);
        c->launches += 2;
    }
    return cudaGetLastError();
}

cudaError_t launch_sc_build(rba_ctx *c) {
    Prof P(c, KID_MARG, c->marg_bytes);
    cudaError_t e = c->d.sc == 2 ? sc_build_t<double>(c) : sc_build_t<float>(c);
    P.end();
    return e;
}

cudaError_t launch_sc_precond(rba_ctx *c) {
    Prof P(c, KID_PRE, c->matvec_bytes);
    if (c->d.sc == 2) k_sc_precond<double><<<nb(c->d.n_p, 128), 128, 0, c->stream>>>(c->d);
    else k_sc_precond<float><<<nb(c->d.n_p, 128), 128, 0, c->stream>>>(c->d);
    c->launches++;
    P.end();
    return cudaGetLastError();
}

// wd = H~_sc v (no damping); v: the PCG direction (p32 for explicit-32, p for explicit-64)
void launch_sc_spmv(rba_ctx *c, const PcgState *st, const float *v32) {
    DevProblem &d = c->d;
    if (d.sc == 2) {
        const double *v = d.p;
        if (v32) {  // test hook: FP32 input
            k_f2d<<<nb(9 * d.n_p, 256), 256, 0, c->stream>>>(v32, d.z, 9 * d.n_p);
            c->launches++;
            v = d.z;
        }
        k_sc_spmv_row<double><<<(unsigned)d.n_p, 128, 0, c->stream>>>(d, v, d.wd, st);
    } else {
        k_sc_spmv_row<float><<<(unsigned)d.n_p, 128, 0, c->stream>>>(d, v32 ? v32 : d.p32, d.wd, st);
    }
    c->launches++;
}

cudaError_t launch_sc_backsub(rba_ctx *c) {
    DevProblem &d = c->d;
    if (d.n_l) {
        const unsigned g = (unsigned)std::min<int64_t>(nb(32 * d.n_l, 256), (int64_t)c->num_sms * 8);
        if (d.sc == 2)
            k_sc_backsub<double><<<g, 256, 0, c->stream>>>(d, (float)c->opt.diag_min, (float)c->opt.diag_max);
        else
            k_sc_backsub<float><<<g, 256, 0, c->stream>>>(d, (float)c->opt.diag_min, (float)c->opt.diag_max);
        c->launches++;
    }
    return cudaGetLastError();
}

}  // namespace rba
