// rba_sqrtba64.cu -- sqrt-BA-64 (the paper's double-precision variant, P:407,
// Table 1): the same QR nullspace marginalization (Householder + compact WY, 6 damping Givens),
// reduced-camera-system product, block-Jacobi blocks and back-substitution as the FP32 path, with
// the landmark blocks stored and all their arithmetic done in FP64.  Storage is the paper's logical
// block, (2k+3) x (9k+4) doubles per landmark in row-major rows (Fig. 2c): the reduced rows
// 3..2k+2 consecutive over landmarks, rows 0..2 and the 6 Givens pairs in a second region.  The
// product and block-Jacobi passes are TMA-staged (k_rcs64_ws / k_rcs64_tma / k_pre64_tma); the
// product's camera-space sums go to per-SM FP64 slices (k_reduce_slices64).
// Product path only (no oracle code).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "rba_internal.cuh"
#include "rba_model.cuh"

namespace rba {

// Block of landmark j, rows of W = 9k + 4 doubles: rows 3..2k+2 (the reduced rows A_j | q_j) at
// lm_r2[j], consecutive over landmarks so the product streams them back to back; rows 0..2 and the 12
// Givens doubles at lm_side[j] (a second region after all reduced rows).
struct Blk64 {
    double *r2, *side;
    int64_t W;
    __device__ __forceinline__ double *row(int a) const { return a < 3 ? side + a * W : r2 + (a - 3) * W; }
    __device__ __forceinline__ double *givens() const { return side + 3 * W; }
};
__device__ __forceinline__ Blk64 blk64(const DevProblem &d, int64_t j, int k) {
    return Blk64{d.arena64 + d.lm_r2[j], d.arena64 + d.lm_side[j], 9 * (int64_t)k + 4};
}

__device__ __forceinline__ void givens64(double a, double b, double &c, double &s) {
    if (b == 0.0) {
        c = 1.0, s = 0.0;
    } else {
        const double r = hypot(a, b);
        c = a / r, s = b / r;
    }
}

// the 6 damping rotations on rows {0,1,2} x {2k, 2k+1, 2k+2} (reading C5 / C6), FP64
__device__ __forceinline__ void damp64(const double *R, const double *sD, double *g) {
    double L6[18] = {};
#pragma unroll
    for (int i = 0; i < 9; i++) L6[i] = R[i];
#pragma unroll
    for (int i = 0; i < 3; i++) L6[(3 + i) * 3 + i] = sD[i];
#pragma unroll
    for (int m = 0; m < 6; m++) {
        const int p = damp_p(m), t = damp_t(m);
        double c, s;
        givens64(L6[p * 3 + p], L6[t * 3 + p], c, s);
        g[2 * m] = c, g[2 * m + 1] = s;
#pragma unroll
        for (int q = 0; q < 3; q++) {
            const double a = L6[p * 3 + q], b = L6[t * 3 + q];
            L6[p * 3 + q] = c * a + s * b;
            L6[t * 3 + q] = -s * a + c * b;
        }
        L6[t * 3 + p] = 0.0;
    }
}

// ---- K2-64: CTA per landmark; thread o' owns observations / camera blocks o = o', o' + NT, ...
// Householder on the scaled 2k x 3 landmark Jacobian in shared memory, compact WY, then every row
// of the block is written from  out[a, 9o+q] = E[a, 9o+q] - V[a] . M_o[:, q]  (rows 0..2k-1), the
// landmark / residual columns, and the damping rows by the 6 rotations of rows 0..2.
// Work item = (landmark, rows [r0, r1) of the pose rows 0..2k-1): the O(k) prologue is recomputed
// per item; the item with r0 == 0 also writes the special rows (0..2, 2k..2k+2) and the Givens.
template <int NT>
__global__ void __launch_bounds__(NT, NT == 32 ? 16 : 1) k_marg64(DevProblem d, const LargeItem *__restrict__ items,
                                               double dmin, double dmax) {
    extern __shared__ double s64[];
    __shared__ double red[4 * (NT / 32)];
    const LargeItem it = items[blockIdx.x];
    const int64_t j = it.lm;
    const int r0 = it.t0, r1 = it.t1;
    const int k = d.lm_k[j], tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double *SX = s64;           // 2k x 3 (scaled J_l, then R / V)
    double *SR = SX + 6 * k;    // 2k residual column
    double *SV = SR + 2 * k;    // 2k x 3 Householder vectors
    const int64_t obs0 = d.lm_obs0[j];
    const double *Xp = d.pts + 3 * j;
    auto bsum = [&](double *v, int n) {  // CTA sum of n <= 4 values, result in every thread
        for (int i = 0; i < n; i++) v[i] = warp_sum_d(v[i]);
        __syncthreads();
        if (lane == 0)
            for (int i = 0; i < n; i++) red[4 * warp + i] = v[i];
        __syncthreads();
        for (int i = 0; i < n; i++) {
            double s = 0.0;
            for (int w = 0; w < NT / 32; w++) s += red[4 * w + i];
            v[i] = s;
        }
        __syncthreads();
    };
    double n2[4] = {0, 0, 0, 0};
    for (int o = tid; o < k; o += NT) {
        double c[CAMPRE], r[2], Jc[18], Jl[6];
        load_pre(d.campre, d.obs_cam[obs0 + o], c);
        const double2 uv = d.obs_uv[obs0 + o];
        cam_model_pre<double>(c, Xp[0], Xp[1], Xp[2], uv.x, uv.y, r, Jc, Jl);
        apply_irls<double>(r, Jc, Jl, d.huber);
        for (int q = 0; q < 3; q++) {
            SX[6 * o + q] = Jl[q], SX[6 * o + 3 + q] = Jl[3 + q];
            n2[q] += Jl[q] * Jl[q] + Jl[3 + q] * Jl[3 + q];
        }
        SR[2 * o] = r[0], SR[2 * o + 1] = r[1];
    }
    bsum(n2, 3);
    double sl[3], Dl[3];
    for (int q = 0; q < 3; q++) {
        sl[q] = 1.0 / (1.0 + sqrt(n2[q]));
        Dl[q] = sqrt(fmin(fmax(n2[q] * sl[q] * sl[q], dmin), dmax));
    }
    for (int a = tid; a < 2 * k; a += NT)
        for (int q = 0; q < 3; q++) SX[3 * a + q] *= sl[q], SV[3 * a + q] = 0.0;
    __syncthreads();
    double tau[3];
    for (int c = 0; c < 3; c++) {  // reflector c on rows c..2k-1 (reading C4 for the sign)
        double sm[4] = {0, 0, 0, 0};
        for (int a = c + tid; a < 2 * k; a += NT) {
            const double x = SX[3 * a + c];
            sm[0] += x * x;
            if (c < 2) sm[1] += x * SX[3 * a + c + 1];
            if (c < 1) sm[2] += x * SX[3 * a + c + 2];
            sm[3] += x * SR[a];
        }
        const double x0 = SX[3 * c + c], y1 = c < 2 ? SX[3 * c + c + 1] : 0.0, y2 = c < 1 ? SX[3 * c + c + 2] : 0.0,
                     yr = SR[c];
        bsum(sm, 4);
        const double sig = sqrt(sm[0]), alpha = x0 >= 0.0 ? -sig : sig;
        const double vtv = 2.0 * sig * (sig + fabs(x0));
        const double tc = vtv > 0.0 ? 2.0 / vtv : 0.0;
        tau[c] = tc;
        const double d1 = sm[1] - alpha * y1, d2 = sm[2] - alpha * y2, dr = sm[3] - alpha * yr;
        for (int a = c + tid; a < 2 * k; a += NT) {
            const double vv = a == c ? x0 - alpha : SX[3 * a + c];
            SV[3 * a + c] = vv;
            if (c < 2) SX[3 * a + c + 1] -= tc * vv * d1;
            if (c < 1) SX[3 * a + c + 2] -= tc * vv * d2;
            SR[a] -= tc * vv * dr;
            SX[3 * a + c] = a == c ? alpha : 0.0;
        }
        __syncthreads();
    }
    double pv[4] = {0, 0, 0, 0};
    for (int a = tid; a < 2 * k; a += NT) {
        pv[0] += SV[3 * a] * SV[3 * a + 1];
        pv[1] += SV[3 * a] * SV[3 * a + 2];
        pv[2] += SV[3 * a + 1] * SV[3 * a + 2];
    }
    bsum(pv, 3);
    const double T00 = tau[0], T11 = tau[1], T22 = tau[2];
    const double T01 = -tau[1] * T00 * pv[0];
    const double T02 = -tau[2] * (T00 * pv[1] + T01 * pv[2]);
    const double T12 = -tau[2] * T11 * pv[2];
    // damping rotations from the undamped R (rows 0..2 of SX) and sqrt(lam) D_l
    double R[9], g[12];
    for (int i = 0; i < 9; i++) R[i] = SX[i];
    const double sq = sqrt(d.scal[SC_LAM]), sD[3] = {sq * Dl[0], sq * Dl[1], sq * Dl[2]};
    damp64(R, sD, g);
    const Blk64 B = blk64(d, j, k);
    // pose columns of every row: thread <-> camera block o (warp <-> 32 consecutive blocks); each
    // row's 9 x 32 values of a warp are staged in shared memory and stored as 9 coalesced 256-byte
    // segments (a thread's own 9 values are 72-byte strided across the warp)
    double *stage = SV + 6 * k + 288 * warp;  // per-warp 288 doubles
    for (int ob = 0; ob < k; ob += NT) {
        const int o = ob + tid;
        const bool act = o < k;
        const int wb = ob + 32 * warp;                       // first block of this warp
        const int ncol = 9 * max(0, min(32, k - wb));        // valid columns of the warp's segment
        double jp[18] = {}, M[27] = {};
        if (act) {
            double c[CAMPRE], r[2], Jc[18], Jl[6];
            const int cam = d.obs_cam[obs0 + o];
            load_pre(d.campre, cam, c);
            const double2 uv = d.obs_uv[obs0 + o];
            cam_model_pre<double>(c, Xp[0], Xp[1], Xp[2], uv.x, uv.y, r, Jc, Jl);
            apply_irls<double>(r, Jc, Jl, d.huber);
            for (int q = 0; q < 9; q++) {
                const double sc = d.sp64[9 * cam + q];
                jp[q] = Jc[q] * sc, jp[9 + q] = Jc[9 + q] * sc;
            }
            const double *v0 = SV + 6 * o, *v1 = v0 + 3;  // M = T^T V_o^T J_o
            for (int q = 0; q < 9; q++) {
                const double W0 = v0[0] * jp[q] + v1[0] * jp[9 + q], W1 = v0[1] * jp[q] + v1[1] * jp[9 + q],
                             W2 = v0[2] * jp[q] + v1[2] * jp[9 + q];
                M[q] = T00 * W0;
                M[9 + q] = T01 * W0 + T11 * W1;
                M[18 + q] = T02 * W0 + T12 * W1 + T22 * W2;
            }
        }
        double top[27];  // undamped rows 0..2, then mixed into rows 0..2 / 2k..2k+2
        for (int a = r0; a < r1; a++) {
            const double *va = SV + 3 * a;
            double row[9];
#pragma unroll
            for (int q = 0; q < 9; q++) {
                double x = -(va[0] * M[q] + va[1] * M[9 + q] + va[2] * M[18 + q]);
                if ((a >> 1) == o) x += jp[9 * (a & 1) + q];
                row[q] = x;
            }
            if (a < 3) {
#pragma unroll
                for (int q = 0; q < 9; q++) top[9 * a + q] = row[q];
                continue;
            }
#pragma unroll
            for (int q = 0; q < 9; q++) stage[9 * lane + q] = row[q];
            __syncwarp();
            double *dst = B.row(a) + 9 * wb;
            for (int i = lane; i < ncol; i += 32) dst[i] = stage[i];
            __syncwarp();
        }
        if (r0 != 0) continue;
        for (int s = 0; s < 6; s++) {  // the damped special rows from rows 0..2 (staged the same way)
            double xs[9];
#pragma unroll
            for (int q = 0; q < 9; q++) {
                double x[6] = {top[q], top[9 + q], top[18 + q], 0.0, 0.0, 0.0};
#pragma unroll
                for (int m = 0; m < 6; m++) {
                    const int p = damp_p(m), t = damp_t(m);
                    const double aa = x[p], bb = x[t];
                    x[p] = g[2 * m] * aa + g[2 * m + 1] * bb;
                    x[t] = -g[2 * m + 1] * aa + g[2 * m] * bb;
                }
                xs[q] = x[s];
            }
#pragma unroll
            for (int q = 0; q < 9; q++) stage[9 * lane + q] = xs[q];
            __syncwarp();
            const int row = s < 3 ? s : 2 * k + s - 3;
            double *dst = B.row(row) + 9 * wb;
            for (int i = lane; i < ncol; i += 32) dst[i] = stage[i];
            __syncwarp();
        }
    }
    // landmark and residual columns (4 per row): R / 0 and Q^T r, damping rows rotated
    for (int a = r0 + tid; a < r1; a += NT) {
        double *rw = B.row(a) + 9 * k;
        if (a >= 3 && a < 2 * k) {
            rw[0] = rw[1] = rw[2] = 0.0;
            rw[3] = SR[a];
        }
    }
    if (tid == 0 && r0 == 0) {
        double X[6][4] = {};
        for (int i = 0; i < 3; i++) {
            for (int q = 0; q < 3; q++) X[i][q] = R[3 * i + q];
            X[i][3] = SR[i];
            X[3 + i][i] = sD[i];
        }
        for (int m = 0; m < 6; m++) {
            const int p = damp_p(m), t = damp_t(m);
            for (int q = 0; q < 4; q++) {
                const double a = X[p][q], b = X[t][q];
                X[p][q] = g[2 * m] * a + g[2 * m + 1] * b;
                X[t][q] = -g[2 * m + 1] * a + g[2 * m] * b;
            }
            X[t][p] = 0.0;
        }
        for (int s = 0; s < 6; s++) {
            const int row = s < 3 ? s : 2 * k + s - 3;
            for (int q = 0; q < 4; q++) B.row(row)[9 * k + q] = X[s][q];
        }
        double *G = B.givens();
        for (int i = 0; i < 12; i++) G[i] = g[i];
    }
    if (tid < 3 && r0 == 0) {
        d.lm_s[3 * j + tid] = (float)sl[tid];
        d.lm_D[3 * j + tid] = (float)Dl[tid];
        d.lm_D64[3 * j + tid] = Dl[tid];
        d.lm_s64[3 * j + tid] = sl[tid];
    }
}

// ---- K2-64 for short tracks (k <= 32): a group of G lanes per landmark (32/G landmarks per warp),
// lane <-> observation / camera block, the Householder reductions as G-lane shuffles (the FP64 port
// of the FP32 small-k kernel's prologue), V rows of other lanes fetched by shuffles row by row.
template <int G>
__device__ __forceinline__ double gsum64(double v) {
#pragma unroll
    for (int m = G / 2; m; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m, G);
    return v;
}

template <int G>
__global__ void __launch_bounds__(256) k_marg64_small(DevProblem d, int64_t lo, int64_t hi, double dmin,
                                                      double dmax) {
    const int lane = threadIdx.x & 31, gl = lane % G;
    const int64_t wfirst = lo + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * (32 / G);
    if (wfirst >= hi) return;  // warp-uniform
    const int64_t j = wfirst + lane / G;
    const bool valid = j < hi;
    const int k = valid ? d.lm_k[j] : 0;
    const bool act = gl < k;
    double r[2] = {0.0, 0.0}, Jc[18] = {}, Jl[6] = {};
    int cam = 0;
    if (act) {
        const int64_t o = d.lm_obs0[j] + gl;
        cam = d.obs_cam[o];
        double c[CAMPRE];
        load_pre(d.campre, cam, c);
        const double *Xp = d.pts + 3 * j;
        const double2 uv = d.obs_uv[o];
        cam_model_pre<double>(c, Xp[0], Xp[1], Xp[2], uv.x, uv.y, r, Jc, Jl);
        apply_irls<double>(r, Jc, Jl, d.huber);
    }
    double sl[3], Dl[3];
#pragma unroll
    for (int q = 0; q < 3; q++) {
        const double n2 = gsum64<G>(Jl[q] * Jl[q] + Jl[3 + q] * Jl[3 + q]);
        sl[q] = 1.0 / (1.0 + sqrt(n2));
        Dl[q] = sqrt(fmin(fmax(n2 * sl[q] * sl[q], dmin), dmax));
    }
    double jp[18], X[2][3], rv[2] = {r[0], r[1]};
#pragma unroll
    for (int q = 0; q < 9; q++) {
        const double sc = act ? d.sp64[9 * cam + q] : 0.0;
        jp[q] = Jc[q] * sc, jp[9 + q] = Jc[9 + q] * sc;
    }
#pragma unroll
    for (int q = 0; q < 3; q++) X[0][q] = Jl[q] * sl[q], X[1][q] = Jl[3 + q] * sl[q];
    double V[2][3], tau[3];
#pragma unroll
    for (int c = 0; c < 3; c++) {  // reflector c (reading C4 for the sign)
        double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
#pragma unroll
        for (int rr = 0; rr < 2; rr++) {
            const int a = 2 * gl + rr;
            const double x = (act && a >= c) ? X[rr][c] : 0.0;
            s0 += x * x;
            if (c + 1 < 3) s1 += x * X[rr][(c + 1) % 3];
            if (c + 2 < 3) s2 += x * X[rr][(c + 2) % 3];
            s3 += x * rv[rr];
        }
        s0 = gsum64<G>(s0), s1 = gsum64<G>(s1), s2 = gsum64<G>(s2), s3 = gsum64<G>(s3);
        const int pl = c >> 1, pr = c & 1;
        const double x0 = __shfl_sync(0xffffffffu, X[pr][c], pl, G);
        const double y1 = __shfl_sync(0xffffffffu, X[pr][(c + 1) % 3], pl, G);
        const double y2 = __shfl_sync(0xffffffffu, X[pr][(c + 2) % 3], pl, G);
        const double yr = __shfl_sync(0xffffffffu, rv[pr], pl, G);
        const double sig = sqrt(s0), alpha = x0 >= 0.0 ? -sig : sig;
        const double vtv = 2.0 * sig * (sig + fabs(x0));
        const double tc = vtv > 0.0 ? 2.0 / vtv : 0.0;
        tau[c] = tc;
        const double d1 = s1 - alpha * y1, d2 = s2 - alpha * y2, dr = s3 - alpha * yr;
#pragma unroll
        for (int rr = 0; rr < 2; rr++) {
            const int a = 2 * gl + rr;
            double vv = 0.0;
            if (act && a >= c) vv = a == c ? x0 - alpha : X[rr][c];
            V[rr][c] = vv;
            if (c + 1 < 3) X[rr][(c + 1) % 3] -= tc * vv * d1;
            if (c + 2 < 3) X[rr][(c + 2) % 3] -= tc * vv * d2;
            rv[rr] -= tc * vv * dr;
            if (a == c) X[rr][c] = alpha;
            else if (a > c) X[rr][c] = 0.0;
        }
    }
    double p01 = 0, p02 = 0, p12 = 0;
#pragma unroll
    for (int rr = 0; rr < 2; rr++) p01 += V[rr][0] * V[rr][1], p02 += V[rr][0] * V[rr][2], p12 += V[rr][1] * V[rr][2];
    p01 = gsum64<G>(p01), p02 = gsum64<G>(p02), p12 = gsum64<G>(p12);
    const double T00 = tau[0], T11 = tau[1], T22 = tau[2];
    const double T01 = -tau[1] * T00 * p01;
    const double T02 = -tau[2] * (T00 * p02 + T01 * p12);
    const double T12 = -tau[2] * T11 * p12;
    double R[9], rr3[3];
#pragma unroll
    for (int q = 0; q < 3; q++) {
        R[q] = __shfl_sync(0xffffffffu, X[0][q], 0, G);
        R[3 + q] = __shfl_sync(0xffffffffu, X[1][q], 0, G);
        R[6 + q] = __shfl_sync(0xffffffffu, X[0][q], 1, G);
    }
    rr3[0] = __shfl_sync(0xffffffffu, rv[0], 0, G);
    rr3[1] = __shfl_sync(0xffffffffu, rv[1], 0, G);
    rr3[2] = __shfl_sync(0xffffffffu, rv[0], 1, G);
    const double sq = sqrt(d.scal[SC_LAM]), sD[3] = {sq * Dl[0], sq * Dl[1], sq * Dl[2]};
    double g[12];
    damp64(R, sD, g);
    double M[27];  // own block: M = T^T V_o^T J_o
#pragma unroll
    for (int q = 0; q < 9; q++) {
        const double W0 = V[0][0] * jp[q] + V[1][0] * jp[9 + q], W1 = V[0][1] * jp[q] + V[1][1] * jp[9 + q],
                     W2 = V[0][2] * jp[q] + V[1][2] * jp[9 + q];
        M[q] = T00 * W0;
        M[9 + q] = T01 * W0 + T11 * W1;
        M[18 + q] = T02 * W0 + T12 * W1 + T22 * W2;
    }
    const Blk64 Bk = blk64(d, valid ? j : 0, valid ? k : 2);
    double top[27];
    for (int a = 0; a < 64; a++) {  // rows 0..2k-1 (V row a from lane a / 2), warp-uniform bound
        double va[3];
#pragma unroll
        for (int q = 0; q < 3; q++) {
            const double x0 = __shfl_sync(0xffffffffu, V[0][q], (a >> 1) % G, G);
            const double x1 = __shfl_sync(0xffffffffu, V[1][q], (a >> 1) % G, G);
            va[q] = (a & 1) ? x1 : x0;
        }
        if (a >= 2 * k || !act) continue;
        double row[9];
#pragma unroll
        for (int q = 0; q < 9; q++) {
            double x = -(va[0] * M[q] + va[1] * M[9 + q] + va[2] * M[18 + q]);
            if ((a >> 1) == gl) x += jp[9 * (a & 1) + q];
            row[q] = x;
        }
        if (a < 3) {
#pragma unroll
            for (int q = 0; q < 9; q++) top[9 * a + q] = row[q];
        } else {
#pragma unroll
            for (int q = 0; q < 9; q++) Bk.row(a)[9 * gl + q] = row[q];
        }
    }
    if (!act) return;
#pragma unroll
    for (int sr = 0; sr < 6; sr++) {
        const int row = sr < 3 ? sr : 2 * k + sr - 3;
#pragma unroll
        for (int q = 0; q < 9; q++) {
            double x[6] = {top[q], top[9 + q], top[18 + q], 0.0, 0.0, 0.0};
#pragma unroll
            for (int m = 0; m < 6; m++) {
                const int p = damp_p(m), t = damp_t(m);
                const double aa = x[p], bb = x[t];
                x[p] = g[2 * m] * aa + g[2 * m + 1] * bb;
                x[t] = -g[2 * m + 1] * aa + g[2 * m] * bb;
            }
            Bk.row(row)[9 * gl + q] = x[sr];
        }
    }
#pragma unroll
    for (int rr = 0; rr < 2; rr++) {  // landmark / residual columns of the lane's rows >= 3
        const int a = 2 * gl + rr;
        if (a >= 3) {
            double *rw = Bk.row(a) + 9 * k;
            rw[0] = rw[1] = rw[2] = 0.0;
            rw[3] = rv[rr];
        }
    }
    if (gl == 0) {
        double Xs[6][4] = {};
        for (int i = 0; i < 3; i++) {
            for (int q = 0; q < 3; q++) Xs[i][q] = R[3 * i + q];
            Xs[i][3] = rr3[i];
            Xs[3 + i][i] = sD[i];
        }
        for (int m = 0; m < 6; m++) {
            const int p = damp_p(m), t = damp_t(m);
            for (int q = 0; q < 4; q++) {
                const double aa = Xs[p][q], bb = Xs[t][q];
                Xs[p][q] = g[2 * m] * aa + g[2 * m + 1] * bb;
                Xs[t][q] = -g[2 * m + 1] * aa + g[2 * m] * bb;
            }
            Xs[t][p] = 0.0;
        }
        for (int sr = 0; sr < 6; sr++) {
            const int row = sr < 3 ? sr : 2 * k + sr - 3;
            for (int q = 0; q < 4; q++) Bk.row(row)[9 * k + q] = Xs[sr][q];
        }
        double *Gp = Bk.givens();
        for (int i = 0; i < 12; i++) Gp[i] = g[i];
        for (int q = 0; q < 3; q++) {
            d.lm_s[3 * j + q] = (float)sl[q];
            d.lm_D[3 * j + q] = (float)Dl[q];
            d.lm_s64[3 * j + q] = sl[q];
            d.lm_D64[3 * j + q] = Dl[q];
        }
    }
}

// ---- K3-64: undo the stored rotations (reverse order, transposed) and re-damp, rows {0,1,2} and
// {2k..2k+2} over all 9k + 4 columns.  Warp per landmark.
__global__ void __launch_bounds__(256) k_redamp64(DevProblem d) {
    const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (j >= d.n_l) return;
    const int k = d.lm_k[j], W = 9 * k + 4;
    const Blk64 B = blk64(d, j, k);
    double *G = B.givens();
    double g[12];
    for (int i = 0; i < 12; i++) g[i] = G[i];
    // R after undo: undo the 6 rotations on the landmark columns (+ damping diag) of rows 0..2
    double X[6][3];
    for (int s = 0; s < 6; s++) {
        const int row = s < 3 ? s : 2 * k + s - 3;
        for (int q = 0; q < 3; q++) X[s][q] = B.row(row)[9 * k + q];
    }
    for (int m = 5; m >= 0; m--) {
        const int p = damp_p(m), t = damp_t(m);
        for (int q = 0; q < 3; q++) {
            const double a = X[p][q], b = X[t][q];
            X[p][q] = g[2 * m] * a - g[2 * m + 1] * b;
            X[t][q] = g[2 * m + 1] * a + g[2 * m] * b;
        }
    }
    double R[9];
    for (int i = 0; i < 3; i++)
        for (int q = 0; q < 3; q++) R[3 * i + q] = q < i ? 0.0 : X[i][q];
    const double sq = sqrt(d.scal[SC_LAM]);
    const double sD[3] = {sq * d.lm_D64[3 * j], sq * d.lm_D64[3 * j + 1], sq * d.lm_D64[3 * j + 2]};
    double gn[12];
    damp64(R, sD, gn);
    for (int c = lane; c < W; c += 32) {
        double x[6];
        for (int s = 0; s < 6; s++) x[s] = B.row(s < 3 ? s : 2 * k + s - 3)[c];
        for (int m = 5; m >= 0; m--) {  // undo
            const int p = damp_p(m), t = damp_t(m);
            const double a = x[p], b = x[t];
            x[p] = g[2 * m] * a - g[2 * m + 1] * b;
            x[t] = g[2 * m + 1] * a + g[2 * m] * b;
        }
        for (int s = 3; s < 6; s++) x[s] = 0.0;  // damping rows dropped
        if (c >= 9 * k && c < 9 * k + 3) x[3 + (c - 9 * k)] = sD[c - 9 * k];
        for (int m = 0; m < 6; m++) {  // re-damp
            const int p = damp_p(m), t = damp_t(m);
            const double a = x[p], b = x[t];
            x[p] = gn[2 * m] * a + gn[2 * m + 1] * b;
            x[t] = -gn[2 * m + 1] * a + gn[2 * m] * b;
        }
        if (c >= 9 * k && c < 9 * k + 3) x[3 + (c - 9 * k)] = 0.0;  // eliminated exactly
        for (int s = 0; s < 6; s++) B.row(s < 3 ? s : 2 * k + s - 3)[c] = x[s];
    }
    __syncwarp();
    if (lane == 0) {
        // lower-triangle entries of R^1 exactly zero
        B.row(1)[9 * k] = 0.0, B.row(2)[9 * k] = 0.0, B.row(2)[9 * k + 1] = 0.0;
        for (int i = 0; i < 12; i++) G[i] = gn[i];
    }
}

// ---- K4-64 / K5-64 for k <= 16, TMA-staged and warp-specialized: persistent CTA (one per SM) of
// 8 consumer warps + 1 producer warp, ring of 4 stages of 48 KB.  A stage holds a batch of
// consecutive landmarks (<= 256 / G): each landmark's reduced rows 3..2k+2 (one cp.async.bulk per
// landmark, 16-byte-aligned superset), the batch's camera indices (one copy), and a table written
// by the producer {k, row-3 offset, camera offset}.  Consumers: groups of G lanes <-> landmark
// (assigned round-robin over the CTA's landmark sequence, so consecutive one-landmark stages go to
// different warps), lane <-> camera block (72-byte lane stride in shared memory), two rows per
// step with G-lane shuffle reductions; a warp releases a stage as soon as it is done with it (no
// CTA-wide barrier).  PRE: block-Jacobi blocks and b~ instead of the product.
constexpr int WS_CW = 8, WS_S = 4, WS_CAMS = 264;  // consumer warps, stages, camera slots per stage
template <int G, bool PRE>
__global__ void __launch_bounds__(32 * (WS_CW + 1), 1) k_rcs64_ws(DevProblem d, const int4 *__restrict__ batches,
                                                                  const int4 *__restrict__ brec, int nbat,
                                                                  const double *__restrict__ v,
                                                                  const PcgState *__restrict__ st) {
    if (!PRE && st && st->done) return;
    constexpr int NG = 32 * WS_CW / G, S = WS_S;
    extern __shared__ __align__(16) double sm64[];  // S x S64_STAGE_DBL
    __shared__ __align__(16) int32_t cams[S][WS_CAMS];
    __shared__ int4 tab[S][NG];  // {k, row-3 offset in the stage, camera offset, 0}
    __shared__ uint64_t full[S], empty[S];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        for (int s = 0; s < S; s++) mbar_init(&full[s], 1), mbar_init(&empty[s], WS_CW);
        fence_mbar_init();
    }
    __syncthreads();
    const int nmine = nbat > (int)blockIdx.x ? (nbat - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
    if (warp == WS_CW) {  // ---- producer: batch headers and records prefetched one batch ahead
        const uint64_t pol = policy_evict_first();
        constexpr int RL = (NG + 31) / 32;  // records per lane
        int4 h_nx = make_int4(0, 0, 0, 0), rb_nx[RL], src_nx = make_int4(0, 0, 0, 0);
        auto fetch = [&](int c) {
            const int64_t bi = blockIdx.x + (int64_t)c * gridDim.x;
            h_nx = batches[bi];
            src_nx = brec[bi * 66 + 64];
#pragma unroll
            for (int u = 0; u < RL; u++) {
                const int i = lane + 32 * u;
                rb_nx[u] = i < NG ? brec[bi * 66 + i] : make_int4(0, 0, 0, 0);
            }
        };
        if (nmine > 0) fetch(0);
        for (int c = 0; c < nmine; c++) {
            const int s = c % S;
            const int4 h = h_nx, src = src_nx;  // {n, doubles, first camera index, cameras}, {source lo}
            int4 rb[RL];
#pragma unroll
            for (int u = 0; u < RL; u++) rb[u] = rb_nx[u];
            if (c + 1 < nmine) fetch(c + 1);
            if (c >= S) mbar_wait(&empty[s], (uint32_t)(((c / S) - 1) & 1));
#pragma unroll
            for (int u = 0; u < RL; u++) {
                const int i = lane + 32 * u;
                if (i < h.x) tab[s][i] = rb[u];
            }
            __syncwarp();
            if (lane == 0) {
                const int64_t lo = (int64_t)(uint32_t)src.x | ((int64_t)src.y << 32);
                mbar_arrive_expect_tx(&full[s], 8u * (uint32_t)h.y + 4u * (uint32_t)h.w);
                bulk_g2s(cams[s], d.obs_cam + h.z, 4u * (uint32_t)h.w, &full[s]);
                bulk_g2s_stream(sm64 + (size_t)s * S64_STAGE_DBL, d.arena64 + lo, 8u * (uint32_t)h.y, &full[s], pol);
            }
        }
        return;
    }
    // ---- consumers.  A batch has at most NG landmarks, so a group owns at most one landmark per
    // stage (assigned round-robin over the CTA's landmark sequence).
    const int gl = lane % G, g = tid / G;  // my group (0 .. NG-1)
    constexpr int U = G >= 8 ? 4 : 2;      // rows per step
    int base = 0;                          // landmarks of this CTA's earlier stages
    for (int c = 0; c < nmine; c++) {
        const int s = c % S;
        const int n = batches[blockIdx.x + (int64_t)c * gridDim.x].x;  // (load issued before the wait)
        mbar_wait(&full[s], (uint32_t)((c / S) & 1));
        const int m = ((g - base) % NG + NG) % NG;
        base += n;
        const int4 e = m < n ? tab[s][m] : make_int4(0, 0, 0, 0);
        const int cam = gl < e.x ? cams[s][e.z + gl] : 0;
        double vo[9];
#pragma unroll
        for (int q = 0; q < 9; q++) vo[q] = (!PRE && gl < e.x) ? v[9 * (int64_t)cam + q] : 0.0;
        const double *stg = sm64 + (size_t)s * S64_STAGE_DBL;
        const int k = e.x, W = 9 * k + 4;
        const bool act = gl < k;
        const double *rows = stg + e.y;
        if (PRE) {
            double P[45], bb[9];
#pragma unroll
            for (int i = 0; i < 45; i++) P[i] = 0.0;
#pragma unroll
            for (int i = 0; i < 9; i++) bb[i] = 0.0;
            if (act)
                for (int r = 0; r < 2 * k; r++) {
                    const double *x = rows + r * W + 9 * gl;
                    const double qa = rows[r * W + 9 * k + 3];
                    int idx = 0;
#pragma unroll
                    for (int q1 = 0; q1 < 9; q1++) {
                        const double x1 = x[q1];
                        bb[q1] = fma(x1, qa, bb[q1]);
#pragma unroll
                        for (int q2 = q1; q2 < 9; q2++, idx++) P[idx] = fma(x1, x[q2], P[idx]);
                    }
                }
            if (act) {
                double *acc = d.pd + 54 * (int64_t)cam;
#pragma unroll
                for (int i = 0; i < 45; i++) atomicAdd(acc + i, P[i]);
#pragma unroll
                for (int i = 0; i < 9; i++) atomicAdd(acc + 45 + i, bb[i]);
            }
        } else {
            double acc[9];
#pragma unroll
            for (int q = 0; q < 9; q++) acc[q] = 0.0;
            int maxrows = 2 * k;
#pragma unroll
            for (int sh = 16; sh; sh >>= 1) maxrows = max(maxrows, __shfl_xor_sync(0xffffffffu, maxrows, sh));
            for (int r = 0; r < maxrows; r += U) {  // U rows per step
                double x[U][9], y[U];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const bool live = act && r + u < 2 * k;
                    const double *p = rows + (r + u) * W + 9 * gl;
                    y[u] = 0.0;
#pragma unroll
                    for (int q = 0; q < 9; q++) {
                        x[u][q] = live ? p[q] : 0.0;
                        y[u] = fma(x[u][q], vo[q], y[u]);
                    }
                }
#pragma unroll
                for (int sh = G / 2; sh; sh >>= 1)
#pragma unroll
                    for (int u = 0; u < U; u++) y[u] += __shfl_xor_sync(0xffffffffu, y[u], sh, G);
#pragma unroll
                for (int u = 0; u < U; u++)
#pragma unroll
                    for (int q = 0; q < 9; q++) acc[q] = fma(x[u][q], y[u], acc[q]);
            }
            if (act) {
                double *out = d.wsl64 + ((int64_t)smid() * d.n_p + cam) * 9;  // this SM's slice
#pragma unroll
                for (int q = 0; q < 9; q++) atomicAdd(out + q, acc[q]);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
}

// ---- K5-64 for k > 32, TMA-staged: CTA per item (rows [t0, t1) of the reduced rows 3..2k+2 of one
// landmark, ~1 MB).  The rows are contiguous in the row-major block, so chunks of CR rows go
// HBM -> shared memory with one cp.async.bulk each (16-byte-aligned superset; the 8-byte offset of
// odd-k rows is skipped in shared memory) through an S-stage mbarrier ring, L2 evict-first.  Thread
// <-> camera blocks o = tid + m NT: per chunk, partial dots over its 9-column segments (shared-memory
// reads at a 72-byte lane stride: conflict-free per half-warp), y_a reduced across the CTA, then
// out_o += A[a, o]^T y_a from the same staged rows.  One HBM read of A_j per product.
template <int NT, int NB>
__global__ void __launch_bounds__(NT) k_rcs64_tma(DevProblem d, const LargeItem *__restrict__ items,
                                                  const double *__restrict__ v, const PcgState *__restrict__ st,
                                                  int CRMAX, int S, int stage_dbl) {
    if (st && st->done) return;
    extern __shared__ __align__(16) double sm64[];
    uint64_t *full = reinterpret_cast<uint64_t *>(sm64 + (size_t)S * stage_dbl);
    double *part = reinterpret_cast<double *>(full + S);  // CRMAX x (NT / 32)
    const LargeItem it = items[blockIdx.x];
    const int64_t j = it.lm;
    const int k = d.lm_k[j], W = 9 * k + 4, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int CR = CRMAX;  // rows per stage (sized for the class's longest track)
    const double *B = d.arena64 + d.lm_r2[j] - 3 * (int64_t)W;  // row a at B + a W for a >= 3
    const int nrows = it.t1 - it.t0, nch = (nrows + CR - 1) / CR;
    if (tid == 0) {
        for (int s = 0; s < S; s++) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const uint64_t pol = policy_evict_first();
    auto issue = [&](int c) {  // thread 0: chunk c -> stage c % S
        const int a0 = it.t0 + c * CR, nr = min(CR, it.t1 - a0);
        const uintptr_t lo = reinterpret_cast<uintptr_t>(B + (int64_t)a0 * W) & ~(uintptr_t)15;
        const uintptr_t hi = (reinterpret_cast<uintptr_t>(B + (int64_t)(a0 + nr) * W) + 15) & ~(uintptr_t)15;
        uint64_t *bar = &full[c % S];
        mbar_arrive_expect_tx(bar, (uint32_t)(hi - lo));
        bulk_g2s_stream(sm64 + (size_t)(c % S) * stage_dbl, reinterpret_cast<const void *>(lo), (uint32_t)(hi - lo),
                        bar, pol);
    };
    if (tid == 0)
        for (int c = 0; c < min(S, nch); c++) issue(c);
    const int32_t *oc = d.obs_cam + d.lm_obs0[j];
    double acc[NB][9], vo[NB][9];
#pragma unroll
    for (int m = 0; m < NB; m++) {
        const int o = tid + m * NT;
#pragma unroll
        for (int q = 0; q < 9; q++) {
            acc[m][q] = 0.0;
            vo[m][q] = o < k ? v[9 * (int64_t)oc[o] + q] : 0.0;
        }
    }
    constexpr int NW = NT / 32;
    for (int c = 0; c < nch; c++) {
        const int s = c % S, a0 = it.t0 + c * CR, nr = min(CR, it.t1 - a0);
        mbar_wait(&full[s], (uint32_t)((c / S) & 1));
        const double *rows = sm64 + (size_t)s * stage_dbl + ((reinterpret_cast<uintptr_t>(B + (int64_t)a0 * W) >> 3) & 1);
        for (int r = 0; r < nr; r++) {
            double y = 0.0;
#pragma unroll
            for (int m = 0; m < NB; m++) {
                const int o = tid + m * NT;
                if (o < k) {
                    const double *x = rows + r * W + 9 * o;
#pragma unroll
                    for (int q = 0; q < 9; q++) y = fma(x[q], vo[m][q], y);
                }
            }
            y = warp_sum_d(y);
            if (lane == 0) part[r * NW + warp] = y;
        }
        __syncthreads();
        for (int r = 0; r < nr; r++) {
            double y = 0.0;
#pragma unroll
            for (int w = 0; w < NW; w++) y += part[r * NW + w];
#pragma unroll
            for (int m = 0; m < NB; m++) {
                const int o = tid + m * NT;
                if (o < k) {
                    const double *x = rows + r * W + 9 * o;
#pragma unroll
                    for (int q = 0; q < 9; q++) acc[m][q] = fma(x[q], y, acc[m][q]);
                }
            }
        }
        __syncthreads();  // stage s and part free
        if (tid == 0 && c + S < nch) issue(c + S);
    }
#pragma unroll
    for (int m = 0; m < NB; m++) {
        const int o = tid + m * NT;
        if (o < k) {
            double *out = d.wsl64 + ((int64_t)smid() * d.n_p + oc[o]) * 9;  // this SM's slice
#pragma unroll
            for (int q = 0; q < 9; q++) atomicAdd(out + q, acc[m][q]);
        }
    }
}

// ---- K4-64 for k > 16, TMA-staged like k_rcs64_tma: 54 FP64 accumulators per thread, so the item
// is streamed once per camera-block pass m < NB (the repeated reads of the ~1 MB item mostly hit
// L2); chunk sequence c = m nch + chunk.
template <int NT, int NB>
__global__ void __launch_bounds__(NT) k_pre64_tma(DevProblem d, const LargeItem *__restrict__ items, int CRMAX,
                                                  int S, int stage_dbl) {
    constexpr bool PRE = true;
    extern __shared__ __align__(16) double sm64[];
    uint64_t *full = reinterpret_cast<uint64_t *>(sm64 + (size_t)S * stage_dbl);
    const LargeItem it = items[blockIdx.x];
    const int64_t j = it.lm;
    const int k = d.lm_k[j], W = 9 * k + 4, tid = threadIdx.x;
    const int CR = CRMAX;  // rows per stage (sized for the class's longest track)
    const double *B = d.arena64 + d.lm_r2[j] - 3 * (int64_t)W;  // row a at B + a W for a >= 3
    const int nrows = it.t1 - it.t0, nch = (nrows + CR - 1) / CR;
    if (tid == 0) {
        for (int s = 0; s < S; s++) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const uint64_t pol = policy_evict_first();
    // PRE streams the item once per camera-block pass m < NB (54 accumulators per thread and
    // pass; the repeated reads of the ~1 MB item mostly hit L2): chunk sequence c = m nch + chunk
    const int ntot = PRE ? NB * nch : nch;
    auto issue = [&](int cc) {  // thread 0: chunk cc -> stage cc % S
        const int c = cc % nch;
        const int a0 = it.t0 + c * CR, nr = min(CR, it.t1 - a0);
        const uintptr_t lo = reinterpret_cast<uintptr_t>(B + (int64_t)a0 * W) & ~(uintptr_t)15;
        const uintptr_t hi = (reinterpret_cast<uintptr_t>(B + (int64_t)(a0 + nr) * W) + 15) & ~(uintptr_t)15;
        uint64_t *bar = &full[cc % S];
        mbar_arrive_expect_tx(bar, (uint32_t)(hi - lo));
        bulk_g2s_stream(sm64 + (size_t)(cc % S) * stage_dbl, reinterpret_cast<const void *>(lo), (uint32_t)(hi - lo),
                        bar, pol);
    };
    if (tid == 0)
        for (int c = 0; c < min(S, ntot); c++) issue(c);
    const int32_t *oc = d.obs_cam + d.lm_obs0[j];
    {
        double P[45], bb[9];
        for (int cc = 0; cc < ntot; cc++) {
            const int c = cc % nch, o = tid + (cc / nch) * NT;
            if (c == 0) {
#pragma unroll
                for (int i = 0; i < 45; i++) P[i] = 0.0;
#pragma unroll
                for (int i = 0; i < 9; i++) bb[i] = 0.0;
            }
            const int s = cc % S, a0 = it.t0 + c * CR, nr = min(CR, it.t1 - a0);
            mbar_wait(&full[s], (uint32_t)((cc / S) & 1));
            const double *rows =
                sm64 + (size_t)s * stage_dbl + ((reinterpret_cast<uintptr_t>(B + (int64_t)a0 * W) >> 3) & 1);
            if (o < k)
                for (int r = 0; r < nr; r++) {
                    const double *x = rows + r * W + 9 * o;
                    const double qa = rows[r * W + 9 * k + 3];
                    int idx = 0;
#pragma unroll
                    for (int q1 = 0; q1 < 9; q1++) {
                        const double x1 = x[q1];
                        bb[q1] = fma(x1, qa, bb[q1]);
#pragma unroll
                        for (int q2 = q1; q2 < 9; q2++, idx++) P[idx] = fma(x1, x[q2], P[idx]);
                    }
                }
            __syncthreads();
            if (tid == 0 && cc + S < ntot) issue(cc + S);
            if (c == nch - 1 && o < k) {  // end of pass: block o's sums
                double *acc = d.pd + 54 * (int64_t)oc[o];
#pragma unroll
                for (int i = 0; i < 45; i++) atomicAdd(acc + i, P[i]);
#pragma unroll
                for (int i = 0; i < 9; i++) atomicAdd(acc + 45 + i, bb[i]);
            }
        }
    }
}

// wd = sum of the per-SM FP64 product slices (32 outputs x 8 slice phases per CTA, all loads in
// flight first), zeroing them for the next product
__global__ void __launch_bounds__(256) k_reduce_slices64(DevProblem d, double *__restrict__ out,
                                                         const PcgState *__restrict__ st) {
    if (st && st->done) return;
    __shared__ double part[8][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int64_t N = 9 * d.n_p, i = (int64_t)blockIdx.x * 32 + tx;
    double s = 0.0;
    if (i < N) {
        double a[24];
#pragma unroll
        for (int u = 0; u < 24; u++) {
            const int k = ty + 8 * u;
            a[u] = k < d.nslice ? d.wsl64[k * N + i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 24; u++) {
            const int k = ty + 8 * u;
            if (k < d.nslice) d.wsl64[k * N + i] = 0.0;
        }
        for (int k = ty + 8 * 24; k < d.nslice; k += 8) {
            s += d.wsl64[k * N + i];
            d.wsl64[k * N + i] = 0.0;
        }
#pragma unroll
        for (int u = 0; u < 24; u++) s += a[u];
    }
    part[ty][tx] = s;
    __syncthreads();
    if (ty == 0 && i < N) {
        double t = 0.0;
#pragma unroll
        for (int y = 0; y < 8; y++) t += part[y][tx];
        out[i] = t;
    }
}
void launch_reduce_slices64(rba_ctx *c, double *out) {
    k_reduce_slices64<<<(unsigned)((9 * c->d.n_p + 31) / 32), 256, 0, c->stream>>>(c->d, out, nullptr);
    c->launches++;
}

// ---- K7-64: dl = -R^1^-1 (Q^1^T r^ + Q^1^T J_p dp), warp per landmark (grid-stride)
__global__ void __launch_bounds__(256) k_backsub64(DevProblem d) {
    __shared__ double red[32];
    if (d.pcg->reason == 2) return;  // indefinite attempt: no step
    const double lam = d.scal[SC_LAM];
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double q1 = 0.0, dd = 0.0;
    for (int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < d.n_l; j += nwarps) {
        const int k = d.lm_k[j], W = 9 * k + 4;
        const double *B = d.arena64 + d.lm_side[j];  // rows 0..2
        const int32_t *oc = d.obs_cam + d.lm_obs0[j];
        double s0 = 0.0, s1 = 0.0, s2 = 0.0;
        for (int c = lane; c < 9 * k; c += 32) {
            const int o = c / 9;
            const double x = d.x[9 * (int64_t)oc[o] + (c - 9 * o)];
            s0 += B[c] * x, s1 += B[W + c] * x, s2 += B[2 * W + c] * x;
        }
        s0 = warp_sum_d(s0), s1 = warp_sum_d(s1), s2 = warp_sum_d(s2);
        if (lane == 0) {
            const double *R0 = B + 9 * k, *R1 = B + W + 9 * k, *R2 = B + 2 * W + 9 * k;
            const double b0 = R0[3] + s0, b1 = R1[3] + s1, b2 = R2[3] + s2;
            const double x2 = b2 / R2[2], x1 = (b1 - R1[2] * x2) / R1[1], x0 = (b0 - R0[1] * x1 - R0[2] * x2) / R0[0];
            const double dl[3] = {-x0, -x1, -x2};
            q1 += R0[3] * R0[3] + R1[3] * R1[3] + R2[3] * R2[3];
            for (int q = 0; q < 3; q++) {
                d.dl[3 * j + q] = (float)dl[q];
                d.pts_trial[3 * j + q] = d.pts[3 * j + q] + d.lm_s64[3 * j + q] * dl[q];
                const double Dd = d.lm_D64[3 * j + q] * dl[q];
                dd += Dd * Dd;
            }
        }
    }
    q1 = block_sum_d(q1, red);
    dd = block_sum_d(dd, red);
    if (threadIdx.x == 0) {
        atomicAdd(d.scal + SC_Q1R2, q1);
        atomicAdd(d.scal + SC_DAMPL, lam * dd);
    }
}

// ============================================================================ launchers
static inline unsigned nb64(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }
__global__ void k_f2d64(const float *__restrict__ a, double *__restrict__ b, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) b[i] = a[i];
}
void launch_f2d64(rba_ctx *c, const float *a, double *b, int64_t n) {
    k_f2d64<<<nb64(n, 256), 256, 0, c->stream>>>(a, b, n);
    c->launches++;
}

template <int NT>
static void marg64_cls(rba_ctx *c, int cls) {
    const int64_t lo = c->s64_ilo[cls], hi = c->s64_ihi[cls];
    if (hi <= lo) return;
    const size_t sm = sizeof(double) * (14 * (size_t)c->s64_kmax[cls] + 288 * (NT / 32));  // SX | SR | SV | stage
    cudaFuncSetAttribute(k_marg64<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k_marg64<NT><<<(unsigned)(hi - lo), NT, sm, c->stream>>>(c->d, c->d.marg_items + lo, c->opt.diag_min,
                                                            c->opt.diag_max);
    c->launches++;
}

cudaError_t launch_marg64(rba_ctx *c) {
    Prof P(c, KID_MARG, c->marg_bytes);
    for (int g = 0; g < 4; g++) {  // k <= 32: grouped kernel by group size 4 / 8 / 16 / 32
        const int64_t lo = c->s64_mlo[g], hi = c->s64_mhi[g];
        if (hi <= lo) continue;
        const int G = 4 << g;
        const unsigned blocks = nb64((hi - lo) * G, 256);
        const double dmin = c->opt.diag_min, dmax = c->opt.diag_max;
        if (g == 0) k_marg64_small<4><<<blocks, 256, 0, c->stream>>>(c->d, lo, hi, dmin, dmax);
        else if (g == 1) k_marg64_small<8><<<blocks, 256, 0, c->stream>>>(c->d, lo, hi, dmin, dmax);
        else if (g == 2) k_marg64_small<16><<<blocks, 256, 0, c->stream>>>(c->d, lo, hi, dmin, dmax);
        else k_marg64_small<32><<<blocks, 256, 0, c->stream>>>(c->d, lo, hi, dmin, dmax);
        c->launches++;
    }
    marg64_cls<128>(c, 1);
    marg64_cls<256>(c, 2);
    marg64_cls<256>(c, 3);
    marg64_cls<256>(c, 4);
    P.end();
    return cudaGetLastError();
}

cudaError_t launch_redamp64(rba_ctx *c) {
    if (c->d.n_l == 0) return cudaSuccess;
    Prof P(c, KID_DAMP, 0.0);
    k_redamp64<<<nb64(32 * c->d.n_l, 256), 256, 0, c->stream>>>(c->d);
    c->launches++;
    P.end();
    return cudaGetLastError();
}


// TMA-staged product / block-Jacobi blocks for the rcs items [lo, hi) (tracks up to kmax): stages
// of CR rows (~32 KB, at least one row), S <= 3
template <int NT, int NB, bool PRE>
static void rcs64_tma_range(rba_ctx *c, int64_t lo, int64_t hi, int64_t kmax, const double *v, const PcgState *st) {
    if (hi <= lo) return;
    const int64_t W = 9 * kmax + 4;
    // stages of ~32 KB (at least one row of the class's longest track); S = 3 keeps 2 CTAs per SM
    // (1 CTA per SM measured 2x slower: the per-item start-up is then exposed)
    // narrow CTAs get smaller stages so that more of them fit per SM (latency hiding)
    static const int64_t tgt_env = getenv("RBA_RCS64_STAGE_DBL") ? atoll(getenv("RBA_RCS64_STAGE_DBL")) : 0;
    const int64_t tgt = tgt_env > 0 ? tgt_env : (NT >= 256 ? 4096 : (NT >= 128 ? 2048 : 1024));
    const int CRMAX = (int)std::max<int64_t>(1, tgt / W);
    const int stage_dbl = (int)((CRMAX * W + 2 + 1) & ~(int64_t)1);
    const size_t fixed = 8 * 4 + sizeof(double) * CRMAX * (NT / 32);
    int S = 3;
    while (S > 2 && sizeof(double) * S * (size_t)stage_dbl + fixed > 200 * 1024) S--;
    const size_t sm = sizeof(double) * S * (size_t)stage_dbl + fixed;
    if constexpr (PRE) {
        cudaFuncSetAttribute(k_pre64_tma<NT, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_pre64_tma<NT, NB><<<(unsigned)(hi - lo), NT, sm, c->stream>>>(c->d, c->d.rcs_items + lo, CRMAX, S, stage_dbl);
    } else {
        cudaFuncSetAttribute(k_rcs64_tma<NT, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_rcs64_tma<NT, NB><<<(unsigned)(hi - lo), NT, sm, c->stream>>>(c->d, c->d.rcs_items + lo, v, st, CRMAX, S,
                                                                        stage_dbl);
    }
    c->launches++;
}
template <int NT, int NB, bool PRE>
static void rcs64_tma_cls(rba_ctx *c, int cls, const double *v, const PcgState *st) {
    rcs64_tma_range<NT, NB, PRE>(c, c->s64_plo[cls], c->s64_phi[cls], c->s64_kmax[cls], v, st);
}
// k <= 16 by group size 4 / 8 / 16: persistent warp-specialized TMA-batch kernel
template <bool PRE>
static void rcs64_small_tma(rba_ctx *c, const double *v, const PcgState *st) {
    const size_t sm = sizeof(double) * WS_S * (size_t)S64_STAGE_DBL;
    for (int g = 0; g < 3; g++) {
        const int64_t lo = c->s64_blo[g], n = c->s64_bhi[g] - lo;
        if (n <= 0) continue;
        const unsigned grid = (unsigned)std::min<int64_t>(n, c->num_sms);
        const int4 *bp = c->d.s64_batches + lo, *rp = c->d.s64_brec + 66 * lo;
#define RBA_WS64(GG)                                                                                       \
    do {                                                                                                   \
        cudaFuncSetAttribute(k_rcs64_ws<GG, PRE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
        k_rcs64_ws<GG, PRE><<<grid, 32 * (WS_CW + 1), sm, c->stream>>>(c->d, bp, rp, (int)n, v, st);     \
    } while (0)
        if (g == 0) RBA_WS64(4);
        else if (g == 1) RBA_WS64(8);
        else RBA_WS64(16);
#undef RBA_WS64
        c->launches++;
    }
}

// wd = sum_j A_j^T A_j v: FP64 atomics into per-SM slices, summed into wd by k_reduce_slices64
void launch_rcs64(rba_ctx *c, const double *v, const PcgState *st) {
    rcs64_small_tma<false>(c, v, st);
    rcs64_tma_range<32, 1, false>(c, c->s64_glo[3], c->s64_ghi[3], 32, v, st);  // 16 < k <= 32
    rcs64_tma_cls<128, 1, false>(c, 1, v, st);
    rcs64_tma_cls<256, 1, false>(c, 2, v, st);
    rcs64_tma_cls<256, 2, false>(c, 3, v, st);
    rcs64_tma_cls<256, KMAX64 / 256, false>(c, 4, v, st);
    k_reduce_slices64<<<nb64(9 * c->d.n_p, 32), 256, 0, c->stream>>>(c->d, c->d.wd, st);
    c->launches++;
}

void launch_pre64(rba_ctx *c) {
    cudaMemsetAsync(c->d.pd, 0, sizeof(double) * 54 * c->d.n_p, c->stream);
    rcs64_small_tma<true>(c, nullptr, nullptr);
    rcs64_tma_range<32, 1, true>(c, c->s64_glo[3], c->s64_ghi[3], 32, nullptr, nullptr);
    rcs64_tma_cls<128, 1, true>(c, 1, nullptr, nullptr);
    rcs64_tma_cls<256, 1, true>(c, 2, nullptr, nullptr);
    rcs64_tma_cls<256, 2, true>(c, 3, nullptr, nullptr);
    rcs64_tma_cls<256, KMAX64 / 256, true>(c, 4, nullptr, nullptr);
}

cudaError_t launch_backsub64(rba_ctx *c) {
    if (c->d.n_l) {
        const unsigned g = (unsigned)std::min<int64_t>(nb64(32 * c->d.n_l, 256), (int64_t)c->num_sms * 8);
        k_backsub64<<<g, 256, 0, c->stream>>>(c->d);
        c->launches++;
    }
    return cudaGetLastError();
}

}  // namespace rba
