// rba_factored.cu -- factored sqrt-BA storage (beyond the paper).  The QR
// marginalization is the paper's (Householder; 6 damping Givens), but instead of
// the dense (2k+3) x (9k+4) block a landmark keeps what defines it:
//   per observation o (28 floats, 112 B):  scaled J_p rows 2o, 2o+1 (2 x 9) | Householder vectors
//       V rows 2o, 2o+1 (2 x 3) | (Q^T r^) rows 2o, 2o+1 (undamped) | pad
//   per landmark (44 floats): undamped R (3x3) | compact-WY T (6) | 6 Givens (c, s) | damped R^1
//       (3x3) | damped special residual entries (6)
// and applies A_j = (Q^^T [J_p; 0])[3:] and its transpose in O(k) (Q is never formed):
//   A v  = rows 3..2k+2 of G (Q^T u (+) 0_3),   u = J_p v,   Q^T = I - V T^T V^T
//   A^T y = J_p^T Q (G^T [0_3; y])[0:2k],       Q = I - V T V^T
// The reduced camera system is the same matrix as with dense blocks (exact algebra), read from
// (176 + 112 k) bytes per landmark instead of 72 k^2 (config 4: 0.74 GB vs 14.9 GB per product).
// Product path only (no oracle code).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "rba_internal.cuh"
#include "rba_model.cuh"

namespace rba {

// the 6 damping rotations (pivot p in {0,1,2}, target t in {d0,d1,d2}) on a 6-vector
// [top0 top1 top2 d0 d1 d2] (reading C5 / C6 order) and their inverse in reverse order
__device__ __forceinline__ int fac_p(int m) { return m == 0 ? 0 : ((m == 1 || m == 3) ? 1 : 2); }
__device__ __forceinline__ int fac_t(int m) { return m < 3 ? 3 : (m < 5 ? 4 : 5); }
__device__ __forceinline__ void givens_fwd(const float *g, float *x) {
#pragma unroll
    for (int m = 0; m < 6; m++) {
        const int p = fac_p(m), t = fac_t(m);
        const float c = g[2 * m], s = g[2 * m + 1], a = x[p], b = x[t];
        x[p] = c * a + s * b;
        x[t] = -s * a + c * b;
    }
}
__device__ __forceinline__ void givens_inv(const float *g, float *x) {
#pragma unroll
    for (int m = 5; m >= 0; m--) {
        const int p = fac_p(m), t = fac_t(m);
        const float c = g[2 * m], s = g[2 * m + 1], a = x[p], b = x[t];
        x[p] = c * a - s * b;
        x[t] = s * a + c * b;
    }
}

// a group of G lanes (G | 32) per landmark; lane gl handles observations o = gl, gl + G, ...
template <int G>
__device__ __forceinline__ float gsum(float v) {
#pragma unroll
    for (int m = G / 2; m; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m, G);
    return v;
}

struct FacHdr {
    float R[9], T[6], g[12], Rd[9], rr6[6];
};

__device__ __forceinline__ void load_hdr(const float *h, FacHdr &H) {
#pragma unroll
    for (int i = 0; i < 9; i++) H.R[i] = h[i];
#pragma unroll
    for (int i = 0; i < 6; i++) H.T[i] = h[9 + i];
#pragma unroll
    for (int i = 0; i < 12; i++) H.g[i] = h[15 + i];
#pragma unroll
    for (int i = 0; i < 9; i++) H.Rd[i] = h[27 + i];
#pragma unroll
    for (int i = 0; i < 6; i++) H.rr6[i] = h[36 + i];
}

// per-observation record: jp[18] | V[6] (rows 2o, 2o+1) | qr[2] | pad[2]
struct FacObs {
    float jp[18], v[6], qr[2];
};
__device__ __forceinline__ void load_obs(const float *rec, FacObs &o) {
    const float4 *r4 = reinterpret_cast<const float4 *>(rec);
    float t[28];
#pragma unroll
    for (int i = 0; i < 7; i++) {
        const float4 x = __ldg(r4 + i);
        t[4 * i] = x.x, t[4 * i + 1] = x.y, t[4 * i + 2] = x.z, t[4 * i + 3] = x.w;
    }
#pragma unroll
    for (int i = 0; i < 18; i++) o.jp[i] = t[i];
#pragma unroll
    for (int i = 0; i < 6; i++) o.v[i] = t[18 + i];
    o.qr[0] = t[24], o.qr[1] = t[25];
}

// Forward half for landmark j (group of G lanes): s = V^T u with u = J_p v, t = T^T s; returns
// through the group: the damped top rows top[3] and damping rows dd[3] (G (Q^T u)_special).
template <int G>
__device__ __forceinline__ void fac_forward(const float *fac, int k, const int32_t *oc, const float *vv, int gl,
                                            const FacHdr &H, float *tvec, float *top, float *dd, float *w012) {
    float s0 = 0.f, s1 = 0.f, s2 = 0.f;
    for (int o = gl; o < k; o += G) {
        FacObs ob;
        load_obs(fac + 28 * o, ob);
        const float *x = vv + 9 * (int64_t)oc[o];
        float u0 = 0.f, u1 = 0.f;
#pragma unroll
        for (int q = 0; q < 9; q++) {
            const float xq = x[q];
            u0 += ob.jp[q] * xq;
            u1 += ob.jp[9 + q] * xq;
        }
        s0 += ob.v[0] * u0 + ob.v[3] * u1;
        s1 += ob.v[1] * u0 + ob.v[4] * u1;
        s2 += ob.v[2] * u0 + ob.v[5] * u1;
    }
    s0 = gsum<G>(s0), s1 = gsum<G>(s1), s2 = gsum<G>(s2);
    // t = T^T s  (T upper: T00 T01 T02 T11 T12 T22)
    tvec[0] = H.T[0] * s0;
    tvec[1] = H.T[1] * s0 + H.T[3] * s1;
    tvec[2] = H.T[2] * s0 + H.T[4] * s1 + H.T[5] * s2;
    // rows 0, 1 (obs 0) and 2 (obs 1) of w = u - V t: every lane recomputes them (L1 hits)
    FacObs o0 = {}, o1 = {};
    float u00 = 0.f, u01 = 0.f, u10 = 0.f;
    if (k > 0) {
        load_obs(fac, o0);
        load_obs(fac + 28, o1);
        const float *x0 = vv + 9 * (int64_t)oc[0], *x1 = vv + 9 * (int64_t)oc[1];
#pragma unroll
        for (int q = 0; q < 9; q++) {
            u00 += o0.jp[q] * x0[q];
            u01 += o0.jp[9 + q] * x0[q];
            u10 += o1.jp[q] * x1[q];
        }
    }
    w012[0] = u00 - (o0.v[0] * tvec[0] + o0.v[1] * tvec[1] + o0.v[2] * tvec[2]);
    w012[1] = u01 - (o0.v[3] * tvec[0] + o0.v[4] * tvec[1] + o0.v[5] * tvec[2]);
    w012[2] = u10 - (o1.v[0] * tvec[0] + o1.v[1] * tvec[1] + o1.v[2] * tvec[2]);
    float x6[6] = {w012[0], w012[1], w012[2], 0.f, 0.f, 0.f};
    givens_fwd(H.g, x6);
    top[0] = x6[0], top[1] = x6[1], top[2] = x6[2];
    dd[0] = x6[3], dd[1] = x6[4], dd[2] = x6[5];
}

// ---- K5F: out_cam += A_j^T (A_j v) for the landmarks [lo, hi) of one group-size class
template <int G>
__global__ void __launch_bounds__(256) k_fac_matvec(DevProblem d, int64_t lo, int64_t hi, const float *__restrict__ v,
                                                    const PcgState *__restrict__ st) {
    if (st && st->done) return;
    const float *vv = v;  // camera vector: L1 / L2 resident (gathered per observation)
    const int lane = threadIdx.x & 31, gl = lane % G;
    const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;  // landmarks per grid sweep
    float *out = wslice(d);
    // warp-uniform trip count (the group shuffles need every lane of the warp): a group whose
    // landmark is past the range runs with k = 0
    const int64_t wfirst = lo + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * (32 / G);
    for (int64_t jb = wfirst; jb < hi; jb += ngroups) {
        const int64_t j = jb + lane / G;
        const bool valid = j < hi;
        const int k = valid ? d.lm_k[j] : 0;
        const float *base = d.arena + (valid ? d.lm_r2[j] : 0);
        const float *fac = base + 44;
        const int32_t *oc = d.obs_cam + (valid ? d.lm_obs0[j] : 0);
        FacHdr H;
        load_hdr(base, H);
        if (G < 32 || __all_sync(0xffffffffu, k <= G)) {
            // fast path: one observation per lane, its record, u and w kept in registers; two group
            // reductions (V^T u, V^T z) and one shuffle round for the special rows 0..2
            const bool act = gl < k;
            FacObs ob = {};
            float u0 = 0.f, u1 = 0.f;
            int cam = 0;
            if (act) {
                load_obs(fac + 28 * gl, ob);
                cam = oc[gl];
                const float *x = vv + 9 * (int64_t)cam;
#pragma unroll
                for (int q = 0; q < 9; q++) {
                    const float xq = x[q];
                    u0 += ob.jp[q] * xq;
                    u1 += ob.jp[9 + q] * xq;
                }
            }
            const float s0 = gsum<G>(ob.v[0] * u0 + ob.v[3] * u1);
            const float s1 = gsum<G>(ob.v[1] * u0 + ob.v[4] * u1);
            const float s2 = gsum<G>(ob.v[2] * u0 + ob.v[5] * u1);
            const float ta = H.T[0] * s0, tb = H.T[1] * s0 + H.T[3] * s1, tc = H.T[2] * s0 + H.T[4] * s1 + H.T[5] * s2;
            float z0 = u0 - (ob.v[0] * ta + ob.v[1] * tb + ob.v[2] * tc);
            float z1 = u1 - (ob.v[3] * ta + ob.v[4] * tb + ob.v[5] * tc);
            const int gbase = lane - gl;
            float x6[6] = {__shfl_sync(0xffffffffu, z0, gbase), __shfl_sync(0xffffffffu, z1, gbase),
                           __shfl_sync(0xffffffffu, z0, gbase + 1), 0.f, 0.f, 0.f};
            givens_fwd(H.g, x6);  // -> [top; dd]; transpose: G^T [0_3; dd]
            x6[0] = x6[1] = x6[2] = 0.f;
            givens_inv(H.g, x6);
            if (gl == 0) z0 = x6[0], z1 = x6[1];
            else if (gl == 1) z0 = x6[2];
            const float r0 = gsum<G>(ob.v[0] * z0 + ob.v[3] * z1);
            const float r1 = gsum<G>(ob.v[1] * z0 + ob.v[4] * z1);
            const float r2 = gsum<G>(ob.v[2] * z0 + ob.v[5] * z1);
            const float t0 = H.T[0] * r0 + H.T[1] * r1 + H.T[2] * r2;
            const float t1 = H.T[3] * r1 + H.T[4] * r2;
            const float t2 = H.T[5] * r2;
            if (act) {
                z0 -= ob.v[0] * t0 + ob.v[1] * t1 + ob.v[2] * t2;
                z1 -= ob.v[3] * t0 + ob.v[4] * t1 + ob.v[5] * t2;
                float acc[9];
#pragma unroll
                for (int q = 0; q < 9; q++) acc[q] = ob.jp[q] * z0 + ob.jp[9 + q] * z1;
                flush_cam12(out, cam, acc);
            }
            continue;
        }
        float t[3], top[3], dd[3], w012[3];
        fac_forward<G>(fac, k, oc, vv, gl, H, t, top, dd, w012);
        // y = rows 3..2k+2 of G(Q^T u): w rows >= 3 and dd.  Transpose: z = G^T [0_3; y] gives
        // z rows 0..2 from dd (rows >= 3 are w); then s' = V^T z, t' = T s', z' = z - V t'.
        float z6[6] = {0.f, 0.f, 0.f, dd[0], dd[1], dd[2]};
        givens_inv(H.g, z6);
        float s0 = 0.f, s1 = 0.f, s2 = 0.f;
        for (int o = gl; o < k; o += G) {
            FacObs ob;
            load_obs(fac + 28 * o, ob);
            const float *x = vv + 9 * (int64_t)oc[o];
            float u0 = 0.f, u1 = 0.f;
#pragma unroll
            for (int q = 0; q < 9; q++) {
                u0 += ob.jp[q] * x[q];
                u1 += ob.jp[9 + q] * x[q];
            }
            float z0 = u0 - (ob.v[0] * t[0] + ob.v[1] * t[1] + ob.v[2] * t[2]);
            float z1 = u1 - (ob.v[3] * t[0] + ob.v[4] * t[1] + ob.v[5] * t[2]);
            if (o == 0) z0 = z6[0], z1 = z6[1];
            else if (o == 1) z0 = z6[2];
            s0 += ob.v[0] * z0 + ob.v[3] * z1;
            s1 += ob.v[1] * z0 + ob.v[4] * z1;
            s2 += ob.v[2] * z0 + ob.v[5] * z1;
        }
        s0 = gsum<G>(s0), s1 = gsum<G>(s1), s2 = gsum<G>(s2);
        const float t0 = H.T[0] * s0 + H.T[1] * s1 + H.T[2] * s2;  // t' = T s'
        const float t1 = H.T[3] * s1 + H.T[4] * s2;
        const float t2 = H.T[5] * s2;
        for (int o = gl; o < k; o += G) {
            FacObs ob;
            load_obs(fac + 28 * o, ob);
            const int cam = oc[o];
            const float *x = vv + 9 * (int64_t)cam;
            float u0 = 0.f, u1 = 0.f;
#pragma unroll
            for (int q = 0; q < 9; q++) {
                u0 += ob.jp[q] * x[q];
                u1 += ob.jp[9 + q] * x[q];
            }
            float z0 = u0 - (ob.v[0] * t[0] + ob.v[1] * t[1] + ob.v[2] * t[2]);
            float z1 = u1 - (ob.v[3] * t[0] + ob.v[4] * t[1] + ob.v[5] * t[2]);
            if (o == 0) z0 = z6[0], z1 = z6[1];
            else if (o == 1) z0 = z6[2];
            z0 -= ob.v[0] * t0 + ob.v[1] * t1 + ob.v[2] * t2;
            z1 -= ob.v[3] * t0 + ob.v[4] * t1 + ob.v[5] * t2;
            float acc[9];
#pragma unroll
            for (int q = 0; q < 9; q++) acc[q] = ob.jp[q] * z0 + ob.jp[9 + q] * z1;
            flush_cam12(out, cam, acc);
        }
    }
}

// ---- K5F for long tracks (k > 32): CTA per landmark, thread <-> observations, the four phases
// (u = J_p v and V^T u | w = u - V T^T (V^T u) | special rows through G, V^T z | out) separated by
// CTA reductions; u / w kept in shared memory (2 floats per observation)
constexpr int FAC_NT = 256;
__device__ __forceinline__ void cta_sum3(float *v, float *red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < 3; i++) v[i] = warp_sum_f(v[i]);
    if (lane == 0)
#pragma unroll
        for (int i = 0; i < 3; i++) red[4 * warp + i] = v[i];
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 3; i++) {
        float s = 0.f;
#pragma unroll
        for (int w = 0; w < FAC_NT / 32; w++) s += red[4 * w + i];
        v[i] = s;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(FAC_NT) k_fac_matvec_cta(DevProblem d, int64_t lo, const float *__restrict__ v,
                                                          const PcgState *__restrict__ st) {
    if (st && st->done) return;
    extern __shared__ float wsm[];  // 2k
    __shared__ float red[4 * (FAC_NT / 32)];
    __shared__ float zr[3];
    const int64_t j = lo + blockIdx.x;
    const int k = d.lm_k[j], tid = threadIdx.x;
    const float *base = d.arena + d.lm_r2[j];
    const float *fac = base + 44;
    const int32_t *oc = d.obs_cam + d.lm_obs0[j];
    float T[6], g[12];
#pragma unroll
    for (int i = 0; i < 6; i++) T[i] = base[9 + i];
#pragma unroll
    for (int i = 0; i < 12; i++) g[i] = base[15 + i];
    float s[3] = {0.f, 0.f, 0.f};
    for (int o = tid; o < k; o += FAC_NT) {
        FacObs ob;
        load_obs(fac + 28 * o, ob);
        const float *x = v + 9 * (int64_t)oc[o];
        float u0 = 0.f, u1 = 0.f;
#pragma unroll
        for (int q = 0; q < 9; q++) {
            u0 += ob.jp[q] * x[q];
            u1 += ob.jp[9 + q] * x[q];
        }
        wsm[2 * o] = u0, wsm[2 * o + 1] = u1;
        s[0] += ob.v[0] * u0 + ob.v[3] * u1;
        s[1] += ob.v[1] * u0 + ob.v[4] * u1;
        s[2] += ob.v[2] * u0 + ob.v[5] * u1;
    }
    cta_sum3(s, red);
    const float ta = T[0] * s[0], tb = T[1] * s[0] + T[3] * s[1], tc = T[2] * s[0] + T[4] * s[1] + T[5] * s[2];
    float r[3] = {0.f, 0.f, 0.f};
    for (int o = tid; o < k; o += FAC_NT) {  // w = u - V t
        FacObs ob;
        load_obs(fac + 28 * o, ob);
        wsm[2 * o] -= ob.v[0] * ta + ob.v[1] * tb + ob.v[2] * tc;
        wsm[2 * o + 1] -= ob.v[3] * ta + ob.v[4] * tb + ob.v[5] * tc;
    }
    __syncthreads();
    if (tid == 0) {  // special rows: G on (w0, w1, w2; 0), then G^T on (0; dd)
        float x6[6] = {wsm[0], wsm[1], wsm[2], 0.f, 0.f, 0.f};
        givens_fwd(g, x6);
        x6[0] = x6[1] = x6[2] = 0.f;
        givens_inv(g, x6);
        zr[0] = x6[0], zr[1] = x6[1], zr[2] = x6[2];
    }
    __syncthreads();
    if (tid == 0) wsm[0] = zr[0], wsm[1] = zr[1], wsm[2] = zr[2];
    __syncthreads();
    for (int o = tid; o < k; o += FAC_NT) {  // s' = V^T z
        FacObs ob;
        load_obs(fac + 28 * o, ob);
        const float z0 = wsm[2 * o], z1 = wsm[2 * o + 1];
        r[0] += ob.v[0] * z0 + ob.v[3] * z1;
        r[1] += ob.v[1] * z0 + ob.v[4] * z1;
        r[2] += ob.v[2] * z0 + ob.v[5] * z1;
    }
    cta_sum3(r, red);
    const float t0 = T[0] * r[0] + T[1] * r[1] + T[2] * r[2], t1 = T[3] * r[1] + T[4] * r[2], t2 = T[5] * r[2];
    float *out = wslice(d);
    for (int o = tid; o < k; o += FAC_NT) {
        FacObs ob;
        load_obs(fac + 28 * o, ob);
        const float z0 = wsm[2 * o] - (ob.v[0] * t0 + ob.v[1] * t1 + ob.v[2] * t2);
        const float z1 = wsm[2 * o + 1] - (ob.v[3] * t0 + ob.v[4] * t1 + ob.v[5] * t2);
        float acc[9];
#pragma unroll
        for (int q = 0; q < 9; q++) acc[q] = ob.jp[q] * z0 + ob.jp[9 + q] * z1;
        flush_cam12(out, oc[o], acc);
    }
}

// ---- K4F: block-Jacobi blocks P_o = A[:, o]^T A[:, o] and b~_o = A[:, o]^T q from the rows of A
// given by the WY formula: A[a, o] = delta(a in {2o, 2o+1}) J_o - V[a] M_o, M_o = T^T V_o^T J_o, the
// damping rows being G-mixtures of rows 0..2.  The rows outside the observation's own two are
// -V[a] M_o, so their sums are M_o^T C_o M_o and -M_o^T e_o with C_o = sum_{a >= 3, not own}
// V[a]^T V[a] and e_o = sum V[a]^T q_a, formed as exclusive prefix + exclusive suffix sums over the
// observations (sums of non-negative parts, no subtraction); the own rows and the rows 0..2 that
// feed the damping rows exactly.  O(k) per landmark.

// C (6 upper) | e (3) contribution of one observation's rows a >= 3
__device__ __forceinline__ void fac_c9(const FacObs &ob, int o, bool act, float *c9) {
#pragma unroll
    for (int i = 0; i < 9; i++) c9[i] = 0.f;
#pragma unroll
    for (int rr = 0; rr < 2; rr++) {
        if (!act || 2 * o + rr < 3) continue;
        const float *v = ob.v + 3 * rr;
        c9[0] += v[0] * v[0], c9[1] += v[0] * v[1], c9[2] += v[0] * v[2];
        c9[3] += v[1] * v[1], c9[4] += v[1] * v[2], c9[5] += v[2] * v[2];
        c9[6] += v[0] * ob.qr[rr], c9[7] += v[1] * ob.qr[rr], c9[8] += v[2] * ob.qr[rr];
    }
}

// exclusive prefix (pre) and suffix (suf) sums of c9 over the G lanes of the group
template <int G>
__device__ __forceinline__ void fac_scans(const float *c9, int gl, float *pre, float *suf) {
#pragma unroll
    for (int i = 0; i < 9; i++) {
        const float x = __shfl_up_sync(0xffffffffu, c9[i], 1, G);
        pre[i] = gl >= 1 ? x : 0.f;
        const float y = __shfl_down_sync(0xffffffffu, c9[i], 1, G);
        suf[i] = gl + 1 < G ? y : 0.f;
    }
#pragma unroll
    for (int dlt = 1; dlt < G; dlt <<= 1) {
#pragma unroll
        for (int i = 0; i < 9; i++) {
            const float x = __shfl_up_sync(0xffffffffu, pre[i], dlt, G);
            const float y = __shfl_down_sync(0xffffffffu, suf[i], dlt, G);
            if (gl >= dlt) pre[i] += x;
            if (gl + dlt < G) suf[i] += y;
        }
    }
}

// P_o, b_o of observation o from its record, C_o | e_o (c9 layout), V rows 0..2, the header and
// the damping mixing Gm; added to the camera's slot of the SM's accumulation slice
__device__ __forceinline__ void fac_pre_obs(float *out, int cam, int o, const FacObs &ob, const float *Ce,
                                            const float *V012, const FacHdr &H, const float *Gm) {
    float C[9];
    C[0] = Ce[0], C[1] = Ce[1], C[2] = Ce[2], C[4] = Ce[3], C[5] = Ce[4], C[8] = Ce[5];
    C[3] = C[1], C[6] = C[2], C[7] = C[5];
    float M[27];
#pragma unroll
    for (int q = 0; q < 9; q++) {
        const float W0 = ob.v[0] * ob.jp[q] + ob.v[3] * ob.jp[9 + q];
        const float W1 = ob.v[1] * ob.jp[q] + ob.v[4] * ob.jp[9 + q];
        const float W2 = ob.v[2] * ob.jp[q] + ob.v[5] * ob.jp[9 + q];
        M[q] = H.T[0] * W0;
        M[9 + q] = H.T[1] * W0 + H.T[3] * W1;
        M[18 + q] = H.T[2] * W0 + H.T[4] * W1 + H.T[5] * W2;
    }
    float P[45], b[9];
    {
        float N[27];  // C M
#pragma unroll
        for (int m = 0; m < 3; m++)
#pragma unroll
            for (int q = 0; q < 9; q++) N[9 * m + q] = C[3 * m] * M[q] + C[3 * m + 1] * M[9 + q] + C[3 * m + 2] * M[18 + q];
        int idx = 0;
#pragma unroll
        for (int q1 = 0; q1 < 9; q1++) {
            b[q1] = -(M[q1] * Ce[6] + M[9 + q1] * Ce[7] + M[18 + q1] * Ce[8]);
#pragma unroll
            for (int q2 = q1; q2 < 9; q2++) P[idx++] = M[q1] * N[q2] + M[9 + q1] * N[9 + q2] + M[18 + q1] * N[18 + q2];
        }
    }
    float X3[27];  // rows 0..2 of X = Q^T E_o
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
        for (int q = 0; q < 9; q++)
            X3[9 * a + q] = -(V012[3 * a] * M[q] + V012[3 * a + 1] * M[9 + q] + V012[3 * a + 2] * M[18 + q]);
#pragma unroll
    for (int rr = 0; rr < 2; rr++) {
        const int a = 2 * o + rr;
        float row[9];
#pragma unroll
        for (int q = 0; q < 9; q++)
            row[q] = ob.jp[9 * rr + q] - (ob.v[3 * rr] * M[q] + ob.v[3 * rr + 1] * M[9 + q] + ob.v[3 * rr + 2] * M[18 + q]);
        if (a < 3) {
#pragma unroll
            for (int q = 0; q < 9; q++) X3[9 * a + q] = row[q];
        } else {
            int idx = 0;
#pragma unroll
            for (int q1 = 0; q1 < 9; q1++) {
                b[q1] += row[q1] * ob.qr[rr];
#pragma unroll
                for (int q2 = q1; q2 < 9; q2++) P[idx++] += row[q1] * row[q2];
            }
        }
    }
#pragma unroll
    for (int s2 = 3; s2 < 6; s2++) {
        float row[9];
#pragma unroll
        for (int q = 0; q < 9; q++) row[q] = Gm[3 * s2] * X3[q] + Gm[3 * s2 + 1] * X3[9 + q] + Gm[3 * s2 + 2] * X3[18 + q];
        const float qa = H.rr6[s2];
        int idx = 0;
#pragma unroll
        for (int q1 = 0; q1 < 9; q1++) {
            b[q1] += row[q1] * qa;
#pragma unroll
            for (int q2 = q1; q2 < 9; q2++) P[idx++] += row[q1] * row[q2];
        }
    }
    float4 *a4 = reinterpret_cast<float4 *>(out + PACC_STRIDE * (int64_t)cam);
#pragma unroll
    for (int i = 0; i < 11; i++) atomicAdd(a4 + i, make_float4(P[4 * i], P[4 * i + 1], P[4 * i + 2], P[4 * i + 3]));
    atomicAdd(a4 + 11, make_float4(P[44], b[0], b[1], b[2]));
    atomicAdd(a4 + 12, make_float4(b[3], b[4], b[5], b[6]));
    atomicAdd(a4 + 13, make_float4(b[7], b[8], 0.f, 0.f));
}

constexpr int FAC_MAXCH = (KMAX + 31) / 32;  // 32-observation chunks of the longest track

template <int G>
__global__ void __launch_bounds__(256) k_fac_precond(DevProblem d, int64_t lo, int64_t hi) {
    // G = 32: per-warp chunk totals / suffix carries for tracks longer than 32 (k > G path)
    extern __shared__ float chunk_sm[];
    const int lane = threadIdx.x & 31, gl = lane % G;
    const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;  // landmarks per grid sweep
    float *out = pslice(d);
    const int64_t wfirst = lo + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * (32 / G);
    for (int64_t jb = wfirst; jb < hi; jb += ngroups) {  // warp-uniform trip count
        const int64_t j = jb + lane / G;
        const bool valid = j < hi;
        const int k = valid ? d.lm_k[j] : 0;
        const float *base = d.arena + (valid ? d.lm_r2[j] : 0);
        const float *fac = base + 44;
        const int32_t *oc = d.obs_cam + (valid ? d.lm_obs0[j] : 0);
        FacHdr H;
        load_hdr(base, H);
        float Gm[18];  // the 6x3 mixing of undamped rows 0..2 into {top, d0, d1, d2}
#pragma unroll
        for (int i = 0; i < 3; i++) {
            float x6[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            x6[i] = 1.f;
            givens_fwd(H.g, x6);
#pragma unroll
            for (int s = 0; s < 6; s++) Gm[3 * s + i] = x6[s];
        }
        if (G < 32 || __all_sync(0xffffffffu, k <= G)) {  // one observation per lane
            const bool act = gl < k;
            FacObs ob = {};
            if (act) load_obs(fac + 28 * gl, ob);
            float c9[9], pre[9], suf[9];
            fac_c9(ob, gl, act, c9);
            fac_scans<G>(c9, gl, pre, suf);
            const int gbase = lane - gl;
            float V012[9];
#pragma unroll
            for (int i = 0; i < 6; i++) V012[i] = __shfl_sync(0xffffffffu, ob.v[i], gbase);
#pragma unroll
            for (int i = 0; i < 3; i++) V012[6 + i] = __shfl_sync(0xffffffffu, ob.v[i], gbase + 1);
            if (!act) continue;
#pragma unroll
            for (int i = 0; i < 9; i++) pre[i] += suf[i];
            fac_pre_obs(out, oc[gl], gl, ob, pre, V012, H, Gm);
            continue;
        }
        // G == 32, k > 32 (the whole warp is one landmark): chunks of 32 observations.  Pass 1:
        // chunk totals; suffix carries built from the last chunk backwards (additions only);
        // pass 2: in-chunk scans + prefix carry + suffix carry.
        float *tot = chunk_sm + (threadIdx.x >> 5) * (2 * 9 * FAC_MAXCH), *sc = tot + 9 * FAC_MAXCH;
        const int nch = (k + 31) / 32;
        for (int c = 0; c < nch; c++) {
            const int o = 32 * c + lane;
            FacObs ob = {};
            if (o < k) load_obs(fac + 28 * o, ob);
            float c9[9];
            fac_c9(ob, o, o < k, c9);
#pragma unroll
            for (int i = 0; i < 9; i++) {
                const float t = gsum<32>(c9[i]);
                if (lane == 0) tot[9 * c + i] = t;
            }
        }
        __syncwarp();
        if (lane < 9) {
            float acc = 0.f;
            for (int c = nch - 1; c >= 0; c--) {
                sc[9 * c + lane] = acc;
                acc += tot[9 * c + lane];
            }
        }
        __syncwarp();
        FacObs o0, o1;
        load_obs(fac, o0);
        load_obs(fac + 28, o1);
        float V012[9];
#pragma unroll
        for (int i = 0; i < 6; i++) V012[i] = o0.v[i];
#pragma unroll
        for (int i = 0; i < 3; i++) V012[6 + i] = o1.v[i];
        float pc[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (int c = 0; c < nch; c++) {
            const int o = 32 * c + lane;
            const bool act = o < k;
            FacObs ob = {};
            if (act) load_obs(fac + 28 * o, ob);
            float c9[9], pre[9], suf[9];
            fac_c9(ob, o, act, c9);
            fac_scans<32>(c9, lane, pre, suf);
#pragma unroll
            for (int i = 0; i < 9; i++) {
                pre[i] += pc[i] + (suf[i] + sc[9 * c + i]);
                pc[i] += tot[9 * c + i];
            }
            if (act) fac_pre_obs(out, oc[o], o, ob, pre, V012, H, Gm);
        }
        __syncwarp();
    }
}

// ---- K7F: dl = -R^1^-1 (Q^1^T r^ + (Q^^T [J_p dp; 0])[0:3]) and the C10 terms
template <int G>
__global__ void __launch_bounds__(256) k_fac_backsub(DevProblem d, int64_t lo, int64_t hi) {
    __shared__ double red[32];
    if (d.pcg->reason == 2) return;  // indefinite attempt: no step
    const int lane = threadIdx.x & 31, gl = lane % G;
    const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;  // landmarks per grid sweep
    double q1 = 0.0, dd2 = 0.0;
    // dp (FP64, 9 n_p) rounded to FP32 per use
    // warp-uniform trip count (the group shuffles need every lane of the warp): a group whose
    // landmark is past the range runs with k = 0
    const int64_t wfirst = lo + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * (32 / G);
    for (int64_t jb = wfirst; jb < hi; jb += ngroups) {
        const int64_t j = jb + lane / G;
        const bool valid = j < hi;
        const int k = valid ? d.lm_k[j] : 0;
        const float *base = d.arena + (valid ? d.lm_r2[j] : 0);
        const float *fac = base + 44;
        const int32_t *oc = d.obs_cam + (valid ? d.lm_obs0[j] : 0);
        FacHdr H;
        load_hdr(base, H);
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, u00 = 0.f, u01 = 0.f, u10 = 0.f;
        for (int o = gl; o < k; o += G) {
            FacObs ob;
            load_obs(fac + 28 * o, ob);
            const double *x = d.x + 9 * (int64_t)oc[o];
            float u0 = 0.f, u1 = 0.f;
#pragma unroll
            for (int q = 0; q < 9; q++) {
                const float xq = (float)x[q];
                u0 += ob.jp[q] * xq;
                u1 += ob.jp[9 + q] * xq;
            }
            if (o == 0) u00 = u0, u01 = u1;
            if (o == 1) u10 = u0;
            s0 += ob.v[0] * u0 + ob.v[3] * u1;
            s1 += ob.v[1] * u0 + ob.v[4] * u1;
            s2 += ob.v[2] * u0 + ob.v[5] * u1;
        }
        s0 = gsum<G>(s0), s1 = gsum<G>(s1), s2 = gsum<G>(s2);
        u00 = gsum<G>(u00), u01 = gsum<G>(u01), u10 = gsum<G>(u10);  // only one lane holds each
        if (gl == 0 && valid) {
            const float t0 = H.T[0] * s0, t1 = H.T[1] * s0 + H.T[3] * s1, t2 = H.T[2] * s0 + H.T[4] * s1 + H.T[5] * s2;
            FacObs o0, o1;
            load_obs(fac, o0);
            load_obs(fac + 28, o1);
            float x6[6] = {u00 - (o0.v[0] * t0 + o0.v[1] * t1 + o0.v[2] * t2),
                           u01 - (o0.v[3] * t0 + o0.v[4] * t1 + o0.v[5] * t2),
                           u10 - (o1.v[0] * t0 + o1.v[1] * t1 + o1.v[2] * t2), 0.f, 0.f, 0.f};
            givens_fwd(H.g, x6);
            const float b0 = H.rr6[0] + x6[0], b1 = H.rr6[1] + x6[1], b2 = H.rr6[2] + x6[2];
            const float *R = H.Rd;  // damped R^1, upper triangular rows
            const float x2 = b2 / R[8];
            const float x1 = (b1 - R[5] * x2) / R[4];
            const float x0 = (b0 - R[1] * x1 - R[2] * x2) / R[0];
            const float dl[3] = {-x0, -x1, -x2};
            q1 += (double)H.rr6[0] * H.rr6[0] + (double)H.rr6[1] * H.rr6[1] + (double)H.rr6[2] * H.rr6[2];
#pragma unroll
            for (int q = 0; q < 3; q++) {
                d.dl[3 * j + q] = dl[q];
                d.pts_trial[3 * j + q] = d.pts[3 * j + q] + (double)(d.lm_s[3 * j + q] * dl[q]);
                const double Dd = (double)d.lm_D[3 * j + q] * dl[q];
                dd2 += Dd * Dd;
            }
        }
    }
    q1 = block_sum_d(q1, red);
    dd2 = block_sum_d(dd2, red);
    if (threadIdx.x == 0) {
        atomicAdd(d.scal + SC_Q1R2, q1);
        atomicAdd(d.scal + SC_DAMPL, d.scal[SC_LAM] * dd2);
    }
}

// ---- K3F: re-damping is O(1) per landmark: new Givens from the undamped R and Q1^T r
__global__ void k_fac_redamp(DevProblem d) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= d.n_l) return;
    const int k = d.lm_k[j];
    float *base = d.arena + d.lm_r2[j];
    const float *fac = base + 44;
    float R[9], rr3[3];
#pragma unroll
    for (int i = 0; i < 9; i++) R[i] = base[i];
    rr3[0] = fac[24], rr3[1] = fac[25], rr3[2] = fac[28 + 24];
    (void)k;
    const float sq = sqrtf((float)d.scal[SC_LAM]);
    const float sD[3] = {sq * d.lm_D[3 * j], sq * d.lm_D[3 * j + 1], sq * d.lm_D[3 * j + 2]};
    float L6[18], Gm[18], rr6[6], g[12];
    damp_rotations(R, rr3, sD, L6, Gm, rr6, g);
#pragma unroll
    for (int i = 0; i < 12; i++) base[15 + i] = g[i];
#pragma unroll
    for (int i = 0; i < 9; i++) base[27 + i] = L6[i];
#pragma unroll
    for (int i = 0; i < 6; i++) base[36 + i] = rr6[i];
}

// ============================================================================ launchers
static inline unsigned nbk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

template <int G>
static void fac_cls(rba_ctx *c, int cls, int what, const float *v, const PcgState *st, cudaStream_t s) {
    const int64_t lo = c->fac_lo[cls], hi = c->fac_hi[cls];
    if (hi <= lo) return;
    const unsigned g = (unsigned)std::min<int64_t>(nbk((hi - lo) * G, 256), (int64_t)c->num_sms * 8);
    if (what == 0) {
        const int64_t hw = G == 32 ? std::min(hi, std::max(lo, c->fac_big)) : hi;  // warp path up to k = 32
        if (hw > lo) {
            const unsigned gw = (unsigned)std::min<int64_t>(nbk((hw - lo) * G, 256), (int64_t)c->num_sms * 8);
            k_fac_matvec<G><<<gw, 256, 0, s>>>(c->d, lo, hw, v, st);
        }
        if (G == 32 && hi > hw) {
            c->launches++;
            const size_t sm = sizeof(float) * 2 * (size_t)c->max_large_k;
            cudaFuncSetAttribute(k_fac_matvec_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(sm, 16));
            k_fac_matvec_cta<<<(unsigned)(hi - hw), FAC_NT, sm, s>>>(c->d, hw, v, st);
        }
    } else if (what == 1) {
        const size_t sm = G == 32 ? sizeof(float) * 8 * 2 * 9 * FAC_MAXCH : 0;
        if (G == 32) cudaFuncSetAttribute(k_fac_precond<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_fac_precond<G><<<g, 256, sm, s>>>(c->d, lo, hi);
    } else {
        k_fac_backsub<G><<<g, 256, 0, s>>>(c->d, lo, hi);
    }
    c->launches++;
}

static void fac_all(rba_ctx *c, int what, const float *v, const PcgState *st) {
    // the classes are independent: fork them over the auxiliary streams and join back
    cudaEventRecord(c->ev_fork, c->stream);
    for (int i = 0; i < rba_ctx::NAUX; i++) cudaStreamWaitEvent(c->aux[i], c->ev_fork, 0);
    fac_cls<32>(c, 4, what, v, st, c->stream);
    fac_cls<16>(c, 3, what, v, st, c->aux[0]);
    fac_cls<8>(c, 2, what, v, st, c->aux[1]);
    fac_cls<4>(c, 1, what, v, st, c->aux[2]);
    fac_cls<2>(c, 0, what, v, st, c->stream);
    for (int i = 0; i < rba_ctx::NAUX; i++) {
        cudaEventRecord(c->ev_join[i], c->aux[i]);
        cudaStreamWaitEvent(c->stream, c->ev_join[i], 0);
    }
}

void launch_fac_matvec(rba_ctx *c, const float *v, const PcgState *st) { fac_all(c, 0, v, st); }
void launch_fac_precond(rba_ctx *c) { fac_all(c, 1, nullptr, nullptr); }
cudaError_t launch_fac_backsub(rba_ctx *c) {
    fac_all(c, 2, nullptr, nullptr);
    return cudaGetLastError();
}
cudaError_t launch_fac_redamp(rba_ctx *c) {
    if (c->d.n_l) {
        k_fac_redamp<<<nbk(c->d.n_l, 256), 256, 0, c->stream>>>(c->d);
        c->launches++;
    }
    return cudaGetLastError();
}

}  // namespace rba
