// rba_model.cuh -- device helpers shared by the sqrt-BA kernels (rba_kernels.cu) and the
// explicit-Schur-complement baseline (rba_sc.cu): the camera model, the robust loss, warp / block
// reductions and the per-SM accumulation slices.  Product path only (no oracle code).
#pragma once
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "rba_internal.cuh"

namespace rba {

// ============================================================================ camera model
// BAL / Snavely (readings C1, C2, C22): P = R(w) X + t, p = -P_xy / P_z,
// d = 1 + k1 |p|^2 + k2 |p|^4, pi = f d p, r = pi - u.  Jacobians for the additive update of all
// 9 camera parameters: dP/dw = -[R X]_x J_left(w), R = I + a K + b K^2, J_left = I + b K + c K^2
// (a = sin th / th, b = (1 - cos th) / th^2, c = (th - sin th) / th^3; series below th = 1e-8 /
// 1e-2).  Evaluated in FP64 from the FP64 state (reading C23): residuals in FP64,
// the Jacobians rounded to JT on output (FP32 for sqrt-BA-32 and explicit-32, FP64 for sqrt-BA-64
// and explicit-64).
// Per-camera precomputation (once per state, k_cam_prep): R(w) and J_left(w) as 3x3 matrices plus
// t, f, k1, k2 -- 24 doubles -- so the per-observation model needs no trigonometry or divisions
// beyond 1/P_z.
__device__ __forceinline__ void cam_prep(const double *__restrict__ cam, double *pre) {
    const double w0 = cam[0], w1 = cam[1], w2 = cam[2];
    const double th2 = w0 * w0 + w1 * w1 + w2 * w2;
    double a, b, cc;
    if (th2 < 1e-16) {
        a = 1. - th2 * (1. / 6.);
        b = 0.5 - th2 * (1. / 24.);
        cc = 1. / 6. - th2 * (1. / 120.);
    } else {
        const double th = sqrt(th2);
        double s, co;
        sincos(th, &s, &co);
        a = s / th;
        const double hs = sin(0.5 * th);
        b = 2. * hs * hs / th2;
        cc = (th < 1e-2) ? (1.0 / 6.0 - th2 * (1.0 / 120.0) + th2 * th2 * (1.0 / 5040.0)) : (th - s) / (th2 * th);
    }
    const double rd = 1. - b * th2, jd = 1. - cc * th2;
    pre[0] = rd + b * w0 * w0, pre[1] = -a * w2 + b * w0 * w1, pre[2] = a * w1 + b * w0 * w2;
    pre[3] = a * w2 + b * w0 * w1, pre[4] = rd + b * w1 * w1, pre[5] = -a * w0 + b * w1 * w2;
    pre[6] = -a * w1 + b * w0 * w2, pre[7] = a * w0 + b * w1 * w2, pre[8] = rd + b * w2 * w2;
    pre[9] = jd + cc * w0 * w0, pre[10] = -b * w2 + cc * w0 * w1, pre[11] = b * w1 + cc * w0 * w2;
    pre[12] = b * w2 + cc * w0 * w1, pre[13] = jd + cc * w1 * w1, pre[14] = -b * w0 + cc * w1 * w2;
    pre[15] = -b * w1 + cc * w0 * w2, pre[16] = b * w0 + cc * w1 * w2, pre[17] = jd + cc * w2 * w2;
    for (int i = 0; i < 6; i++) pre[18 + i] = cam[3 + i];
}

__device__ __forceinline__ void load_pre(const double *__restrict__ campre, int cam, double *c) {
    const double2 *p2 = reinterpret_cast<const double2 *>(campre + CAMPRE * (int64_t)cam);
#pragma unroll
    for (int i = 0; i < CAMPRE / 2; i++) {
        const double2 x = __ldg(p2 + i);
        c[2 * i] = x.x, c[2 * i + 1] = x.y;
    }
}

template <typename JT = float>
__device__ __forceinline__ double cam_model_pre(const double *__restrict__ c, double X0, double X1, double X2,
                                                double u, double v, double *r, JT *Jc, JT *Jl) {
    const double *R = c, *L = c + 9;
    const double RX0 = R[0] * X0 + R[1] * X1 + R[2] * X2;
    const double RX1 = R[3] * X0 + R[4] * X1 + R[5] * X2;
    const double RX2 = R[6] * X0 + R[7] * X1 + R[8] * X2;
    const double P0 = RX0 + c[18], P1 = RX1 + c[19], P2 = RX2 + c[20];
    const double iz = -1. / P2;
    const double px = P0 * iz, py = P1 * iz;
    const double n = px * px + py * py;
    const double f = c[21], k1 = c[22], k2 = c[23];
    const double dd = 1. + k1 * n + k2 * n * n;
    r[0] = f * dd * px - u;
    r[1] = f * dd * py - v;
    if (!Jc) return P2;
    const double e = 2. * (k1 + 2. * k2 * n);
    const double D00 = f * (dd + e * px * px), D01 = f * e * px * py, D11 = f * (dd + e * py * py);
    const double A00 = iz * D00, A01 = iz * D01, A02 = iz * (D00 * px + D01 * py);
    const double A10 = iz * D01, A11 = iz * D11, A12 = iz * (D01 * px + D11 * py);
#pragma unroll
    for (int q = 0; q < 3; q++) {
        Jl[q] = (JT)(A00 * R[q] + A01 * R[3 + q] + A02 * R[6 + q]);
        Jl[3 + q] = (JT)(A10 * R[q] + A11 * R[3 + q] + A12 * R[6 + q]);
    }
    const double B00 = A01 * RX2 - A02 * RX1, B01 = -A00 * RX2 + A02 * RX0, B02 = A00 * RX1 - A01 * RX0;
    const double B10 = A11 * RX2 - A12 * RX1, B11 = -A10 * RX2 + A12 * RX0, B12 = A10 * RX1 - A11 * RX0;
#pragma unroll
    for (int q = 0; q < 3; q++) {
        Jc[q] = (JT)(-(B00 * L[q] + B01 * L[3 + q] + B02 * L[6 + q]));
        Jc[9 + q] = (JT)(-(B10 * L[q] + B11 * L[3 + q] + B12 * L[6 + q]));
    }
    Jc[3] = (JT)A00; Jc[4] = (JT)A01; Jc[5] = (JT)A02;
    Jc[12] = (JT)A10; Jc[13] = (JT)A11; Jc[14] = (JT)A12;
    Jc[6] = (JT)(dd * px); Jc[7] = (JT)(f * n * px); Jc[8] = (JT)(f * n * n * px);
    Jc[15] = (JT)(dd * py); Jc[16] = (JT)(f * n * py); Jc[17] = (JT)(f * n * n * py);
    return P2;
}

// Huber norm on s = |r|^2 and its IRLS weight sqrt(rho'(s)) (Ceres' corrector with
// rho'' = 0); delta <= 0: squared loss.
__device__ __forceinline__ double robust_rho(double s, double delta) {
    return (delta <= 0.0 || s <= delta * delta) ? s : 2.0 * delta * sqrt(s) - delta * delta;
}
__device__ __forceinline__ double robust_w(double s, double delta) {
    return (delta <= 0.0 || s <= delta * delta) ? 1.0 : sqrt(delta / sqrt(s));
}
// weight the residual and the Jacobian rows of one observation (IRLS)
template <typename JT>
__device__ __forceinline__ void apply_irls(double *r, JT *Jc, JT *Jl, double delta) {
    if (delta <= 0.0) return;
    const double w = robust_w(r[0] * r[0] + r[1] * r[1], delta);
    const JT wf = (JT)w;
    r[0] *= w;
    r[1] *= w;
#pragma unroll
    for (int i = 0; i < 18; i++) Jc[i] *= wf;
#pragma unroll
    for (int i = 0; i < 6; i++) Jl[i] *= wf;
}


// ============================================================================ reductions
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int m = 16; m; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
    return v;
}
__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
    for (int m = 16; m; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
    return v;
}
template <int G>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
    for (int m = G / 2; m; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m, G);
    return v;
}
// block-wide sum of NV floats; every thread gets the result.  scratch: >= 32*NV floats.
template <int NV>
__device__ __forceinline__ void block_sum(float *v, float *scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int i = 0; i < NV; i++) v[i] = warp_sum_f(v[i]);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int i = 0; i < NV; i++) scratch[i * 32 + warp] = v[i];
    __syncthreads();
#pragma unroll
    for (int i = 0; i < NV; i++) {
        float s = 0.f;
        for (int w = 0; w < nw; w++) s += scratch[i * 32 + w];
        v[i] = s;
    }
    __syncthreads();
}
__device__ __forceinline__ double block_sum_d(double v, double *scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum_d(v);
    __syncthreads();
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < nw; w++) s += scratch[w];
    __syncthreads();
    return s;
}

// Camera-space partial sums of K4/K5 (matvec output, block-Jacobi blocks, b~) are accumulated in
// FP32 into the slice of the SM that runs the thread and summed across slices in FP64 by
// k_reduce_slices (reading C24): a single FP32 accumulator per camera summed the
// contributions of thousands of landmarks in one chain, and its cancellation error was amplified by
// PCG into a 1e-3 change of the solution.
__device__ __forceinline__ unsigned smid() {
    unsigned r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}
__device__ __forceinline__ float *wslice(const DevProblem &d) { return d.wsl + (int64_t)smid() * 12 * d.n_p; }
__device__ __forceinline__ float *pslice(const DevProblem &d) {
    return d.psl + (int64_t)smid() * PACC_STRIDE * d.n_p;
}

// out12: camera stride 12 so the 9 entries of a camera go out as three 16-byte vector atomics
__device__ __forceinline__ void flush_cam12(float *out12, int cam, const float *acc) {
    float4 *o4 = reinterpret_cast<float4 *>(out12 + 12 * (int64_t)cam);
    atomicAdd(o4, make_float4(acc[0], acc[1], acc[2], acc[3]));
    atomicAdd(o4 + 1, make_float4(acc[4], acc[5], acc[6], acc[7]));
    atomicAdd(o4 + 2, make_float4(acc[8], 0.f, 0.f, 0.f));
}

// ============================================================================ damping rotations
// 6 Givens rotations (pivot, target) = (0,d0),(1,d0),(2,d0),(1,d1),(2,d1),(2,d2) fold sqrt(lam) D_l
// into R1 (Fig. 3b).  Reading C5: c = a/rho, s = b/rho, new_p = c p + s t,
// new_t = -s p + c t; b == 0 -> identity.  In:  R (3x3 upper, row-major), rr[0..2] residual of
// rows 0..2, sD[3] = sqrt(lam) D_l.  Out: L6 rows 0..2 = damped R1 (rows 3..5 end up exactly 0),
// Gm (6x3) maps undamped rows 0..2 to the damped rows {0,1,2,d0,d1,d2} in the pose / residual
// columns, rr6 the damped residual entries, g[12] the (c, s) pairs.
__host__ __device__ constexpr int damp_p(int m) { return m == 0 ? 0 : ((m == 1 || m == 3) ? 1 : 2); }
__host__ __device__ constexpr int damp_t(int m) { return m < 3 ? 3 : (m < 5 ? 4 : 5); }

__device__ __forceinline__ void givens(float a, float b, float &c, float &s) {
    if (b == 0.f) {
        c = 1.f;
        s = 0.f;
    } else {
        // 1/rho by the reciprocal square root (a few instructions; hypotf + two IEEE divisions were
        // ~10% of the small-k K2's instructions), hypotf where a^2 + b^2 leaves the normal range
        const float r2 = fmaf(a, a, b * b);
        if (r2 > 1e-30f && r2 < 1e30f) {
            const float ri = rsqrtf(r2);
            c = a * ri;
            s = b * ri;
        } else {
            const float r = hypotf(a, b);
            c = a / r;
            s = b / r;
        }
    }
}

__device__ __forceinline__ void damp_rotations(const float *R, const float *rr, const float *sD, float *L6, float *Gm,
                                               float *rr6, float *g) {
#pragma unroll
    for (int i = 0; i < 18; i++) L6[i] = 0.f, Gm[i] = 0.f;
#pragma unroll
    for (int i = 0; i < 9; i++) L6[i] = R[i];
#pragma unroll
    for (int i = 0; i < 3; i++) {
        L6[(3 + i) * 3 + i] = sD[i];
        Gm[i * 3 + i] = 1.f;
        rr6[i] = rr[i];
        rr6[3 + i] = 0.f;
    }
#pragma unroll
    for (int m = 0; m < 6; m++) {
        const int p = damp_p(m), t = damp_t(m);
        float c, s;
        givens(L6[p * 3 + p], L6[t * 3 + p], c, s);
        g[2 * m] = c;
        g[2 * m + 1] = s;
#pragma unroll
        for (int q = 0; q < 3; q++) {
            float a = L6[p * 3 + q], b = L6[t * 3 + q];
            L6[p * 3 + q] = c * a + s * b;
            L6[t * 3 + q] = -s * a + c * b;
            a = Gm[p * 3 + q], b = Gm[t * 3 + q];
            Gm[p * 3 + q] = c * a + s * b;
            Gm[t * 3 + q] = -s * a + c * b;
        }
        float a = rr6[p], b = rr6[t];
        rr6[p] = c * a + s * b;
        rr6[t] = -s * a + c * b;
        L6[t * 3 + p] = 0.f;
    }
}

// ---- TMA bulk copies (cp.async.bulk + mbarrier) for the streaming pipelines
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// streaming variant for the landmark blocks: L2 evict-first, so the read-once R2 stream does not
// evict the L2-resident camera vectors and per-SM accumulation slices
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void bulk_g2s_stream(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                                uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// TMA prefetch of a global range into L2 (no shared memory, no completion tracking)
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// shared -> global bulk store (TMA), its commit and the wait until the shared source was read
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit_wait_read() {
    asm volatile("cp.async.bulk.commit_group;\n\tcp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// wait until the committed bulk stores have completed, i.e. their global writes are performed (a
// kernel that exits after bulk_wait_read() alone can leave writes in flight that a following kernel
// then reads stale)
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

}  // namespace rba
