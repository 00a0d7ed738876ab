// rba_lm.cu -- the device-side Levenberg-Marquardt loop of librba (readings C9, C10, C13)
// and the CUDA graphs that run it without host round trips.  Product path only (no oracle code).
//
// The LM schedule (lambda, nu, E at the current state, the accept decision) lives in device memory
// (rba::LmDev) and is advanced by k_lm_control after each attempt; every kernel that needs lambda
// reads it from scal[SC_LAM].  One LM attempt is
//
//     k_lm_begin                      lambda of this attempt -> scal, zero the scalar sums
//     if (need_lin) { K1 linearize (+ all-reduce of the camera norms), K2 marginalize + damp }
//     else          { K3 re-damp the blocks of the previous linearization (backtracking) }
//     K4 block-Jacobi + b~ (+ all-reduce), k_pcg_init
//     while (PCG not done) { K5 product (+ all-reduce), K6 update }
//     K7 back-substitution, K8 trial cost (+ all-reduce of the 4 trial scalars)
//     k_lm_control                    gain ratio, accept / reject, lambda / nu update, report
//     k_lm_commit                     x <- x + dx if accepted
//
// On a single GPU the whole loop `while (attempts < target && !converged) { attempt }` is one CUDA
// graph with conditional nodes (if / else for relinearize vs re-damp, while for PCG and for LM), so
// rba_lm_step / rba_lm_solve synchronize only to copy the reports.  Where a graph cannot be used
// (RBA_NO_GRAPH, instantiation failure, e.g. NCCL inside conditional bodies, or the k > 512
// product whose fused kernel runs slower inside graph branches) the same sequence is issued
// eagerly and only the PCG loop polls its done flag from the host.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "rba_internal.cuh"

namespace rba {

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// ============================================================================ kernels
__global__ void k_set_lambda(DevProblem d, double lam) { d.scal[SC_LAM] = lam; }

__global__ void k_set_pcg_limits(DevProblem d, double tol, int max_iters) {
    d.pcg->tol = tol;
    d.pcg->max_iters = max_iters;
}

__global__ void k_lm_init(DevProblem d, double lam, double nu, double mrd, int reset_iter) {
    LmDev *L = d.lm;
    L->lambda = lam;
    L->nu = nu;
    L->min_rel_decrease = mrd;
    if (reset_iter) L->iter = 0;
    L->rep_cap = rba_ctx::REP_CAP;
}

__global__ void k_lm_need_lin(DevProblem d) { d.lm->need_lin = 1; }

__global__ void k_stamp(DevProblem d, int slot) { d.lm->ts[slot] = globaltimer(); }

// start of rba_lm_step / rba_lm_solve (issued before the graph): attempts to run, tolerance
__global__ void k_lm_request(DevProblem d, int64_t target, double ftol) {
    LmDev *L = d.lm;
    L->target = target;
    L->n_done = 0;
    L->stop = 0;
    L->ftol = ftol;
}
// first node of the LM graph: the loop condition
__global__ void k_lm_loop_begin(DevProblem d, cudaGraphConditionalHandle h) {
    cudaGraphSetConditional(h, (d.lm->n_done < d.lm->target && d.lm->stop == 0) ? 1 : 0);
}

// start of one attempt: lambda -> scal[SC_LAM]; zero the scalar sums of this attempt; choose the branch
__global__ void k_lm_begin(DevProblem d, cudaGraphConditionalHandle h, int use_h) {
    LmDev *L = d.lm;
    const unsigned long long t = globaltimer();
    L->ts[TS_BEGIN] = t;
    L->ts[TS_LIN] = t;
    d.scal[SC_LAM] = L->lambda;
    L->lin_now = L->need_lin;
    L->accepted_now = 0;
    if (L->need_lin) d.scal[SC_E] = 0.0, d.scal[SC_BAD] = 0.0;
    d.scal[SC_ET] = d.scal[SC_BADT] = d.scal[SC_Q1R2] = d.scal[SC_DAMPL] = d.scal[SC_MODELP] = 0.0;
    d.scal[SC_NSPD] = 0.0;
    if (use_h) cudaGraphSetConditional(h, L->need_lin ? 1 : 0);
}

// after K1 (and its all-reduce): E at the new linearization point; a point behind a camera or a
// non-finite E at the current state is an error (the loop stops, the host reports it)
__global__ void k_lin_done(DevProblem d) {
    LmDev *L = d.lm;
    L->ts[TS_LIN] = globaltimer();
    const double E = d.scal[SC_E];
    L->cost = E;
    L->need_lin = 0;
    if (d.scal[SC_BAD] > 0.0 || !isfinite(E)) L->stop = 2;
}

// after the trial cost: gain ratio (C10), accept iff rho > min_rel_decrease (C9), lambda / nu
// update, clamp [1e-16, 1e16]; report; LM loop condition
__global__ void k_lm_control(DevProblem d, cudaGraphConditionalHandle h, int use_h) {
    LmDev *L = d.lm;
    const PcgState *st = d.pcg;
    const double *s = d.scal;
    const unsigned long long t_end = globaltimer();
    L->ts[TS_END] = t_end;
    rba_lm_report R;
    memset(&R, 0, sizeof(R));
    R.iter = L->iter;
    R.lambda = L->lambda;
    R.cost = L->cost;
    R.pcg_iters = st->it;
    R.pcg_reason = st->reason;
    R.relinearized = L->lin_now;
    R.cost_trial = INFINITY;
    const bool indefinite = st->reason == 2;
    bool accept = false;
    int status = L->stop == 2 ? 2 : 0;
    if (!indefinite && status != 2) {
        const double Et = s[SC_BADT] > 0.0 ? INFINITY : s[SC_ET];
        const double model = s[SC_Q1R2] + s[SC_DAMPL] + s[SC_MODELP];
        const double rho = (L->cost - Et) / model;
        R.cost_trial = Et;
        R.model = model;
        R.rho = rho;
        accept = model > 0.0 && isfinite(Et) && rho > L->min_rel_decrease;
        if (accept) {
            const double E0 = L->cost;
            L->cost = Et;
            const double tt = 2.0 * rho - 1.0;
            L->lambda *= fmax(1.0 / 3.0, 1.0 - tt * tt * tt);
            L->nu = 2.0;
            L->need_lin = 1;
            // "terminating early if a relative function tolerance of 1e-6 is reached"
            if (L->ftol > 0.0 && (E0 - Et) < L->ftol * E0) status = 1;
        }
    }
    if (!accept) {
        L->lambda *= L->nu;
        L->nu *= 2.0;
    }
    L->lambda = fmin(fmax(L->lambda, 1e-16), 1e16);
    L->accepted_now = accept ? 1 : 0;
    R.accepted = accept ? 1 : 0;
    R.cost_after = L->cost;
    R.lambda_next = L->lambda;
    R.status = status;
    const unsigned long long *ts = L->ts;
    auto ms = [](unsigned long long a, unsigned long long b) { return b > a ? (double)(b - a) * 1e-6 : 0.0; };
    R.t_linearize_ms = ms(ts[TS_BEGIN], ts[TS_LIN]);
    R.t_marginalize_ms = ms(ts[TS_LIN], ts[TS_MARG]);
    R.t_precond_ms = ms(ts[TS_MARG], ts[TS_PRE]);
    R.t_pcg_ms = ms(ts[TS_PRE], ts[TS_PCG]);
    R.t_trial_ms = ms(ts[TS_PCG], ts[TS_TRIAL]);
    R.t_total_ms = ms(ts[TS_BEGIN], t_end);
    if (L->n_done < L->rep_cap) d.reps[L->n_done] = R;
    L->n_done++;
    L->iter++;
    if (status) L->stop = status;
    if (use_h) cudaGraphSetConditional(h, (L->n_done < L->target && L->stop == 0) ? 1 : 0);
}

// x <- x + dx (the trial state) if the attempt was accepted
__global__ void k_lm_commit(DevProblem d) {
    if (!d.lm->accepted_now) return;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 9 * d.n_p + 3 * d.n_l; i += stride) {
        if (i < 9 * d.n_p) d.cams[i] = d.cams_trial[i];
        else d.pts[i - 9 * d.n_p] = d.pts_trial[i - 9 * d.n_p];
    }
}

// ============================================================================ small launchers
cudaError_t launch_set_lambda(rba_ctx *c, double lam) {
    k_set_lambda<<<1, 1, 0, c->stream>>>(c->d, lam);
    c->launches++;
    return cudaGetLastError();
}
cudaError_t launch_set_pcg_limits(rba_ctx *c, double tol, int max_iters) {
    k_set_pcg_limits<<<1, 1, 0, c->stream>>>(c->d, tol, max_iters);
    c->launches++;
    return cudaGetLastError();
}
cudaError_t launch_lm_init(rba_ctx *c, double lam, double nu, int reset_iter) {
    k_lm_init<<<1, 1, 0, c->stream>>>(c->d, lam, nu, c->opt.min_rel_decrease, reset_iter);
    c->launches++;
    return cudaGetLastError();
}
cudaError_t launch_lm_need_lin(rba_ctx *c) {
    k_lm_need_lin<<<1, 1, 0, c->stream>>>(c->d);
    c->launches++;
    return cudaGetLastError();
}
static void stamp(rba_ctx *c, int slot) {
    k_stamp<<<1, 1, 0, c->stream>>>(c->d, slot);
    c->launches++;
}

// ============================================================================ the attempt's parts
// Each part is issued on c->stream (the context stream, or the capture stream of a graph body) and
// returns an rba_status; `h` / `use_h` are the conditional handles its kernels drive.
#define CKE(call)                                                                                  \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess) return set_error(RBA_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)
#define CKR(call)                                                                                  \
    do {                                                                                           \
        rba_status s_ = (call);                                                                    \
        if (s_ != RBA_OK) return s_;                                                               \
    } while (0)

// K1 + K2 (relinearize, marginalize, fuse the damping of this attempt)
static rba_status part_linearize_marginalize(rba_ctx *c) {
    DevProblem &d = c->d;
    CKE(launch_linearize(c));
    CKE(launch_reduce_cam_norms(c));
    CKR(allreduce(c, d.cam_n2d, 9 * d.n_p, ncclDouble));
    CKR(allreduce(c, d.scal + SC_E, 2, ncclDouble));
    CKE(launch_cam_scale(c));
    k_lin_done<<<1, 1, 0, c->stream>>>(d);
    c->launches++;
    if (d.s64) CKE(launch_marg64(c));
    else if (d.sc) CKE(launch_sc_build(c));
    else CKE(launch_marginalize(c));
    stamp(c, TS_MARG);
    return RBA_OK;
}

// K3 (backtracking: re-damp the blocks of the current linearization with this attempt's lambda; the
// explicit-SC baselines re-form H~, whose H_ll depends on lambda)
static rba_status part_redamp(rba_ctx *c) {
    if (c->d.s64) CKE(launch_redamp64(c));
    else if (c->d.sc) CKE(launch_sc_build(c));
    else CKE(launch_redamp(c));
    stamp(c, TS_MARG);
    return RBA_OK;
}

// K4 + PCG initialization (h: the PCG loop's handle)
static rba_status part_precond(rba_ctx *c, cudaGraphConditionalHandle h, int use_h) {
    DevProblem &d = c->d;
    CKE(d.sc ? launch_sc_precond(c) : launch_precond_rhs(c));
    CKR(allreduce(c, d.pd, 54 * d.n_p, ncclDouble));
    CKE(launch_precond_finalize(c));
    CKE(launch_pcg_init(c, h, use_h));
    stamp(c, TS_PRE);
    return RBA_OK;
}

// one PCG iteration: K5 (+ all-reduce of the product), K6
static rba_status part_pcg_iteration(rba_ctx *c, cudaGraphConditionalHandle h, int use_h) {
    CKE(launch_matvec_pcg(c));
    if (c->host_reduce_path()) CKR(allreduce(c, c->d.wd, 9 * c->d.n_p, ncclDouble));
    CKE(launch_pcg_step(c, h, use_h));
    return RBA_OK;
}

// K7 + K8 (+ all-reduce of E_trial, bad count, and the two landmark model-decrease sums)
static rba_status part_trial(rba_ctx *c) {
    DevProblem &d = c->d;
    stamp(c, TS_PCG);
    CKE(launch_backsub(c));
    CKE(launch_trial_cost(c));
    CKR(allreduce(c, d.scal + SC_ET, 4, ncclDouble));
    stamp(c, TS_TRIAL);
    return RBA_OK;
}

static rba_status part_control(rba_ctx *c, cudaGraphConditionalHandle h, int use_h) {
    k_lm_control<<<1, 1, 0, c->stream>>>(c->d, h, use_h);
    const int64_t n = 9 * c->d.n_p + 3 * c->d.n_l;
    k_lm_commit<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4 * (int64_t)c->num_sms), 256, 0, c->stream>>>(c->d);
    c->launches += 2;
    return cudaGetLastError() == cudaSuccess ? RBA_OK : set_error(RBA_ERR_CUDA, "k_lm_control / k_lm_commit launch");
}

// ============================================================================ graph capture helpers
// A stream capture into graph `g` on fresh streams (a main stream + NAUX auxiliaries for the
// per-class forks) swapped into the context, so that nested captures (conditional bodies) never
// share a stream with the capture they are nested in.  Counts the kernel nodes it captures.
struct Capture {
    rba_ctx *c;
    cudaStream_t cs = nullptr, aux[rba_ctx::NAUX] = {};
    cudaStream_t saved = nullptr, saved_aux[rba_ctx::NAUX] = {};
    bool saved_prof = false, active = false;
    int64_t launches0 = 0;
    explicit Capture(rba_ctx *c_) : c(c_) {}
    cudaError_t begin(cudaGraph_t g) {
        cudaError_t e;
        if ((e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking))) return e;
        for (int i = 0; i < rba_ctx::NAUX; i++)
            if ((e = cudaStreamCreateWithFlags(&aux[i], cudaStreamNonBlocking))) return e;
        if ((e = cudaStreamBeginCaptureToGraph(cs, g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed))) return e;
        active = true;
        saved = c->stream;
        for (int i = 0; i < rba_ctx::NAUX; i++) saved_aux[i] = c->aux[i], c->aux[i] = aux[i];
        c->stream = cs;
        saved_prof = c->profiling;
        c->profiling = false;
        launches0 = c->launches;
        return cudaSuccess;
    }
    // returns the number of kernel nodes captured; restores the context's streams
    cudaError_t end(int64_t *nkernels) {
        cudaError_t e = cudaSuccess;
        if (active) {
            cudaGraph_t out = nullptr;
            e = cudaStreamEndCapture(cs, &out);
            c->stream = saved;
            for (int i = 0; i < rba_ctx::NAUX; i++) c->aux[i] = saved_aux[i];
            c->profiling = saved_prof;
            if (nkernels) *nkernels = c->launches - launches0;
            c->launches = launches0;
            active = false;
        }
        return e;
    }
    ~Capture() {
        if (active) end(nullptr);
        if (cs) cudaStreamDestroy(cs);
        for (int i = 0; i < rba_ctx::NAUX; i++)
            if (aux[i]) cudaStreamDestroy(aux[i]);
    }
};

// a conditional handle on the graph being captured on c->stream
static cudaError_t capture_handle(rba_ctx *c, cudaGraphConditionalHandle *h, unsigned dflt) {
    cudaStreamCaptureStatus st;
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamGetCaptureInfo(c->stream, &st, nullptr, &g, nullptr, nullptr);
    if (e) return e;
    if (st != cudaStreamCaptureStatusActive || !g) return cudaErrorStreamCaptureInvalidated;
    return cudaGraphConditionalHandleCreate(h, g, dflt, cudaGraphCondAssignDefault);
}

// a conditional node at the current point of the capture on c->stream (it depends on everything
// captured so far and everything captured later depends on it); bodies[0..size) receive its graphs
static cudaError_t capture_conditional(rba_ctx *c, cudaGraphConditionalNodeType type, unsigned size,
                                       cudaGraphConditionalHandle h, cudaGraph_t *bodies) {
    cudaStreamCaptureStatus st;
    cudaGraph_t g = nullptr;
    const cudaGraphNode_t *deps = nullptr;
    size_t nd = 0;
    cudaError_t e = cudaStreamGetCaptureInfo(c->stream, &st, nullptr, &g, &deps, &nd);
    if (e) return e;
    if (st != cudaStreamCaptureStatusActive || !g) return cudaErrorStreamCaptureInvalidated;
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = type;
    np.conditional.size = size;
    cudaGraphNode_t node;
    if ((e = cudaGraphAddNode(&node, g, deps, nd, &np))) return e;
    for (unsigned i = 0; i < size; i++) bodies[i] = np.conditional.phGraph_out[i];
    return cudaStreamUpdateCaptureDependencies(c->stream, &node, 1, cudaStreamSetCaptureDependencies);
}

// capture `part` into graph g; *n = its kernel nodes
template <typename F>
static rba_status capture_into(rba_ctx *c, cudaGraph_t g, int64_t *n, F &&part) {
    Capture cap(c);
    cudaError_t e = cap.begin(g);
    if (e) return set_error(RBA_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    rba_status s = part();
    e = cap.end(n);
    if (s != RBA_OK) return s;
    if (e) return set_error(RBA_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    return RBA_OK;
}

// ---- the standalone PCG graph (rba_pcg_solve): while (cond) { K5; [all-reduce]; K6 }.  k_pcg_init
// (issued before the launch) marks the solve done when there is nothing to do; the first update
// kernel then clears the condition.
rba_status build_pcg_graph(rba_ctx *c) {
    cudaGraph_t g;
    cudaError_t e;
    if ((e = cudaGraphCreate(&g, 0))) return set_error(RBA_ERR_CUDA, cudaGetErrorString(e));
    cudaGraphConditionalHandle h;
    if ((e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault))) {
        cudaGraphDestroy(g);
        return set_error(RBA_ERR_CUDA, cudaGetErrorString(e));
    }
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    if ((e = cudaGraphAddNode(&node, g, nullptr, 0, &np))) {
        cudaGraphDestroy(g);
        return set_error(RBA_ERR_CUDA, cudaGetErrorString(e));
    }
    static const bool nofork = getenv("RBA_GRAPH_NOFORK") != nullptr;
    c->nofork = nofork;
    rba_status s = capture_into(c, np.conditional.phGraph_out[0], &c->graph_body_kernels,
                                [&] { return part_pcg_iteration(c, h, 1); });
    c->nofork = false;
    if (s == RBA_OK && (e = cudaGraphInstantiate(&c->pcg_exec, g, 0))) {
        cudaGetLastError();
        s = set_error(RBA_ERR_CUDA, std::string("PCG graph instantiation: ") + cudaGetErrorString(e));
    }
    if (s != RBA_OK) {
        cudaGraphDestroy(g);
        c->pcg_exec = nullptr;
        return s;
    }
    c->pcg_graph = g;
    return RBA_OK;
}

// ---- the LM graph: k_lm_loop_begin; while (LM) { k_lm_begin; if (relinearize) {K1, K2} else {K3};
// K4, k_pcg_init; while (PCG) {K5, K6}; K7, K8; k_lm_control; k_lm_commit }
static rba_status build_lm_graph(rba_ctx *c) {
    rba_ctx::LmGraph &G = c->lmg;
    cudaGraph_t g;
    cudaError_t e;
    if ((e = cudaGraphCreate(&g, 0))) return set_error(RBA_ERR_CUDA, cudaGetErrorString(e));
    static const bool nofork = getenv("RBA_GRAPH_NOFORK") != nullptr;
    c->nofork = nofork;
    rba_status s = capture_into(c, g, nullptr, [&]() -> rba_status {
        cudaGraphConditionalHandle h_lm;
        CKE(capture_handle(c, &h_lm, 0));
        k_lm_loop_begin<<<1, 1, 0, c->stream>>>(c->d, h_lm);
        cudaGraph_t lm_body;
        CKE(capture_conditional(c, cudaGraphCondTypeWhile, 1, h_lm, &lm_body));
        return capture_into(c, lm_body, nullptr, [&]() -> rba_status {
            cudaGraphConditionalHandle h_lin, h_pcg;
            CKE(capture_handle(c, &h_lin, 0));
            CKE(capture_handle(c, &h_pcg, 0));
            int64_t n0 = c->launches;
            k_lm_begin<<<1, 1, 0, c->stream>>>(c->d, h_lin, 1);
            c->launches++;
            G.n_head = c->launches - n0;
            cudaGraph_t br[2];
            CKE(capture_conditional(c, cudaGraphCondTypeIf, 2, h_lin, br));
            CKR(capture_into(c, br[0], &G.n_lin, [&] { return part_linearize_marginalize(c); }));
            CKR(capture_into(c, br[1], &G.n_redamp, [&] { return part_redamp(c); }));
            n0 = c->launches;
            CKR(part_precond(c, h_pcg, 1));
            G.n_mid = c->launches - n0;
            cudaGraph_t pcg_body;
            CKE(capture_conditional(c, cudaGraphCondTypeWhile, 1, h_pcg, &pcg_body));
            CKR(capture_into(c, pcg_body, &G.n_pcg, [&] { return part_pcg_iteration(c, h_pcg, 1); }));
            n0 = c->launches;
            CKR(part_trial(c));
            CKR(part_control(c, h_lm, 1));
            G.n_tail = c->launches - n0;
            return RBA_OK;
        });
    });
    c->nofork = false;
    if (s == RBA_OK && (e = cudaGraphInstantiate(&G.exec, g, 0))) {
        cudaGetLastError();
        s = set_error(RBA_ERR_CUDA, std::string("LM graph instantiation: ") + cudaGetErrorString(e));
    }
    if (s != RBA_OK) {
        cudaGraphDestroy(g);
        G.exec = nullptr;
        return s;
    }
    G.graph = g;
    return RBA_OK;
}

// graphs are used on one GPU (and, when NCCL captures into conditional bodies, on several); the
// k > 512 product keeps the eager issue order (its fused kernel is slower inside graph branches)
static bool huge_eager(rba_ctx *c) {
    static const bool force = getenv("RBA_HUGE_GRAPH") != nullptr;
    return (c->n_huge_fused > 0 || c->n_huge_out > 0) && !force;
}
bool use_lm_graph(rba_ctx *c) {
    if (c->no_graph || huge_eager(c)) return false;
    if (!c->lmg.built) {
        c->lmg.built = true;
        if (build_lm_graph(c) != RBA_OK) c->lmg.failed = true;
    }
    return !c->lmg.failed && c->lmg.exec;
}
bool use_pcg_graph(rba_ctx *c) {
    if (c->no_graph || huge_eager(c)) return false;
    if (!c->pcg_exec && !c->pcg_graph_failed)
        if (build_pcg_graph(c) != RBA_OK) c->pcg_graph_failed = true;
    return c->pcg_exec != nullptr;
}

// The PCG loop issued eagerly (after k_pcg_init): the standalone graph, or host batches of
// iterations (1, 2, 4, ... 64) between polls of the done flag.
rba_status run_pcg_loop(rba_ctx *c) {
    DevProblem &d = c->d;
    if (use_pcg_graph(c)) {
        Prof P(c, KID_MATVEC, 0.0);
        CKE(cudaGraphLaunch(c->pcg_exec, c->stream));
        P.end();
        CKE(cudaMemcpyAsync(c->h_pcg, d.pcg, sizeof(PcgState), cudaMemcpyDeviceToHost, c->stream));
        CKE(cudaStreamSynchronize(c->stream));
        c->launches += c->graph_body_kernels * std::max(1, c->h_pcg->it);
        return RBA_OK;
    }
    int batch = 1;
    for (;;) {
        CKE(cudaMemcpyAsync(c->h_pcg, d.pcg, sizeof(PcgState), cudaMemcpyDeviceToHost, c->stream));
        CKE(cudaStreamSynchronize(c->stream));
        if (c->h_pcg->done || c->h_pcg->it >= c->opt.pcg_max_iters) break;
        const int todo = std::min(batch, c->opt.pcg_max_iters - c->h_pcg->it);
        for (int b = 0; b < todo; b++) CKR(part_pcg_iteration(c, 0, 0));
        batch = std::min(batch * 2, 64);
    }
    return RBA_OK;
}

// ============================================================================ the LM driver
// launches of the graph's kernel nodes for the attempts of these reports
static int64_t graph_launches(const rba_ctx::LmGraph &G, const rba_lm_report *r, int n) {
    int64_t t = 1;  // k_lm_loop_begin
    for (int i = 0; i < n; i++) {
        const int bodies = r[i].pcg_iters + ((r[i].pcg_reason == 2 && r[i].pcg_iters > 0) ? 1 : 0);
        t += G.n_head + (r[i].relinearized ? G.n_lin : G.n_redamp) + G.n_mid + (int64_t)bodies * G.n_pcg + G.n_tail;
    }
    return t;
}

// Run up to `target` attempts (stop early at ftol / error).  Reports -> reps (may be NULL).
static rba_status run_lm(rba_ctx *c, int64_t target, double ftol, rba_lm_report *reps, int64_t *n_out) {
    DevProblem &d = c->d;
    *n_out = 0;
    CKE(cudaSetDevice(c->device));
    if (c->lm_dirty) {
        CKE(launch_lm_need_lin(c));
        c->lm_dirty = false;
    }
    // the step-by-step API's view of the blocks is invalid from here on
    c->linearized = c->marginalized = c->solved = c->backsubbed = false;
    const bool graph = use_lm_graph(c);
    int64_t done = 0;
    bool stop = false;
    LmDev hl;
    while (done < target && !stop) {
        const int64_t chunk = graph ? std::min<int64_t>(target - done, rba_ctx::REP_CAP) : 1;
        k_lm_request<<<1, 1, 0, c->stream>>>(d, chunk, ftol);
        c->launches++;
        if (graph) {
            CKE(cudaGraphLaunch(c->lmg.exec, c->stream));
        } else {
            // eager: the branch is known from the previous attempt's copy of the schedule
            CKE(cudaMemcpyAsync(&hl, d.lm, sizeof(LmDev), cudaMemcpyDeviceToHost, c->stream));
            CKE(cudaStreamSynchronize(c->stream));
            k_lm_begin<<<1, 1, 0, c->stream>>>(d, 0, 0);
            c->launches++;
            CKR(hl.need_lin ? part_linearize_marginalize(c) : part_redamp(c));
            CKR(part_precond(c, 0, 0));
            CKR(run_pcg_loop(c));
            CKR(part_trial(c));
            CKR(part_control(c, 0, 0));
        }
        CKE(cudaMemcpyAsync(&hl, d.lm, sizeof(LmDev), cudaMemcpyDeviceToHost, c->stream));
        CKE(cudaMemcpyAsync(c->h_reps, d.reps, sizeof(rba_lm_report) * chunk, cudaMemcpyDeviceToHost, c->stream));
        CKE(cudaStreamSynchronize(c->stream));
        const int64_t n = std::min<int64_t>(hl.n_done, chunk);
        if (graph) c->launches += graph_launches(c->lmg, c->h_reps, (int)n);
        for (int64_t i = 0; i < n; i++) {
            c->h_reps[i].device_bytes = c->device_bytes;
            if (reps) reps[done + i] = c->h_reps[i];
        }
        done += n;
        stop = hl.stop != 0 || n < chunk;
        c->cost = hl.cost;
        if (hl.stop == 2) {
            *n_out = done;
            return set_error(RBA_ERR_BAD_PROBLEM, "a point is not in front of its camera (or E is not finite) at the current state");
        }
    }
    *n_out = done;
    return RBA_OK;
}

}  // namespace rba

using namespace rba;

extern "C" rba_status rba_lm_step(rba_ctx *c, rba_lm_report *rep) {
    if (!c) return set_error(RBA_ERR_INVALID_ARG, "null ctx");
    nvtxRangePushA("rba_lm_step");
    rba_lm_report r;
    int64_t n = 0;
    rba_status s = run_lm(c, 1, 0.0, &r, &n);
    nvtxRangePop();
    if (s == RBA_OK && n != 1) s = set_error(RBA_ERR_CUDA, "rba_lm_step: no report");
    if (rep && n == 1) *rep = r;
    return s;
}

extern "C" rba_status rba_lm_solve(rba_ctx *c, int max_iters, double ftol, rba_lm_report *reports, int *n_done) {
    if (!c) return set_error(RBA_ERR_INVALID_ARG, "null ctx");
    if (max_iters < 0 || !(ftol >= 0) || !std::isfinite(ftol)) return set_error(RBA_ERR_INVALID_ARG, "rba_lm_solve: bad max_iters / ftol");
    nvtxRangePushA("rba_lm_solve");
    int64_t n = 0;
    rba_status s = run_lm(c, max_iters, ftol, reports, &n);
    nvtxRangePop();
    if (n_done) *n_done = (int)n;
    return s;
}

extern "C" rba_status rba_reset_lm(rba_ctx *c) {
    if (!c) return set_error(RBA_ERR_INVALID_ARG, "null ctx");
    if (launch_lm_init(c, c->opt.lambda0, 2.0, 1)) return set_error(RBA_ERR_CUDA, "rba_reset_lm");
    return RBA_OK;
}

extern "C" rba_status rba_set_lm(rba_ctx *c, double lambda, double nu) {
    if (!c) return set_error(RBA_ERR_INVALID_ARG, "null ctx");
    if (!(lambda > 0) || !std::isfinite(lambda) || !(nu >= 1) || !std::isfinite(nu))
        return set_error(RBA_ERR_INVALID_ARG, "rba_set_lm: lambda > 0 and nu >= 1 required");
    if (launch_lm_init(c, lambda, nu, 0)) return set_error(RBA_ERR_CUDA, "rba_set_lm");
    return RBA_OK;
}

extern "C" rba_status rba_get_lm(rba_ctx *c, double *lambda, double *nu, int64_t *iter) {
    if (!c) return set_error(RBA_ERR_INVALID_ARG, "null ctx");
    LmDev hl;
    CKE(cudaMemcpyAsync(&hl, c->d.lm, sizeof(LmDev), cudaMemcpyDeviceToHost, c->stream));
    CKE(cudaStreamSynchronize(c->stream));
    if (lambda) *lambda = hl.lambda;
    if (nu) *nu = hl.nu;
    if (iter) *iter = hl.iter;
    return RBA_OK;
}

extern "C" rba_status rba_set_pcg_limits(rba_ctx *c, double rel_tol, int max_iters) {
    if (!c) return set_error(RBA_ERR_INVALID_ARG, "null ctx");
    if (!(rel_tol >= 0) || !std::isfinite(rel_tol) || max_iters < 0)
        return set_error(RBA_ERR_INVALID_ARG, "rba_set_pcg_limits: rel_tol >= 0 and max_iters >= 0 required");
    c->opt.pcg_rel_tol = rel_tol;
    c->opt.pcg_max_iters = max_iters;
    if (launch_set_pcg_limits(c, rel_tol, max_iters)) return set_error(RBA_ERR_CUDA, "rba_set_pcg_limits");
    return RBA_OK;
}

extern "C" rba_status rba_device_bytes(rba_ctx *c, int64_t *bytes) {
    if (!c || !bytes) return set_error(RBA_ERR_INVALID_ARG, "null argument");
    *bytes = c->device_bytes;
    return RBA_OK;
}

extern "C" rba_status rba_plan_bytes(rba_ctx *c, double *marginalize_bytes, double *matvec_bytes) {
    if (!c || !marginalize_bytes || !matvec_bytes) return set_error(RBA_ERR_INVALID_ARG, "null argument");
    *marginalize_bytes = c->marg_bytes;
    *matvec_bytes = c->matvec_bytes;
    return RBA_OK;
}

extern "C" rba_status rba_get_info(rba_ctx *c, rba_info *info) {
    if (!c || !info) return set_error(RBA_ERR_INVALID_ARG, "null argument");
    memset(info, 0, sizeof(*info));
    info->lm_graph = c->lmg.failed ? -1 : (c->lmg.exec ? 1 : 0);
    info->pcg_graph = c->pcg_graph_failed ? -1 : (c->pcg_exec ? 1 : 0);
    info->nccl = c->have_comm ? 1 : 0;
    info->deterministic = c->d.det;
    info->n_landmarks = c->d.n_l;
    info->n_observations = c->d.n_obs;
    return RBA_OK;
}

static uint64_t fnv1a(const void *p, size_t n, uint64_t h = 1469598103934665603ull) {
    const unsigned char *b = static_cast<const unsigned char *>(p);
    for (size_t i = 0; i < n; i++) h = (h ^ b[i]) * 1099511628211ull;
    return h;
}

extern "C" rba_status rba_checksums(rba_ctx *c, uint64_t out[4]) {
    if (!c || !out) return set_error(RBA_ERR_INVALID_ARG, "null argument");
    const int64_t np = c->d.n_p;
    std::vector<double> buf(54 * std::max<int64_t>(np, 1));
    const double *src[4] = {c->d.cam_n2d, c->d.pd, c->d.wd, c->d.x};
    const int64_t cnt[4] = {9 * np, 54 * np, 9 * np, 9 * np};
    for (int i = 0; i < 4; i++) {
        CKE(cudaMemcpyAsync(buf.data(), src[i], sizeof(double) * cnt[i], cudaMemcpyDeviceToHost, c->stream));
        CKE(cudaStreamSynchronize(c->stream));
        out[i] = fnv1a(buf.data(), sizeof(double) * cnt[i]);
    }
    return RBA_OK;
}
