// rba_api.cu -- C ABI of librba (include/rba.h): planner (landmark grouping, bucketing by track
// length, LPT sharding, arena layout), NCCL plumbing and the host-side LM / PCG drivers.  All
// arithmetic of the method runs in the kernels of rba_kernels.cu.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <queue>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "rba_internal.cuh"

using namespace rba;

static thread_local std::string g_err;

static rba_status fail(rba_status s, const std::string &msg) {
    g_err = msg;
    return s;
}

#define CK(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            return fail(RBA_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));          \
    } while (0)
#define CKN(call)                                                                                  \
    do {                                                                                           \
        ncclResult_t r_ = (call);                                                                  \
        if (r_ != ncclSuccess) return fail(RBA_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
    } while (0)
#define CKS(call)                                                                                  \
    do {                                                                                           \
        rba_status s_ = (call);                                                                    \
        if (s_ != RBA_OK) return s_;                                                               \
    } while (0)

namespace rba {
rba_status set_error(rba_status s, const std::string &msg) { return fail(s, msg); }
bool use_pcg_graph(rba_ctx *c);
rba_status run_pcg_loop(rba_ctx *c);
double plan_marg_bytes(rba_ctx *c) { return c->marg_bytes; }
double plan_backsub_bytes(rba_ctx *c) { return c->backsub_bytes; }
double plan_matvec_bytes(rba_ctx *c) { return c->matvec_bytes; }

Prof::Prof(rba_ctx *c_, int kid_, double bytes_) : c(c_), kid(kid_), bytes(bytes_) {
    if (!c->profiling) return;
    if (c->ev_pool.empty()) {
        cudaEventCreate(&a);
    } else {
        a = c->ev_pool.back();
        c->ev_pool.pop_back();
    }
    cudaEventRecord(a, c->stream);
}
void Prof::end() {
    if (!c->profiling || !a) return;
    cudaEvent_t b;
    if (c->ev_pool.empty()) {
        cudaEventCreate(&b);
    } else {
        b = c->ev_pool.back();
        c->ev_pool.pop_back();
    }
    cudaEventRecord(b, c->stream);
    c->prof.push_back(Launch{kid, a, b, bytes});
    a = nullptr;
}
}  // namespace rba

// ------------------------------------------------------------------------------------ memory
static rba_status dalloc(rba_ctx *c, void **p, size_t bytes) {
    *p = nullptr;
    if (bytes == 0) bytes = 16;
    if (c->opt.alloc) {
        *p = c->opt.alloc(bytes, c->opt.alloc_ctx);
        if (!*p) return fail(RBA_ERR_OOM, "device allocation of " + std::to_string(bytes) + " bytes failed");
    } else {
        cudaError_t e = cudaMalloc(p, bytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(RBA_ERR_OOM, "cudaMalloc of " + std::to_string(bytes) + " bytes failed: " +
                                         cudaGetErrorString(e));
        }
    }
    // stale-memory check (test switch): RBA_POISON_ALLOC=<byte>[:lo:hi] fills every new allocation
    // (allocation indices lo..hi-1) with that byte, so a kernel that reads memory before writing it
    // changes the results (tests/test_gpu_deterministic.py compares two poison patterns bitwise)
    if (const char *pz = getenv("RBA_POISON_ALLOC")) {  // <byte>[:lo:hi[:other byte]]
        int byte = 0, other = -1;
        long long plo = 0, phi = -1;
        const int n = sscanf(pz, "%d:%lld:%lld:%d", &byte, &plo, &phi, &other);
        const long long idx = (long long)c->allocations.size();
        const bool in = n >= 1 && idx >= plo && (n < 3 || idx < phi);
        if (in || other >= 0) cudaMemset(*p, (in ? byte : other) & 255, bytes), cudaDeviceSynchronize();
        if (getenv("RBA_ALLOC_TRACE")) fprintf(stderr, "rba alloc %lld: %zu bytes\n", idx, bytes);
    }
    c->allocations.push_back(*p);
    c->device_bytes += (int64_t)bytes;
    return RBA_OK;
}
template <typename T>
static rba_status dalloc_n(rba_ctx *c, T **p, int64_t n) {
    return dalloc(c, reinterpret_cast<void **>(p), sizeof(T) * (size_t)std::max<int64_t>(n, 1));
}

// ------------------------------------------------------------------------------------ sharding
// Deterministic LPT on block bytes (2k+3)(9k+4): landmarks by bytes descending (ties by index),
// each to the least-loaded rank (ties by lowest rank).  SURVEY §8e.
static void lpt_shards(const int32_t *k, int64_t n, int world, int32_t *owner) {
    if (world <= 1) {
        std::fill(owner, owner + n, 0);
        return;
    }
    std::vector<int64_t> idx(n);
    std::iota(idx.begin(), idx.end(), 0);
    auto bytes = [&](int64_t j) { return (int64_t)(2 * k[j] + 3) * (9 * k[j] + 4); };
    std::stable_sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) { return bytes(a) > bytes(b); });
    using E = std::pair<int64_t, int>;
    std::priority_queue<E, std::vector<E>, std::greater<E>> pq;
    for (int r = 0; r < world; r++) pq.push({0, r});
    for (int64_t j : idx) {
        E e = pq.top();
        pq.pop();
        owner[j] = e.second;
        e.first += bytes(j);
        pq.push(e);
    }
}

extern "C" rba_status rba_plan_shards(const int32_t *k, int64_t n, int world, int32_t *owner) {
    if (!k || !owner || n < 0 || world < 1) return fail(RBA_ERR_INVALID_ARG, "rba_plan_shards: bad argument");
    lpt_shards(k, n, world, owner);
    return RBA_OK;
}

extern "C" void rba_default_options(rba_options *o) {
    std::memset(o, 0, sizeof(*o));
    o->device = 0;
    o->world = 1;
    o->rank = 0;
    o->lambda0 = 1e-4;
    o->pcg_rel_tol = 1e-2;
    o->pcg_max_iters = 500;
    o->min_rel_decrease = 1e-3;
    o->diag_min = 1e-6;
    o->diag_max = 1e32;
    o->huber_delta = 0.0;
    o->deterministic = 0;
}

extern "C" const char *rba_last_error(void) { return g_err.c_str(); }

extern "C" rba_status rba_nccl_unique_id(void *id128) {
    if (!id128) return fail(RBA_ERR_INVALID_ARG, "null id");
    ncclUniqueId id;
    CKN(ncclGetUniqueId(&id));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    std::memcpy(id128, &id, 128);
    return RBA_OK;
}

static void free_ctx(rba_ctx *c) {
    if (!c) return;
    if (c->device >= 0) cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (auto &l : c->prof) {
        cudaEventDestroy(l.a);
        cudaEventDestroy(l.b);
    }
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    for (void *p : c->allocations) {
        if (c->opt.free) c->opt.free(p, c->opt.alloc_ctx);
        else cudaFree(p);
    }
    if (c->h_scal) cudaFreeHost(c->h_scal);
    if (c->h_pcg) cudaFreeHost(c->h_pcg);
    if (c->h_reps) cudaFreeHost(c->h_reps);
    if (c->lmg.exec) cudaGraphExecDestroy(c->lmg.exec);
    if (c->lmg.graph) cudaGraphDestroy(c->lmg.graph);
    if (c->have_comm) ncclCommDestroy(c->comm);
    if (c->pcg_exec) cudaGraphExecDestroy(c->pcg_exec);
    if (c->pcg_graph) cudaGraphDestroy(c->pcg_graph);
    for (int i = 0; i < rba_ctx::NAUX; i++) {
        if (c->aux[i]) cudaStreamDestroy(c->aux[i]);
        if (c->ev_join[i]) cudaEventDestroy(c->ev_join[i]);
    }
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

extern "C" rba_status rba_destroy(rba_ctx *c) {
    free_ctx(c);
    return RBA_OK;
}

// Persistent CTAs of a product / preconditioner class kernel (one per SM at most: their smem
// rings take the SM): every class kernel gets all SMs.  RBA_PROP_GRID=1: SMs in proportion to the
// class's bytes of the product, so that the classes, forked over separate streams, could run side
// by side -- measured 1.8x slower (cfg 4 product 2.22 -> 4.01 ms): the class kernels do not share
// the GPU that way.
static int64_t prop_ctas(const rba_ctx *c, double bytes) {
    static const bool prop = getenv("RBA_PROP_GRID") && atoi(getenv("RBA_PROP_GRID")) != 0;
    if (!prop || c->matvec_bytes <= 0) return c->num_sms;
    return std::max<int64_t>(1, std::min<int64_t>(c->num_sms, std::llround(c->num_sms * bytes / c->matvec_bytes)));
}

// ------------------------------------------------------------------------------------ create
extern "C" rba_status rba_create(const double *cameras, int64_t n_cams, const double *points, int64_t n_points,
                                 const int32_t *obs_cam, const int32_t *obs_pt, const double *obs_uv,
                                 int64_t n_obs, const rba_options *opt_in, rba_ctx **out) {
    if (!out) return fail(RBA_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    rba_options opt;
    if (opt_in) opt = *opt_in;
    else rba_default_options(&opt);
    if (!cameras || !points || (n_obs > 0 && (!obs_cam || !obs_pt || !obs_uv)) || n_cams < 1 || n_points < 0 ||
        n_obs < 0)
        return fail(RBA_ERR_INVALID_ARG, "rba_create: null pointer or negative size");
    if (opt.world > 1 && opt.solver != 0)
        return fail(RBA_ERR_INVALID_ARG, "rba_create: the explicit-SC baselines are single-GPU (world must be 1)");
    if (opt.world < 1 || opt.rank < 0 || opt.rank >= opt.world || !(opt.lambda0 > 0) || !(opt.pcg_rel_tol >= 0) ||
        opt.pcg_max_iters < 0 || !(opt.diag_min > 0) || !(opt.diag_max >= opt.diag_min) ||
        !(opt.huber_delta >= 0) || !std::isfinite(opt.huber_delta) || opt.solver < 0 || opt.solver > 2 ||
        opt.storage < 0 || opt.storage > 1 || (opt.storage == 1 && opt.solver != 0) || opt.precision < 0 ||
        opt.precision > 1 || (opt.precision == 1 && (opt.solver != 0 || opt.storage != 0)) || opt.deterministic < 0 ||
        opt.deterministic > 1 || (opt.deterministic == 1 && (opt.solver != 0 || opt.storage != 0 || opt.precision != 0)))
        return fail(RBA_ERR_INVALID_ARG, "rba_create: bad options");
    if (n_obs >= (int64_t)1 << 31 || n_points >= (int64_t)1 << 31 || n_cams >= (int64_t)1 << 28)
        return fail(RBA_ERR_INVALID_ARG, "rba_create: problem too large for int32 indices");
    // ---- validation (RBA_ERR_BAD_PROBLEM)
    for (int64_t i = 0; i < 9 * n_cams; i++)
        if (!std::isfinite(cameras[i])) return fail(RBA_ERR_BAD_PROBLEM, "non-finite camera parameter at camera " + std::to_string(i / 9));
    for (int64_t i = 0; i < n_cams; i++)
        if (!(cameras[9 * i + 6] > 0)) return fail(RBA_ERR_BAD_PROBLEM, "focal length <= 0 at camera " + std::to_string(i));
    for (int64_t i = 0; i < 3 * n_points; i++)
        if (!std::isfinite(points[i])) return fail(RBA_ERR_BAD_PROBLEM, "non-finite point at landmark " + std::to_string(i / 3));
    std::vector<int32_t> kcount(n_points, 0);
    for (int64_t i = 0; i < n_obs; i++) {
        if (obs_cam[i] < 0 || obs_cam[i] >= n_cams)
            return fail(RBA_ERR_BAD_PROBLEM, "observation " + std::to_string(i) + ": camera index out of range");
        if (obs_pt[i] < 0 || obs_pt[i] >= n_points)
            return fail(RBA_ERR_BAD_PROBLEM, "observation " + std::to_string(i) + ": landmark index out of range");
        if (!std::isfinite(obs_uv[2 * i]) || !std::isfinite(obs_uv[2 * i + 1]))
            return fail(RBA_ERR_BAD_PROBLEM, "observation " + std::to_string(i) + ": non-finite pixel");
        kcount[obs_pt[i]]++;
    }
    for (int64_t j = 0; j < n_points; j++) {
        if (kcount[j] < 2)
            return fail(RBA_ERR_BAD_PROBLEM, "landmark " + std::to_string(j) + " has " + std::to_string(kcount[j]) +
                                                 " < 2 observations (P:469)");
        if (opt.precision == 1 && kcount[j] > KMAX64)
            return fail(RBA_ERR_BAD_PROBLEM, "landmark " + std::to_string(j) + ": track length " +
                                                 std::to_string(kcount[j]) + " exceeds sqrt-BA-64's " +
                                                 std::to_string(KMAX64));
        if (kcount[j] > KMAX)
            return fail(RBA_ERR_BAD_PROBLEM, "landmark " + std::to_string(j) + ": track length " +
                                                 std::to_string(kcount[j]) + " exceeds this build's KMAX " +
                                                 std::to_string(KMAX));
    }
    // observations sorted by (landmark, camera)
    std::vector<int64_t> ord(n_obs);
    std::iota(ord.begin(), ord.end(), 0);
    std::sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) {
        return obs_pt[a] != obs_pt[b] ? obs_pt[a] < obs_pt[b] : obs_cam[a] < obs_cam[b];
    });
    for (int64_t i = 1; i < n_obs; i++)
        if (obs_pt[ord[i]] == obs_pt[ord[i - 1]] && obs_cam[ord[i]] == obs_cam[ord[i - 1]])
            return fail(RBA_ERR_BAD_PROBLEM, "duplicate observation of landmark " + std::to_string(obs_pt[ord[i]]) +
                                                 " by camera " + std::to_string(obs_cam[ord[i]]));
    std::vector<int64_t> gptr(n_points + 1, 0);
    for (int64_t j = 0; j < n_points; j++) gptr[j + 1] = gptr[j] + kcount[j];

    rba_ctx *c = new rba_ctx();
    c->opt = opt;
    c->device = opt.device;
    c->world = opt.world;
    c->rank = opt.rank;
    c->n_p = n_cams;
    c->n_l_global = n_points;
    c->n_obs_global = n_obs;
    auto bail = [&](rba_status s) {
        free_ctx(c);
        return s;
    };
#define CKC(call)                                                                                  \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess) {                                                                   \
            g_err = std::string(#call) + ": " + cudaGetErrorString(e_);                            \
            return bail(RBA_ERR_CUDA);                                                             \
        }                                                                                          \
    } while (0)
#define CKSC(call)                                                                                 \
    do {                                                                                           \
        rba_status s_ = (call);                                                                    \
        if (s_ != RBA_OK) return bail(s_);                                                         \
    } while (0)
    CKC(cudaSetDevice(opt.device));
    CKC(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, opt.device));
    for (int i = 0; i < rba_ctx::NAUX; i++) {
        CKC(cudaStreamCreateWithFlags(&c->aux[i], cudaStreamNonBlocking));
        CKC(cudaEventCreateWithFlags(&c->ev_join[i], cudaEventDisableTiming));
    }
    CKC(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    if (opt.stream) {
        c->stream = (cudaStream_t)opt.stream;
    } else {
        CKC(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
    }
    // ---- shard and order the local landmarks: by k, then first camera, then index
    std::vector<int32_t> owner(n_points);
    lpt_shards(kcount.data(), n_points, opt.world, owner.data());
    std::vector<int32_t> loc;
    for (int64_t j = 0; j < n_points; j++)
        if (owner[j] == opt.rank) loc.push_back((int32_t)j);
    std::stable_sort(loc.begin(), loc.end(), [&](int32_t a, int32_t b) {
        if (kcount[a] != kcount[b]) return kcount[a] < kcount[b];
        const int32_t ca = obs_cam[ord[gptr[a]]], cb = obs_cam[ord[gptr[b]]];
        if (ca != cb) return ca < cb;
        return a < b;
    });
    const int64_t nl = (int64_t)loc.size();
    c->lm_orig = loc;
    c->orig_to_int.assign(n_points, -1);
    for (int64_t i = 0; i < nl; i++) c->orig_to_int[loc[i]] = (int32_t)i;
    c->h_k.resize(nl);
    c->h_r2.resize(nl);
    c->h_side.resize(nl);
    c->h_pk.assign(nl, 0);
    std::vector<int32_t> h_obs0(nl);
    int64_t nobs_loc = 0;
    for (int64_t i = 0; i < nl; i++) {
        const int k = kcount[loc[i]];
        c->h_k[i] = k;
        h_obs0[i] = (int32_t)nobs_loc;
        nobs_loc += k;
        c->logical_bytes += (int64_t)(2 * k + 3) * (9 * k + 4) * 4 + 48;
        c->marg_bytes += (double)(2 * k + 3) * (9 * k + 4) * 4 + 48 + 20.0 * k;
        c->matvec_bytes += 72.0 * k * k;
        // K7: R^1 rows, TL, camera indices, landmark header / point / scaling / D reads, dl + trial writes
        c->backsub_bytes += 112.0 * k + 148;
        const int rg = k <= 16 ? 0 : k <= 256 ? 1 : 2;  // K7 regimes (landmarks sorted by k)
        c->bs_bytes[rg] += 112.0 * k + 148;
        c->bs_hi[rg] = i + 1;
    }
    // ---- R2 arena: packs of same-k small landmarks (classes G = 2, 4, 8, 16), then large ones
    std::vector<Pack> packs;
    const int bounds[4] = {2, 4, 8, 16};
    int64_t r2_total = 0, pos = 0, q_total = 0;
    c->h_q.assign(nl, -1);
    for (int cls = 0; cls < 4; cls++) {
        const int NG = 32 / bounds[cls];
        c->pack_lo[cls] = (int64_t)packs.size();
        while (pos < nl && c->h_k[pos] <= bounds[cls]) {
            const int k = c->h_k[pos];
            int np = 0;
            while (pos + np < nl && np < NG && c->h_k[pos + np] == k &&
                   4 * small_pack_floats(k, np + 1) <= SMALL_STAGE_BYTES)  // (a pack fits a pipeline stage)
                np++;
            packs.push_back(Pack{(int32_t)pos, np, r2_total, h_obs0[pos], k, (int32_t)q_total, 0});
            for (int m = 0; m < np; m++) {
                c->h_r2[pos + m] = r2_total;
                c->h_pk[pos + m] = m | (np << 8);
                c->h_q[pos + m] = (int32_t)(q_total + 2 * k * m);
            }
            q_total += 2 * k * np;
            r2_total += pad4(small_pack_floats(k, np));
            pos += np;
        }
        c->pack_hi[cls] = (int64_t)packs.size();
    }
    c->n_packs = (int64_t)packs.size();
    // small-k pipeline stages: consecutive packs up to SMALL_STAGE_BYTES, 320 camera indices and
    // 64 packs, each with its table of work units (pack slot, 4-row-pair range)
    std::vector<SmallChunk> chunks;
    std::vector<uint16_t> units;
    for (int64_t p0 = 0; p0 < c->n_packs;) {
        SmallChunk ch{};
        ch.p0 = (int32_t)p0;
        ch.base = packs[p0].base;
        int64_t bytes = 0;
        const int32_t cam0 = packs[p0].obs0 & ~3;
        int32_t cam_end = cam0;
        int64_t q = p0;
        while (q < c->n_packs) {
            const int64_t pb = 4 * pad4(small_pack_floats(packs[q].k, packs[q].np));
            const int32_t ce = (packs[q].obs0 + packs[q].np * packs[q].k + 3) & ~3;
            const int32_t qe = (packs[q].q0 + 2 * packs[q].np * packs[q].k + 3) & ~3;
            if (q > p0 && (bytes + pb > SMALL_STAGE_BYTES || ce - cam0 > 320 || q - p0 >= 64 ||
                           qe - (packs[p0].q0 & ~3) > SP_QCAP))
                break;
            bytes += pb;
            cam_end = ce;
            q++;
        }
        ch.np = (int32_t)(q - p0);
        ch.bytes = (int32_t)bytes;
        ch.q0 = packs[p0].q0 & ~3;
        ch.nq = ((packs[q - 1].q0 + 2 * packs[q - 1].np * packs[q - 1].k + 3) & ~3) - ch.q0;
        ch.cam0 = cam0;
        ch.ncam = cam_end - cam0;
        ch.unit0 = (int32_t)units.size();
        for (int64_t sl = 0; sl < ch.np; sl++) {
            const int nr = (packs[p0 + sl].k + 3) / 4;
            for (int r = 0; r < nr; r++) units.push_back((uint16_t)(sl | (r << 8)));
        }
        ch.nreal = (int32_t)(units.size() - ch.unit0);
        while ((units.size() - ch.unit0) % 8) units.push_back(0xFFFF);
        ch.nunit = (int32_t)(units.size() - ch.unit0);
        chunks.push_back(ch);
        p0 = q;
    }
    c->n_chunks = (int64_t)chunks.size();
    std::vector<int64_t> chunk_lo;
    {
        double tot = 0;
        for (auto &ch : chunks) tot += ch.bytes;
        const int64_t G = std::min<int64_t>(prop_ctas(c, tot), c->n_chunks);
        c->chunk_ctas = G;
        chunk_lo.push_back(0);
        double accb = 0;
        int64_t next = 1;
        for (int64_t i = 0; i < c->n_chunks && next < G; i++) {
            accb += chunks[i].bytes;
            if (accb >= tot * next / G) {
                chunk_lo.push_back(i + 1);
                next++;
            }
        }
        while ((int64_t)chunk_lo.size() < G) chunk_lo.push_back(c->n_chunks);
        chunk_lo.push_back(c->n_chunks);
    }
    r2_total = pad4(r2_total);
    std::vector<LargeItem> marg_items;
    std::vector<TileRef> tiles;
    std::vector<int64_t> cta_lo;
    const int ntb[6] = {32, 64, 128, 256, 512, KMAX};
    static const int64_t marg_item_floats =
        getenv("RBA_MARG_ITEM_FLOATS") ? atoll(getenv("RBA_MARG_ITEM_FLOATS")) : 1048576;  // 4 MB of output per item (measured: 3.91 -> 3.34 ms on cfg4 vs 1 MB)
#ifndef RBA_HUGE_ITEM_DEFAULT
#define RBA_HUGE_ITEM_DEFAULT (1 << 20)  // bytes of tiles per fused huge-product item (tuning knob RBA_HUGE_ITEM_BYTES)
#endif
    std::vector<HugeItem> huge_y, huge_out, huge_fused;
    int64_t ybuf_n = 0;
    const int64_t large_lo = pos;
    for (int64_t i = pos; i < nl; i++) {
        const int k = c->h_k[i];
        c->h_r2[i] = r2_total;
        r2_total += large_r2_floats(k);
        c->max_large_k = std::max<int64_t>(c->max_large_k, k);
    }
    for (int cls = 0; cls < 6; cls++) {
        auto in_cls = [&](int k) { return k <= ntb[cls] && (cls == 0 || k > ntb[cls - 1]); };
        c->marg_lo[cls] = (int64_t)marg_items.size();
        const int64_t t_lo = (int64_t)tiles.size();
        double bytes = 0;
        // K2 work item: ~item_floats of emitted output (the O(k) prologue is recomputed per item):
        // 4 MB, but at least ~2 items per SM for a class too small to fill the GPU otherwise (a
        // single 2.8-MB item of a k = 196 track on one CTA was the tail of config 3's K2)
        double cls_floats = 0;
        for (int64_t i = large_lo; i < nl; i++)
            if (in_cls(c->h_k[i])) cls_floats += large_r2_floats(c->h_k[i]);
        const int64_t item_floats = getenv("RBA_MARG_ITEM_FLOATS") ? marg_item_floats :
            std::min<int64_t>(marg_item_floats, std::max<int64_t>(131072, (int64_t)(cls_floats / (2.0 * c->num_sms))));
        for (int64_t i = large_lo; i < nl; i++) {
            const int k = c->h_k[i];
            if (!in_cls(k)) continue;
            const int T = large_tiles(k);
            const int tpi2 = opt.storage ? T : (int)std::max<int64_t>(1, item_floats / (36 * k));
            for (int t0 = 0; t0 < T; t0 += tpi2)
                marg_items.push_back(LargeItem{(int32_t)i, t0, std::min(T, t0 + tpi2), 0});
            if (cls == 5) {
                // huge (k > KLARGE): y pass per tile; out / precond pass per (HUGE_NT camera
                // blocks, ~1 MB of tiles)
                c->huge_max_k = std::max<int64_t>(c->huge_max_k, k);
                for (int t = 0; t < T; t++) huge_y.push_back(HugeItem{(int32_t)i, 0, t, t + 1, ybuf_n});
                for (int o0 = 0; o0 < k; o0 += HUGE_NT)
                    for (int t0 = 0; t0 < T; t0 += HUGE_TPO)
                        huge_out.push_back(HugeItem{(int32_t)i, o0, t0, std::min(T, t0 + HUGE_TPO), ybuf_n});
                // fused product items; yoff = the item's index within its landmark (deterministic mode)
                static const int64_t huge_item = getenv("RBA_HUGE_ITEM_BYTES") ? atoll(getenv("RBA_HUGE_ITEM_BYTES")) : RBA_HUGE_ITEM_DEFAULT;
                const int tpf = (int)std::max<int64_t>(1, huge_item / (144 * k));
                for (int t0 = 0; t0 < T; t0 += tpf)
                    huge_fused.push_back(HugeItem{(int32_t)i, 0, t0, std::min(T, t0 + tpf), (int64_t)(t0 / tpf)});
                ybuf_n += 4 * (int64_t)T;
                continue;
            }
            for (int t = 0; t < T; t++)
                tiles.push_back(TileRef{(int32_t)i, t, c->h_r2[i] + (int64_t)36 * k * t, k, h_obs0[i], 0});
            bytes += 144.0 * k * T;
        }
        c->marg_hi[cls] = (int64_t)marg_items.size();
        if (cls == 5) break;
        const int64_t t_hi = (int64_t)tiles.size();
        // persistent CTAs (one per SM) over contiguous tile ranges balanced by bytes
        c->cta_off[cls] = (int64_t)cta_lo.size();
        const int64_t ntl = t_hi - t_lo;
        const int64_t G = std::min<int64_t>(prop_ctas(c, bytes), ntl);
        c->cta_n[cls] = G;
        if (G > 0) {
            cta_lo.push_back(t_lo);
            double accb = 0;
            int64_t next = 1;
            for (int64_t ti = t_lo; ti < t_hi && next < G; ti++) {
                accb += 144.0 * tiles[ti].k;
                if (accb >= bytes * next / G) {
                    cta_lo.push_back(ti + 1);
                    next++;
                }
            }
            while ((int64_t)cta_lo.size() - c->cta_off[cls] < G) cta_lo.push_back(t_hi);
            cta_lo.push_back(t_hi);
        } else {
            cta_lo.push_back(t_hi);
        }
    }
    int64_t side_total = r2_total;
    for (int64_t i = 0; i < nl; i++) {
        c->h_side[i] = side_total;
        side_total += side_floats(c->h_k[i]);
    }
    c->arena_floats = side_total;
    if (opt.storage == 1) {  // factored (f4): header 44 + 28 per observation floats per landmark
        int64_t off = 0;
        c->matvec_bytes = 0;
        c->marg_bytes = 0;
        c->logical_bytes = 0;
        const int gb[5] = {2, 4, 8, 16, 1 << 30};
        int cls = 0;
        for (int64_t i = 0; i < nl; i++) {
            const int k = c->h_k[i];
            while (k > gb[cls]) {
                c->fac_hi[cls] = i;
                c->fac_lo[++cls] = i;
            }
            c->h_r2[i] = off;
            off += 44 + 28 * (int64_t)k;
            c->matvec_bytes += 176.0 + 112.0 * k;
            c->marg_bytes += 176.0 + 112.0 * k + 20.0 * k;
            c->logical_bytes += 176 + 112 * (int64_t)k;
        }
        for (int q = cls; q < 5; q++) c->fac_hi[q] = nl;
        for (int q = cls + 1; q < 5; q++) c->fac_lo[q] = nl;
        c->fac_big = nl;
        for (int64_t i = 0; i < nl; i++)
            if (c->h_k[i] > 32) {
                c->fac_big = i;
                break;
            }
        c->arena_floats = std::max<int64_t>(off, 4);
    }
    // ---- deterministic mode: slot numbering of the camera-space contributions.  Parts per
    // observation: K5 small-k pack units (row-pair groups of 4), large-pipe consumer runs a track's
    // tiles span (shared by K4 and K5), huge-track tile-range items (separately for K4 and K5).
    // Slots are camera-major: camera i owns [camptrF[i], camptrF[i+1]), its observations in
    // landmark order, each with its parts consecutive.
    std::vector<int32_t> h_slot[3], h_run0;
    std::vector<int64_t> h_cp[3];
    int64_t n_slots[3] = {0, 0, 0};
    if (opt.deterministic) {
        std::vector<int32_t> p4(nl, 1), p5(nl, 1);
        for (int64_t i = 0; i < large_lo; i++) p5[i] = (c->h_k[i] + 3) / 4;
        // consumer runs (CTA b, slot sl) of the large-pipe classes: a run's landmarks other than its
        // first start in it (part 0); its first landmark's part = the runs of that landmark before it
        std::vector<int32_t> cnt(nl, 0);
        for (int cls = 0; cls < 5; cls++) {
            const int NS = PIPE_NSLOT[cls];
            c->run_off[cls] = (int64_t)h_run0.size();
            for (int64_t b = 0; b < c->cta_n[cls]; b++) {
                const int64_t lo = cta_lo[c->cta_off[cls] + b], hi = cta_lo[c->cta_off[cls] + b + 1];
                const int64_t nst = (hi - lo + NS - 1) / NS;
                for (int sl = 0; sl < NS; sl++) {
                    const int64_t a = lo + sl * nst, e = std::min(hi, lo + (sl + 1) * nst);
                    h_run0.push_back(a < e ? cnt[tiles[a].lm] : 0);
                    int32_t prev = -1;
                    for (int64_t t = a; t < e; t++)
                        if (tiles[t].lm != prev) prev = tiles[t].lm, cnt[prev]++;
                }
            }
        }
        for (int64_t i = large_lo; i < nl; i++)
            if (cnt[i] > 0) p5[i] = p4[i] = cnt[i];
        for (auto &it : huge_fused) p5[it.lm] = std::max<int32_t>(p5[it.lm], (int32_t)it.yoff + 1);
        for (auto &it : huge_out) p4[it.lm] = std::max<int32_t>(p4[it.lm], it.t0 / HUGE_TPO + 1);
        std::vector<int32_t> ocam(nobs_loc), olm(nobs_loc);
        for (int64_t i = 0; i < nl; i++)
            for (int o = 0; o < c->h_k[i]; o++) {
                ocam[h_obs0[i] + o] = obs_cam[ord[gptr[loc[i]] + o]];
                olm[h_obs0[i] + o] = (int32_t)i;
            }
        std::vector<int64_t> first(n_cams + 1, 0);  // observations by camera (stable: landmarks ascending)
        for (int64_t ob = 0; ob < nobs_loc; ob++) first[ocam[ob] + 1]++;
        for (int64_t q = 0; q < n_cams; q++) first[q + 1] += first[q];
        std::vector<int64_t> bycam(nobs_loc), fill(first.begin(), first.end() - 1);
        for (int64_t ob = 0; ob < nobs_loc; ob++) bycam[fill[ocam[ob]]++] = ob;
        for (int F = 0; F < 3; F++) {
            const std::vector<int32_t> *parts = F == 1 ? &p4 : (F == 2 ? &p5 : nullptr);
            h_slot[F].assign(std::max<int64_t>(nobs_loc, 1), 0);
            h_cp[F].assign(n_cams + 1, 0);
            int64_t pos = 0;
            for (int64_t q = 0; q < n_cams; q++) {
                h_cp[F][q] = pos;
                for (int64_t m = first[q]; m < first[q + 1]; m++) {
                    const int64_t ob = bycam[m];
                    h_slot[F][ob] = (int32_t)pos;
                    pos += parts ? (*parts)[olm[ob]] : 1;
                }
            }
            h_cp[F][n_cams] = pos;
            n_slots[F] = pos;
            if (pos >= ((int64_t)1 << 31))
                return bail(fail(RBA_ERR_INVALID_ARG, "deterministic mode: too many camera-sum slots for int32"));
        }
    }
    // ---- device buffers
    DevProblem &d = c->d;
    d.n_p = n_cams;
    d.n_l = nl;
    d.huber = opt.huber_delta;
    d.sc = opt.solver;
    d.fac = opt.storage;
    d.s64 = opt.precision;
    d.n_obs = nobs_loc;
    CKSC(dalloc_n(c, &d.cams, 9 * n_cams));
    CKSC(dalloc_n(c, &d.cams_trial, 9 * n_cams));
    CKSC(dalloc_n(c, &d.pts, 3 * nl));
    CKSC(dalloc_n(c, &d.pts_trial, 3 * nl));
    CKSC(dalloc_n(c, &d.campre, CAMPRE * n_cams));
    CKSC(dalloc_n(c, &d.lm_orig, std::max<int64_t>(nl, 1)));
    CKSC(dalloc_n(c, &d.pts_io, 3 * std::max<int64_t>(n_points, 1)));
    if (nl) CKC(cudaMemcpyAsync(d.lm_orig, loc.data(), sizeof(int32_t) * nl, cudaMemcpyHostToDevice, c->stream));
    CKSC(dalloc_n(c, &d.campre_trial, CAMPRE * n_cams));
    CKSC(dalloc_n(c, &d.lm_k, nl));
    CKSC(dalloc_n(c, &d.lm_obs0, nl));
    CKSC(dalloc_n(c, &d.lm_pk, nl));
    CKSC(dalloc_n(c, &d.lm_q, nl));
    CKSC(dalloc_n(c, &d.qpk, q_total + 8));
    CKSC(dalloc_n(c, &d.lm_r2, nl));
    CKSC(dalloc_n(c, &d.lm_side, nl));
    CKSC(dalloc_n(c, &d.obs_cam, nobs_loc + 8));  // +8: 16-byte aligned camera-index bulk copies
    CKSC(dalloc_n(c, &d.obs_lm, nobs_loc));
    CKSC(dalloc_n(c, &d.obs_uv, nobs_loc));
    CKSC(dalloc_n(c, &d.sp, 9 * n_cams));
    CKSC(dalloc_n(c, &d.Dp2, 9 * n_cams));
    CKSC(dalloc_n(c, &d.sp64, 9 * n_cams));
    CKSC(dalloc_n(c, &d.Dp264, 9 * n_cams));
    CKSC(dalloc_n(c, &d.cam_n2d, 9 * n_cams));
    CKSC(dalloc_n(c, &d.lm_s, 3 * nl));
    CKSC(dalloc_n(c, &d.lm_D, 3 * nl));
    if (d.s64) {
        // sqrt-BA-64: row-major FP64 logical blocks + 12 Givens doubles; classes k <= 32, <= 128, else
        int64_t off = 0;
        c->logical_bytes = 0;
        c->matvec_bytes = 0;
        c->marg_bytes = 0;
        const int lim[5] = {32, 128, 256, 512, KMAX64};
        int cls = 0;
        for (int64_t i = 0; i < nl; i++) {
            const int k = c->h_k[i];
            while (k > lim[cls]) {
                c->s64_hi[cls] = i;
                c->s64_lo[++cls] = i;
            }
            c->s64_kmax[cls] = std::max<int64_t>(c->s64_kmax[cls], k);
            c->h_r2[i] = off;  // rows 3..2k+2 (the reduced rows A | q), consecutive over landmarks
            off += (int64_t)(2 * k) * (9 * k + 4);
            c->logical_bytes += (int64_t)(2 * k + 3) * (9 * k + 4) * 8 + 96;
            c->matvec_bytes += 8.0 * 2 * k * (9 * k + 1);  // reduced rows A | q read once
            c->marg_bytes += 8.0 * (2 * k + 3) * (9 * k + 4) + 96 + 40.0 * k;
        }
        for (int64_t i = 0; i < nl; i++) {  // rows 0..2 and the 12 Givens doubles after all reduced rows
            const int k = c->h_k[i];
            c->h_side[i] = off;
            off += (int64_t)3 * (9 * k + 4) + 12;
        }
        for (int q = cls; q < 5; q++) c->s64_hi[q] = nl;
        for (int q = cls + 1; q < 5; q++) c->s64_lo[q] = nl;
        // K2-64 work items: (landmark, pose-row range of ~4 MB of output); the FP32 items are unused
        marg_items.clear();
        for (int q = 0; q < 5; q++) {
            c->s64_ilo[q] = (int64_t)marg_items.size();
            for (int64_t i = c->s64_lo[q]; i < c->s64_hi[q]; i++) {
                const int k = c->h_k[i];
                const int rpi = (int)std::max<int64_t>(8, (int64_t)524288 / (9 * k + 4));
                for (int r = 0; r < 2 * k; r += rpi)
                    marg_items.push_back(LargeItem{(int32_t)i, r, std::min(2 * k, r + rpi), 0});
            }
            c->s64_ihi[q] = (int64_t)marg_items.size();
        }
        std::vector<LargeItem> rcs;  // product items: ~1 MB of the reduced rows 3..2k+2 each
        for (int q = 0; q < 5; q++) {
            c->s64_plo[q] = (int64_t)rcs.size();
            for (int64_t i = c->s64_lo[q]; i < c->s64_hi[q]; i++) {
                const int k = c->h_k[i];
                const int rpi = (int)std::max<int64_t>(8, (int64_t)131072 / (9 * k + 4));
                for (int r = 3; r < 2 * k + 3; r += rpi)
                    rcs.push_back(LargeItem{(int32_t)i, r, std::min(2 * k + 3, r + rpi), 0});
            }
            c->s64_phi[q] = (int64_t)rcs.size();
        }
        {  // class 0 (k <= 32): one item per landmark, in k order; split by group size
            const int gl[4] = {4, 8, 16, 32};
            int64_t pos = c->s64_plo[0];
            for (int g = 0; g < 4; g++) {
                c->s64_glo[g] = pos;
                while (pos < c->s64_phi[0] && c->h_k[rcs[pos].lm] <= gl[g]) pos++;
                c->s64_ghi[g] = pos;
                c->s64_mlo[g] = c->s64_lo[0] + (c->s64_glo[g] - c->s64_plo[0]);  // one item per landmark
                c->s64_mhi[g] = c->s64_lo[0] + (c->s64_ghi[g] - c->s64_plo[0]);
            }
        }
        {  // k <= 16 (groups of 4 / 8 / 16 lanes): TMA batches of consecutive landmarks; their reduced
           // rows are contiguous, so one 16-byte-aligned copy per batch (offsets in doubles; arena64
           // is 16-byte aligned); at most 48 KB, 256 / G landmarks and 256 observations per batch
            std::vector<int4> bat, rec;
            for (int g = 0; g < 3; g++) {
                const int NG = 256 / (4 << g);  // = the consumer groups of k_rcs64_ws (8 warps)
                c->s64_blo[g] = (int64_t)bat.size();
                int64_t i = c->s64_mlo[g];
                while (i < c->s64_mhi[g]) {
                    int n = 0, nob = 0;
                    const int64_t ob0 = h_obs0[i], c_lo = ob0 & ~(int64_t)3, lo = c->h_r2[i] & ~(int64_t)1;
                    int64_t hi = lo;
                    const size_t r0 = rec.size();
                    rec.resize(r0 + 64, int4{0, 0, 0, 0});
                    while (i < c->s64_mhi[g] && n < NG) {
                        const int64_t k = c->h_k[i], W = 9 * k + 4, end = (c->h_r2[i] + 2 * k * W + 1) & ~(int64_t)1;
                        if (end - lo > S64_STAGE_DBL || nob + k > 256) break;
                        rec[r0 + n] = int4{(int)k, (int)(c->h_r2[i] - lo), (int)(h_obs0[i] - c_lo), 0};
                        hi = end;
                        nob += (int)k;
                        n++;
                        i++;
                    }
                    const int64_t c_hi = (ob0 + nob + 3) & ~(int64_t)3;
                    bat.push_back(int4{n, (int)(hi - lo), (int)c_lo, (int)(c_hi - c_lo)});
                    rec.push_back(int4{(int)(lo & 0xffffffff), (int)(lo >> 32), 0, 0});  // slot 64: source
                    rec.resize(r0 + 66, int4{0, 0, 0, 0});
                }
                c->s64_bhi[g] = (int64_t)bat.size();
            }
            CKSC(dalloc_n(c, &d.s64_batches, std::max<size_t>(1, bat.size())));
            CKSC(dalloc_n(c, &d.s64_brec, std::max<size_t>(1, rec.size())));
            if (!bat.empty()) {
                CKC(cudaMemcpyAsync(d.s64_batches, bat.data(), sizeof(int4) * bat.size(), cudaMemcpyHostToDevice,
                                    c->stream));
                CKC(cudaMemcpyAsync(d.s64_brec, rec.data(), sizeof(int4) * rec.size(), cudaMemcpyHostToDevice,
                                    c->stream));
            }
            CKC(cudaStreamSynchronize(c->stream));
        }
        CKSC(dalloc_n(c, &d.rcs_items, std::max<size_t>(1, rcs.size())));
        if (!rcs.empty())
            CKC(cudaMemcpyAsync(d.rcs_items, rcs.data(), sizeof(LargeItem) * rcs.size(), cudaMemcpyHostToDevice,
                                c->stream));
        CKC(cudaStreamSynchronize(c->stream));
        c->arena_floats = 4;
        CKSC(dalloc_n(c, &d.arena64, std::max<int64_t>(off, 1)));
        CKSC(dalloc_n(c, &d.lm_s64, 3 * std::max<int64_t>(nl, 1)));
        CKSC(dalloc_n(c, &d.lm_D64, 3 * std::max<int64_t>(nl, 1)));
    }
    if (d.sc) {
        // explicit SC: no landmark blocks; the covisibility graph of the local landmarks as BSR
        // (both triangles, columns ascending per camera row)
        c->arena_floats = 4;
        std::vector<std::vector<int32_t>> cam_lms(n_cams);
        std::vector<int32_t> hcam(nobs_loc);
        for (int64_t i = 0; i < nl; i++) {
            const int64_t g0 = gptr[loc[i]];
            for (int o = 0; o < c->h_k[i]; o++) {
                hcam[h_obs0[i] + o] = obs_cam[ord[g0 + o]];
                cam_lms[obs_cam[ord[g0 + o]]].push_back((int32_t)i);
            }
        }
        std::vector<int32_t> bptr(n_cams + 1, 0), bcol, mark(n_cams, -1);
        for (int64_t c1 = 0; c1 < n_cams; c1++) {
            const size_t r0 = bcol.size();
            for (int32_t i : cam_lms[c1])
                for (int o = 0; o < c->h_k[i]; o++) {
                    const int32_t c2 = hcam[h_obs0[i] + o];
                    if (mark[c2] != (int32_t)c1) mark[c2] = (int32_t)c1, bcol.push_back(c2);
                }
            if (mark[c1] != (int32_t)c1) bcol.push_back((int32_t)c1);  // diagonal block always present
            std::sort(bcol.begin() + r0, bcol.end());
            bptr[c1 + 1] = (int32_t)bcol.size();
            if (bcol.size() >= (size_t)1 << 31) return bail(fail(RBA_ERR_BAD_PROBLEM, "explicit SC: too many blocks"));
        }
        d.nnzb = (int64_t)bcol.size();
        const size_t ts = d.sc == 2 ? sizeof(double) : sizeof(float);
        CKSC(dalloc_n(c, &d.bsr_ptr, n_cams + 1));
        CKSC(dalloc_n(c, &d.bsr_col, d.nnzb));
        CKSC(dalloc(c, &d.bsr_val, ts * SC_BS * (size_t)d.nnzb));
        CKSC(dalloc(c, &d.sc_b, ts * 9 * (size_t)n_cams));
        CKSC(dalloc(c, &d.sc_scratch, ts * 54 * (size_t)std::max<int64_t>(nobs_loc, 1)));
        CKC(cudaMemcpyAsync(d.bsr_ptr, bptr.data(), sizeof(int32_t) * bptr.size(), cudaMemcpyHostToDevice, c->stream));
        CKC(cudaMemcpyAsync(d.bsr_col, bcol.data(), sizeof(int32_t) * bcol.size(), cudaMemcpyHostToDevice, c->stream));
        CKC(cudaStreamSynchronize(c->stream));  // host staging vectors go out of scope
        c->matvec_bytes = (double)ts * 81 * d.nnzb;       // one read of H~ per product
        c->marg_bytes = (double)ts * 81 * d.nnzb + 48.0 * nobs_loc;
    }
    CKSC(dalloc_n(c, &d.arena, c->arena_floats));
    d.arena_n = c->arena_floats;
    for (int F = 0; F < 3; F++) d.n_slots[F] = n_slots[F];
    {
        int nsm = 0;
        CKSC(dalloc_n(c, &d.pcg, 1));
        CKC(query_nsmid(c, reinterpret_cast<int *>(d.pcg), &nsm));
        d.nslice = std::max(nsm, 1);
        CKC(cudaMemsetAsync(d.pcg, 0, sizeof(PcgState), c->stream));
        CKC(launch_set_pcg_limits(c, opt.pcg_rel_tol, opt.pcg_max_iters));
    }
    CKSC(dalloc_n(c, &d.pcg_part, 2 * ((9 * n_cams + 31) / 32) + 64));
    CKSC(dalloc_n(c, &d.psl, (int64_t)d.nslice * PACC_STRIDE * n_cams));
    CKSC(dalloc_n(c, &d.wsl, (int64_t)d.nslice * 12 * n_cams));
    CKC(cudaMemsetAsync(d.psl, 0, sizeof(float) * d.nslice * PACC_STRIDE * n_cams, c->stream));
    CKC(cudaMemsetAsync(d.wsl, 0, sizeof(float) * d.nslice * 12 * n_cams, c->stream));
    if (d.s64) {
        CKSC(dalloc_n(c, &d.wsl64, (int64_t)d.nslice * 9 * n_cams));
        CKC(cudaMemsetAsync(d.wsl64, 0, sizeof(double) * d.nslice * 9 * n_cams, c->stream));
    }
    CKSC(dalloc_n(c, &d.pd, 54 * n_cams));
    CKSC(dalloc_n(c, &d.wd, 9 * n_cams));
    CKSC(dalloc_n(c, &d.p32, 9 * n_cams));
    CKSC(dalloc_n(c, &d.bt, 9 * n_cams));
    CKSC(dalloc_n(c, &d.Minv, 81 * n_cams));
    CKSC(dalloc_n(c, &d.x, 9 * n_cams));
    CKSC(dalloc_n(c, &d.r, 9 * n_cams));
    CKSC(dalloc_n(c, &d.z, 9 * n_cams));
    CKSC(dalloc_n(c, &d.p, 9 * n_cams));
    CKSC(dalloc_n(c, &d.w, 9 * n_cams));
    CKSC(dalloc_n(c, &d.dl, 3 * nl));
    CKSC(dalloc_n(c, &d.scal, SC_N));
    CKSC(dalloc_n(c, &d.lm, 1));
    d.det = opt.deterministic;
    if (d.det) {
        const int64_t of = std::max({56 * n_slots[1], 12 * n_slots[2], 12 * n_slots[0], (int64_t)16});
        CKSC(dalloc_n(c, &d.obuf, of));
        CKC(cudaMemsetAsync(d.obuf, 0, sizeof(float) * of, c->stream));
        int32_t **sl[3] = {&d.slot1, &d.slot4, &d.slot5};
        int64_t **cp[3] = {&d.camptr1, &d.camptr4, &d.camptr5};
        for (int F = 0; F < 3; F++) {
            CKSC(dalloc_n(c, sl[F], (int64_t)h_slot[F].size()));
            CKSC(dalloc_n(c, cp[F], n_cams + 1));
            CKC(cudaMemcpyAsync(*sl[F], h_slot[F].data(), sizeof(int32_t) * h_slot[F].size(), cudaMemcpyHostToDevice,
                                c->stream));
            CKC(cudaMemcpyAsync(*cp[F], h_cp[F].data(), sizeof(int64_t) * (n_cams + 1), cudaMemcpyHostToDevice,
                                c->stream));
        }
        CKSC(dalloc_n(c, &d.run_part, std::max<int64_t>((int64_t)h_run0.size(), 1)));
        if (!h_run0.empty())
            CKC(cudaMemcpyAsync(d.run_part, h_run0.data(), sizeof(int32_t) * h_run0.size(), cudaMemcpyHostToDevice,
                                c->stream));
        CKSC(dalloc_n(c, &d.det_part, (int64_t)DS_N * DET_PART));
        CKSC(dalloc_n(c, &d.det_ctr, DS_N));
        CKC(cudaMemsetAsync(d.det_ctr, 0, sizeof(unsigned int) * DS_N, c->stream));
        CKC(cudaStreamSynchronize(c->stream));  // host staging vectors go out of scope
    }
    CKSC(dalloc_n(c, &d.reps, rba_ctx::REP_CAP));
    CKSC(dalloc_n(c, &d.packs, std::max<size_t>(1, packs.size())));
    {  // 17 <= k <= 32 with dense FP32 storage: K2 warp per landmark (k_marg_small<32>, tile layout)
        std::vector<Pack> mid;
        if (!opt.storage && !opt.precision && !opt.solver && !getenv("RBA_NO_MID_K2"))
            for (int64_t i = large_lo; i < nl; i++)
                if (c->h_k[i] <= 32) mid.push_back(Pack{(int32_t)i, 1, c->h_r2[i], h_obs0[i], c->h_k[i], 0, 0});
        c->n_mid_packs = (int64_t)mid.size();
        CKSC(dalloc_n(c, &d.mid_packs, std::max<size_t>(1, mid.size())));
        if (!mid.empty())
            CKC(cudaMemcpyAsync(d.mid_packs, mid.data(), sizeof(Pack) * mid.size(), cudaMemcpyHostToDevice, c->stream));
        CKC(cudaStreamSynchronize(c->stream));
    }
    CKSC(dalloc_n(c, &d.marg_items, std::max<size_t>(1, marg_items.size())));
    CKSC(dalloc_n(c, &d.tiles, std::max<size_t>(1, tiles.size())));
    CKSC(dalloc_n(c, &d.cta_lo, std::max<size_t>(1, cta_lo.size())));
    CKSC(dalloc_n(c, &d.chunks, std::max<size_t>(1, chunks.size())));
    CKSC(dalloc_n(c, &d.units, std::max<size_t>(8, units.size())));
    CKSC(dalloc_n(c, &d.chunk_lo, std::max<size_t>(1, chunk_lo.size())));
    c->n_huge_y = (int64_t)huge_y.size();
    c->n_huge_out = (int64_t)huge_out.size();
    c->n_huge_fused = (int64_t)huge_fused.size();
    // the register-resident fused product takes the items of k <= 1024 (2 camera blocks per thread)
    std::stable_partition(huge_fused.begin(), huge_fused.end(),
                          [&](const HugeItem &it) { return c->h_k[it.lm] <= 1024; });
    c->n_huge_reg = std::count_if(huge_fused.begin(), huge_fused.end(),
                                  [&](const HugeItem &it) { return c->h_k[it.lm] <= 1024; });
    CKSC(dalloc_n(c, &d.huge_fused, std::max<size_t>(1, huge_fused.size())));
    CKSC(dalloc_n(c, &d.huge_y, std::max<size_t>(1, huge_y.size())));
    CKSC(dalloc_n(c, &d.huge_out, std::max<size_t>(1, huge_out.size())));
    CKSC(dalloc_n(c, &d.ybuf, std::max<int64_t>(4, ybuf_n)));
    CKC(cudaMallocHost(&c->h_scal, sizeof(double) * SC_N));
    CKC(cudaMallocHost(&c->h_pcg, sizeof(PcgState)));
    CKC(cudaMallocHost(&c->h_reps, sizeof(rba_lm_report) * rba_ctx::REP_CAP));
    // ---- upload (host staging in the device layout)
    {
        std::vector<double> hc(cameras, cameras + 9 * n_cams), hp(3 * std::max<int64_t>(nl, 1));
        for (int64_t i = 0; i < nl; i++)
            for (int q = 0; q < 3; q++) hp[3 * i + q] = points[3 * (int64_t)loc[i] + q];
        std::vector<int32_t> ocam(std::max<int64_t>(nobs_loc, 1)), olm(std::max<int64_t>(nobs_loc, 1));
        std::vector<double2> ouv(std::max<int64_t>(nobs_loc, 1));
        for (int64_t i = 0; i < nl; i++) {
            const int64_t g0 = gptr[loc[i]];
            for (int o = 0; o < c->h_k[i]; o++) {
                const int64_t src = ord[g0 + o];
                const int64_t dst = h_obs0[i] + o;
                ocam[dst] = obs_cam[src];
                olm[dst] = (int32_t)i;
                ouv[dst] = make_double2(obs_uv[2 * src], obs_uv[2 * src + 1]);
            }
        }
        CKC(cudaMemcpyAsync(d.cams, hc.data(), sizeof(double) * hc.size(), cudaMemcpyHostToDevice, c->stream));
        CKC(cudaMemcpyAsync(d.pts, hp.data(), sizeof(double) * 3 * nl, cudaMemcpyHostToDevice, c->stream));
        CKC(cudaMemcpyAsync(d.lm_k, c->h_k.data(), sizeof(int32_t) * nl, cudaMemcpyHostToDevice, c->stream));
        CKC(cudaMemcpyAsync(d.lm_obs0, h_obs0.data(), sizeof(int32_t) * nl, cudaMemcpyHostToDevice, c->stream));
        CKC(cudaMemcpyAsync(d.lm_r2, c->h_r2.data(), sizeof(int64_t) * nl, cudaMemcpyHostToDevice, c->stream));
        CKC(cudaMemcpyAsync(d.lm_side, c->h_side.data(), sizeof(int64_t) * nl, cudaMemcpyHostToDevice, c->stream));
        CKC(cudaMemsetAsync(d.obs_cam + nobs_loc, 0, sizeof(int32_t) * 8, c->stream));
        CKC(cudaMemcpyAsync(d.obs_cam, ocam.data(), sizeof(int32_t) * nobs_loc, cudaMemcpyHostToDevice, c->stream));
        CKC(cudaMemcpyAsync(d.obs_lm, olm.data(), sizeof(int32_t) * nobs_loc, cudaMemcpyHostToDevice, c->stream));
        CKC(cudaMemcpyAsync(d.obs_uv, ouv.data(), sizeof(double2) * nobs_loc, cudaMemcpyHostToDevice, c->stream));
        CKC(cudaMemcpyAsync(d.lm_pk, c->h_pk.data(), sizeof(int32_t) * nl, cudaMemcpyHostToDevice, c->stream));
        CKC(cudaMemcpyAsync(d.lm_q, c->h_q.data(), sizeof(int32_t) * nl, cudaMemcpyHostToDevice, c->stream));
        if (!packs.empty())
            CKC(cudaMemcpyAsync(d.packs, packs.data(), sizeof(Pack) * packs.size(), cudaMemcpyHostToDevice, c->stream));
        if (!marg_items.empty())
            CKC(cudaMemcpyAsync(d.marg_items, marg_items.data(), sizeof(LargeItem) * marg_items.size(),
                                cudaMemcpyHostToDevice, c->stream));
        if (!units.empty())
            CKC(cudaMemcpyAsync(d.units, units.data(), sizeof(uint16_t) * units.size(), cudaMemcpyHostToDevice,
                                c->stream));
        if (!chunks.empty())
            CKC(cudaMemcpyAsync(d.chunks, chunks.data(), sizeof(SmallChunk) * chunks.size(), cudaMemcpyHostToDevice,
                                c->stream));
        CKC(cudaMemcpyAsync(d.chunk_lo, chunk_lo.data(), sizeof(int64_t) * chunk_lo.size(), cudaMemcpyHostToDevice,
                            c->stream));
        if (!huge_y.empty())
            CKC(cudaMemcpyAsync(d.huge_y, huge_y.data(), sizeof(HugeItem) * huge_y.size(), cudaMemcpyHostToDevice,
                                c->stream));
        if (!huge_fused.empty())
            CKC(cudaMemcpyAsync(d.huge_fused, huge_fused.data(), sizeof(HugeItem) * huge_fused.size(),
                                cudaMemcpyHostToDevice, c->stream));
        if (!huge_out.empty())
            CKC(cudaMemcpyAsync(d.huge_out, huge_out.data(), sizeof(HugeItem) * huge_out.size(),
                                cudaMemcpyHostToDevice, c->stream));
        for (TileRef &tr : tiles) tr.tl = c->h_side[tr.lm] + side_tl(tr.k) + 4 * (3 + 4 * (int64_t)tr.t);
        if (!tiles.empty())
            CKC(cudaMemcpyAsync(d.tiles, tiles.data(), sizeof(TileRef) * tiles.size(), cudaMemcpyHostToDevice,
                                c->stream));
        if (!cta_lo.empty())
            CKC(cudaMemcpyAsync(d.cta_lo, cta_lo.data(), sizeof(int64_t) * cta_lo.size(), cudaMemcpyHostToDevice,
                                c->stream));
        CKC(cudaMemsetAsync(d.scal, 0, sizeof(double) * SC_N, c->stream));
        CKC(cudaMemsetAsync(d.lm, 0, sizeof(LmDev), c->stream));
        CKC(launch_lm_init(c, opt.lambda0, 2.0, 1));
        CKC(launch_lm_need_lin(c));
        CKC(launch_set_lambda(c, opt.lambda0));
        // front-of-camera validation at the initial state, in a kernel
        int *dbad = reinterpret_cast<int *>(d.pcg);  // scratch
        CKC(cudaMemsetAsync(dbad, 0, sizeof(int), c->stream));
        CKC(launch_check_depth(c, dbad));
        int hbad = 0;
        CKC(cudaMemcpyAsync(&hbad, dbad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        CKC(cudaStreamSynchronize(c->stream));
        if (hbad) {
            g_err = std::to_string(hbad) + " observation(s) not in front of their camera (P_z >= -1e-8) at the initial state";
            return bail(RBA_ERR_BAD_PROBLEM);
        }
    }
    // world == 1 with an id: a one-rank communicator, so the sharded code path (all-reduces between
    // product and update, captured into the LM graph) runs for real on one GPU
    if (opt.nccl_unique_id) {
        ncclUniqueId id;
        std::memcpy(&id, opt.nccl_unique_id, sizeof(id));
        ncclResult_t r = ncclCommInitRank(&c->comm, opt.world, id, opt.rank);
        if (r != ncclSuccess) {
            g_err = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
            return bail(RBA_ERR_NCCL);
        }
        c->have_comm = true;
    }
    c->emulate_comm = getenv("RBA_EMULATE_COMM") != nullptr;  // test hook (tests/test_gpu_parity.py)
    c->no_graph = getenv("RBA_NO_GRAPH") != nullptr;
    *out = c;
    return RBA_OK;
#undef CKC
#undef CKSC
}

// ------------------------------------------------------------------------------------ helpers
namespace rba {
rba_status allreduce(rba_ctx *c, void *buf, size_t count, ncclDataType_t t) {
    if (!c->have_comm || count == 0) return RBA_OK;
    CKN(ncclAllReduce(buf, buf, count, t, ncclSum, c->comm, c->stream));
    return RBA_OK;
}
}  // namespace rba

static rba_status read_scal(rba_ctx *c) {
    CK(cudaMemcpyAsync(c->h_scal, c->d.scal, sizeof(double) * SC_N, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return RBA_OK;
}

// ------------------------------------------------------------------------------------ steps
extern "C" rba_status rba_linearize(rba_ctx *c) {
    if (!c) return fail(RBA_ERR_INVALID_ARG, "null ctx");
    CK(cudaSetDevice(c->device));
    DevProblem &d = c->d;
    CK(cudaMemsetAsync(d.scal + SC_E, 0, sizeof(double) * 2, c->stream));
    CK(launch_linearize(c));
    CK(launch_reduce_cam_norms(c));
    CKS(allreduce(c, d.cam_n2d, 9 * d.n_p, ncclDouble));
    CKS(allreduce(c, d.scal + SC_E, 2, ncclDouble));
    CK(launch_cam_scale(c));
    CKS(read_scal(c));
    if (c->h_scal[SC_BAD] > 0) return fail(RBA_ERR_BAD_PROBLEM, "a point is not in front of its camera at the current state");
    c->cost = c->h_scal[SC_E];
    c->linearized = true;
    c->marginalized = false;
    c->solved = false;
    c->backsubbed = false;
    c->lm_dirty = true;
    return RBA_OK;
}

extern "C" rba_status rba_marginalize_qr(rba_ctx *c, double lambda) {
    if (!c) return fail(RBA_ERR_INVALID_ARG, "null ctx");
    if (!(lambda >= 0) || !std::isfinite(lambda)) return fail(RBA_ERR_INVALID_ARG, "lambda must be finite and >= 0");
    if (!c->linearized) return fail(RBA_ERR_STATE, "rba_marginalize_qr before rba_linearize");
    CK(cudaSetDevice(c->device));
    nvtxRangePushA("rba_marginalize_qr");
    CK(launch_set_lambda(c, lambda));  // every kernel reads lambda (FP64) from the device
    if (c->d.s64) {  // sqrt-BA-64: marginalize once per linearization, then re-damp in place
        if (!c->marginalized) CK(launch_marg64(c));
        else if (lambda != c->lambda_blocks) CK(launch_redamp64(c));
        c->marginalized = true;
    } else if (c->d.sc) {  // explicit SC: H_ll depends on lambda, so every new lambda re-forms H~
        if (!c->marginalized || lambda != c->lambda_blocks) CK(launch_sc_build(c));
        c->marginalized = true;
    } else if (!c->marginalized) {
        CK(launch_marginalize(c));
        c->marginalized = true;
    } else if (lambda != c->lambda_blocks) {
        CK(launch_redamp(c));
    }
    nvtxRangePop();
    c->lambda_blocks = lambda;
    c->solved = false;
    c->backsubbed = false;
    c->lm_dirty = true;
    return RBA_OK;
}

extern "C" rba_status rba_pcg_solve(rba_ctx *c, rba_pcg_stats *stats) {
    if (!c) return fail(RBA_ERR_INVALID_ARG, "null ctx");
    if (!c->marginalized) return fail(RBA_ERR_STATE, "rba_pcg_solve before rba_marginalize_qr");
    CK(cudaSetDevice(c->device));
    nvtxRangePushA("rba_pcg_solve");
    DevProblem &d = c->d;
    CK(launch_set_lambda(c, c->lambda_blocks));
    CK(cudaMemsetAsync(d.scal + SC_NSPD, 0, sizeof(double), c->stream));
    CK(c->d.sc ? launch_sc_precond(c) : launch_precond_rhs(c));  // (sqrt-BA-64 dispatches inside)
    CKS(allreduce(c, d.pd, 54 * d.n_p, ncclDouble));
    CK(launch_precond_finalize(c));
    CK(launch_pcg_init(c));
    CKS(run_pcg_loop(c));  // the device-side loop (CUDA graph `while` node) or host batches
    CKS(read_scal(c));
    CK(cudaMemcpyAsync(c->h_pcg, d.pcg, sizeof(PcgState), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    nvtxRangePop();
    c->prof_real_matvecs += c->h_pcg->it;
    if (stats) {
        stats->iters = c->h_pcg->it;
        stats->reason = c->h_pcg->reason;
        stats->rel_residual = c->h_pcg->r0 > 0 ? c->h_pcg->rn / c->h_pcg->r0 : 0.0;
    }
    c->solved = true;
    c->backsubbed = false;
    return RBA_OK;
}

extern "C" rba_status rba_backsubstitute(rba_ctx *c) {
    if (!c) return fail(RBA_ERR_INVALID_ARG, "null ctx");
    if (!c->solved) return fail(RBA_ERR_STATE, "rba_backsubstitute before rba_pcg_solve");
    CK(cudaSetDevice(c->device));
    CK(cudaMemsetAsync(c->d.scal + SC_Q1R2, 0, sizeof(double) * 2, c->stream));
    CK(launch_backsub(c));
    c->backsubbed = true;
    return RBA_OK;
}

extern "C" rba_status rba_cost(rba_ctx *c, int at_trial, double *cost) {
    if (!c || !cost) return fail(RBA_ERR_INVALID_ARG, "null argument");
    if (at_trial && !c->backsubbed) return fail(RBA_ERR_STATE, "trial cost before rba_backsubstitute");
    CK(cudaSetDevice(c->device));
    const int slot = at_trial ? SC_ET : SC_E;
    CK(cudaMemsetAsync(c->d.scal + slot, 0, sizeof(double) * 2, c->stream));
    CK(launch_cost(c, at_trial, slot));
    CKS(allreduce(c, c->d.scal + slot, 2, ncclDouble));
    CKS(read_scal(c));
    *cost = c->h_scal[slot + 1] > 0 ? INFINITY : c->h_scal[slot];
    return RBA_OK;
}

// ------------------------------------------------------------------------------------ state
// State I/O: one contiguous copy each way; the landmark permutation (caller order <-> the
// internal k-sorted order) runs on the device (k_pts_permute).
extern "C" rba_status rba_get_state(rba_ctx *c, double *cameras, double *points) {
    if (!c || !cameras || !points) return fail(RBA_ERR_INVALID_ARG, "null argument");
    CK(cudaSetDevice(c->device));
    const DevProblem &d = c->d;
    const int64_t np3 = 3 * c->n_l_global;
    if (c->world > 1) CK(cudaMemsetAsync(d.pts_io, 0, sizeof(double) * std::max<int64_t>(np3, 1), c->stream));
    CK(launch_pts_permute(c, 0));
    CKS(allreduce(c, d.pts_io, np3, ncclDouble));  // every rank owns a disjoint landmark shard
    CK(cudaMemcpyAsync(cameras, d.cams, sizeof(double) * 9 * d.n_p, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(points, d.pts_io, sizeof(double) * np3, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return RBA_OK;
}

extern "C" rba_status rba_set_state(rba_ctx *c, const double *cameras, const double *points) {
    if (!c || !cameras || !points) return fail(RBA_ERR_INVALID_ARG, "null argument");
    CK(cudaSetDevice(c->device));
    const DevProblem &d = c->d;
    CK(cudaMemcpyAsync(d.cams, cameras, sizeof(double) * 9 * d.n_p, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(d.pts_io, points, sizeof(double) * 3 * c->n_l_global, cudaMemcpyHostToDevice, c->stream));
    CK(launch_pts_permute(c, 1));
    CK(cudaStreamSynchronize(c->stream));
    c->linearized = c->marginalized = c->solved = c->backsubbed = false;
    c->lm_dirty = true;
    return RBA_OK;
}

// ------------------------------------------------------------------------------------ hooks
extern "C" rba_status rba_matvec(rba_ctx *c, const float *v, float *outv) {
    if (!c || !v || !outv) return fail(RBA_ERR_INVALID_ARG, "null argument");
    if (!c->marginalized) return fail(RBA_ERR_STATE, "rba_matvec before rba_marginalize_qr");
    CK(cudaSetDevice(c->device));
    CK(launch_matvec(c, v, outv));
    CKS(allreduce(c, c->d.wd, 9 * c->d.n_p, ncclDouble));
    CK(launch_set_lambda(c, c->lambda_blocks));
    CK(launch_add_damping(c, v, outv));
    c->prof_real_matvecs++;
    return RBA_OK;
}

extern "C" rba_status rba_get_rhs(rba_ctx *c, double *b) {
    if (!c || !b) return fail(RBA_ERR_INVALID_ARG, "null argument");
    if (!c->solved) return fail(RBA_ERR_STATE, "rba_get_rhs before rba_pcg_solve");
    CK(cudaMemcpyAsync(b, c->d.bt, sizeof(double) * 9 * c->d.n_p, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return RBA_OK;
}

extern "C" rba_status rba_get_precond(rba_ctx *c, double *blocks) {
    if (!c || !blocks) return fail(RBA_ERR_INVALID_ARG, "null argument");
    if (!c->solved) return fail(RBA_ERR_STATE, "rba_get_precond before rba_pcg_solve");
    if (c->d.sc) return fail(RBA_ERR_STATE, "rba_get_precond: not kept in explicit-SC mode");
    CK(cudaMemcpyAsync(blocks, c->d.pd, sizeof(double) * 54 * c->d.n_p, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return RBA_OK;
}

extern "C" rba_status rba_get_step(rba_ctx *c, double *dp, double *dl) {
    if (!c || !dp || !dl) return fail(RBA_ERR_INVALID_ARG, "null argument");
    if (!c->solved) return fail(RBA_ERR_STATE, "rba_get_step before rba_pcg_solve");
    std::vector<float> l(3 * std::max<int64_t>(c->d.n_l, 1));
    CK(cudaMemcpyAsync(dp, c->d.x, sizeof(double) * 9 * c->d.n_p, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(l.data(), c->d.dl, sizeof(float) * 3 * c->d.n_l, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (int64_t i = 0; i < 3 * c->n_l_global; i++) dl[i] = 0.0;
    if (c->backsubbed)
        for (int64_t i = 0; i < c->d.n_l; i++)
            for (int q = 0; q < 3; q++) dl[3 * (int64_t)c->lm_orig[i] + q] = l[3 * i + q];
    return RBA_OK;
}

extern "C" rba_status rba_get_scaling(rba_ctx *c, double *sp, double *Dp2, double *sl, double *Dl2) {
    if (!c || !sp || !Dp2 || !sl || !Dl2) return fail(RBA_ERR_INVALID_ARG, "null argument");
    if (!c->linearized) return fail(RBA_ERR_STATE, "rba_get_scaling before rba_linearize");
    const int64_t n = 9 * c->d.n_p, m = 3 * std::max<int64_t>(c->d.n_l, 1);
    std::vector<float> s(m), D(m);
    CK(cudaMemcpyAsync(sp, c->d.sp64, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(Dp2, c->d.Dp264, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(s.data(), c->d.lm_s, sizeof(float) * 3 * c->d.n_l, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(D.data(), c->d.lm_D, sizeof(float) * 3 * c->d.n_l, cudaMemcpyDeviceToHost, c->stream));
    std::vector<double> s64, D64;
    if (c->d.s64) {  // the exact FP64 landmark scaling of sqrt-BA-64
        s64.resize(m), D64.resize(m);
        CK(cudaMemcpyAsync(s64.data(), c->d.lm_s64, sizeof(double) * 3 * c->d.n_l, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(D64.data(), c->d.lm_D64, sizeof(double) * 3 * c->d.n_l, cudaMemcpyDeviceToHost, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    for (int64_t i = 0; i < 3 * c->n_l_global; i++) sl[i] = 0.0, Dl2[i] = 0.0;
    if (c->marginalized)
        for (int64_t i = 0; i < c->d.n_l; i++)
            for (int q = 0; q < 3; q++) {
                const double sv = c->d.s64 ? s64[3 * i + q] : s[3 * i + q];
                const double Dv = c->d.s64 ? D64[3 * i + q] : D[3 * i + q];
                sl[3 * (int64_t)c->lm_orig[i] + q] = sv;
                Dl2[3 * (int64_t)c->lm_orig[i] + q] = Dv * Dv;
            }
    return RBA_OK;
}

extern "C" rba_status rba_export_block(rba_ctx *c, int64_t landmark, double *buf, int64_t cap, int64_t *rows,
                                       int64_t *cols) {
    if (!c || !buf || !rows || !cols) return fail(RBA_ERR_INVALID_ARG, "null argument");
    if (landmark < 0 || landmark >= c->n_l_global || c->orig_to_int[landmark] < 0)
        return fail(RBA_ERR_INVALID_ARG, "landmark not owned by this rank");
    if (!c->marginalized) return fail(RBA_ERR_STATE, "rba_export_block before rba_marginalize_qr");
    if (c->d.sc) return fail(RBA_ERR_STATE, "rba_export_block: explicit-SC mode keeps no landmark blocks");
    if (c->d.fac) return fail(RBA_ERR_STATE, "rba_export_block: factored storage keeps no dense blocks");
    if (c->d.s64) {
        const int64_t j = c->orig_to_int[landmark];
        const int k = c->h_k[j];
        const int64_t R = 2 * k + 3, C = 9 * k + 4;
        *rows = R, *cols = C;
        if (cap < R * C) return fail(RBA_ERR_INVALID_ARG, "buffer too small");
        CK(cudaMemcpyAsync(buf, c->d.arena64 + c->h_side[j], sizeof(double) * 3 * C, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(buf + 3 * C, c->d.arena64 + c->h_r2[j], sizeof(double) * (R - 3) * C, cudaMemcpyDeviceToHost,
                           c->stream));
        CK(cudaStreamSynchronize(c->stream));
        return RBA_OK;
    }
    const int64_t j = c->orig_to_int[landmark];
    const int k = c->h_k[j];
    const int64_t R = 2 * k + 3, C = 9 * k + 4;
    *rows = R;
    *cols = C;
    if (cap < R * C) return fail(RBA_ERR_INVALID_ARG, "buffer too small");
    const int32_t pk = c->h_pk[j];
    const int64_t r2n = k <= KSMALL ? small_pack_floats(k, pk >> 8) : large_r2_floats(k);
    std::vector<float> r2(r2n), side(side_floats(k));
    CK(cudaMemcpyAsync(r2.data(), c->d.arena + c->h_r2[j], sizeof(float) * r2.size(), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(side.data(), c->d.arena + c->h_side[j], sizeof(float) * side.size(), cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaStreamSynchronize(c->stream));
    const float *TL = side.data() + side_tl(k);
    for (int64_t row = 0; row < R; row++) {
        double *out = buf + row * C;
        for (int o = 0; o < k; o++)
            for (int q = 0; q < 9; q++)
                out[9 * o + q] = row < 3 ? side[row * 9 * k + 9 * o + q] : r2[r2_index(k, pk, (int)row - 3, o, q)];
        for (int q = 0; q < 4; q++) out[9 * k + q] = TL[4 * row + q];
    }
    return RBA_OK;
}

extern "C" rba_status rba_arena_bytes(rba_ctx *c, int64_t *logical, int64_t *physical) {
    if (!c || !logical || !physical) return fail(RBA_ERR_INVALID_ARG, "null argument");
    if (c->d.sc) {  // explicit SC: the block-sparse H~
        *logical = (int64_t)(c->d.sc == 2 ? 8 : 4) * 81 * c->d.nnzb;
        *physical = (int64_t)(c->d.sc == 2 ? 8 : 4) * SC_BS * c->d.nnzb;
        return RBA_OK;
    }
    *logical = c->logical_bytes;
    *physical = c->d.s64 ? c->logical_bytes : c->arena_floats * 4;
    return RBA_OK;
}

extern "C" rba_status rba_kernel_launches(rba_ctx *c, int64_t *count) {
    if (!c || !count) return fail(RBA_ERR_INVALID_ARG, "null argument");
    *count = c->launches;
    return RBA_OK;
}

extern "C" rba_status rba_profile(rba_ctx *c, int enable) {
    if (!c) return fail(RBA_ERR_INVALID_ARG, "null ctx");
    CK(cudaStreamSynchronize(c->stream));
    for (auto &l : c->prof) {
        c->ev_pool.push_back(l.a);
        c->ev_pool.push_back(l.b);
    }
    c->prof.clear();
    c->prof_real_matvecs = 0;
    c->profiling = enable != 0;
    return RBA_OK;
}

extern "C" rba_status rba_profile_get(rba_ctx *c, int kernel, double *total_ms, int64_t *launches, double *bytes) {
    if (!c || !total_ms || !launches || !bytes || kernel < 0 || kernel >= KID_N)
        return fail(RBA_ERR_INVALID_ARG, "bad argument");
    CK(cudaStreamSynchronize(c->stream));
    double ms = 0, by = 0;
    int64_t n = 0;
    for (auto &l : c->prof)
        if (l.kid == kernel) {
            float t = 0.f;
            CK(cudaEventElapsedTime(&t, l.a, l.b));
            ms += t;
            by += l.bytes;
            n++;
        }
    if (kernel == KID_MATVEC) {
        // PCG launches iterations in batches; launches after convergence exit at once (device-side
        // done flag).  Count only the matvecs that did work; their time includes the no-op ones.
        n = c->prof_real_matvecs;
        by = c->matvec_bytes * (double)n;
    }
    *total_ms = ms;
    *launches = n;
    *bytes = by;
    return RBA_OK;
}
