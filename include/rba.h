/*
 * rba.h -- C ABI of librba.so, the B200 (sm_100a) FP32 hot path of square-root bundle adjustment
 * (sqrt-BA; Demmel, Sommer, Cremers, Usenko, arXiv 2103.01843).  Passages are cited as P:<line>
 * of /root/reference/PAPER.md (LaTeX source of the paper) with the section / equation they fall in.
 *
 * Problem statement (Sec. 4 "Square root bundle adjustment"): state x = (x_p, x_l) with
 * n_p cameras of d_p = 9 parameters each (BAL/Snavely: angle-axis w[3], translation t[3], focal f,
 * radial k1, k2) and n_l landmarks of 3 coordinates; observations j in O(i) with
 * residual r_ij = pi(x_i, X_j) - u_ij, energy E = sum |r_ij|^2 (Eq. ba_energy).
 *
 * Every call below runs its arithmetic in CUDA kernels of this library; there is no CPU fallback.
 * All device work is stream-ordered on the context's stream; only calls that return host values
 * synchronize.  A context is not thread-safe.  Nothing throws across the ABI: every function
 * returns an rba_status and rba_last_error() gives a thread-local message.
 *
 * Multi-GPU (landmark sharding, "parallel for / parallel reduce"): every rank passes the
 * FULL problem and identical options; the context keeps a deterministic LPT shard of whole
 * landmarks (cameras replicated) and all-reduces camera-space partial sums over NCCL.  All ranks
 * must issue the same call sequence (collective semantics).  With world > 1 and
 * nccl_unique_id == NULL the context runs a "virtual shard": it computes only its partial sums and
 * performs no collective (used by single-GPU tests of the sharded decomposition).
 */
#ifndef RBA_H
#define RBA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rba_ctx rba_ctx; /* opaque; owns every device buffer it allocates */

typedef enum {
    RBA_OK = 0,
    RBA_ERR_INVALID_ARG = 1, /* bad option, lambda < 0, null pointer, out-of-range landmark id   */
    RBA_ERR_BAD_PROBLEM = 2, /* index out of range, landmark with k < 2, duplicate (cam, pt),
                                non-finite value, f <= 0, point not in front of a camera (P_z >= -1e-8)
                                at the initial state, unsupported track length        */
    RBA_ERR_STATE = 3,       /* call out of order (e.g. PCG before marginalization)              */
    RBA_ERR_OOM = 4,         /* device allocation failed; rba_last_error() names the bytes       */
    RBA_ERR_CUDA = 5,        /* CUDA runtime error                                               */
    RBA_ERR_NCCL = 6         /* NCCL error                                                       */
} rba_status;

typedef struct {
    int device;                 /* CUDA device ordinal                                          */
    void *stream;               /* cudaStream_t to run on; NULL = a stream owned by the context */
    int world, rank;            /* landmark sharding; world = 1 for a single GPU                */
    const void *nccl_unique_id; /* 128-byte ncclUniqueId broadcast by the caller, or NULL       */
    double lambda0;             /* initial LM damping, 1e-4                             */
    double pcg_rel_tol;         /* PCG: stop when |rho| <= tol |rho_0| (reading C11), 1e-2 */
    int pcg_max_iters;          /* 500                                                  */
    double min_rel_decrease;    /* accept a step iff gain ratio > this (reading C9), 1e-3       */
    double diag_min, diag_max;  /* clamp of D^2 = diag((JS)^T JS) (reading C8), 1e-6/1e32 */
    /* optional device allocator (e.g. torch's caching allocator); NULL = cudaMalloc/cudaFree   */
    void *(*alloc)(size_t bytes, void *alloc_ctx);
    void (*free)(void *ptr, void *alloc_ctx);
    void *alloc_ctx;
    /* robust loss ("Huber norm with a parameter of 1 pixel ... IRLS as in Ceres"): Huber
     * parameter delta in pixels; 0 = squared loss (the default; BASELINE's configs use none).  E
     * becomes sum rho(|r|^2) with rho(s) = s (s <= delta^2) else 2 delta sqrt(s) - delta^2, and every
     * residual / Jacobian row is weighted by sqrt(rho'(|r|^2)) at linearization (IRLS). */
    double huber_delta;
    /* landmark elimination: RBA_SOLVER_SQRTBA (default; nullspace
     * marginalization by QR), or the paper's explicit Schur-complement baselines
     * "explicit-32" / "explicit-64": H~ formed explicitly as 9 x 9 blocks on
     * the covisibility graph in FP32 / FP64, solved by the same PCG / LM.  In the SC modes
     * rba_marginalize_qr forms the Schur complement, rba_export_block is RBA_ERR_STATE, world must be 1 and
     * rba_arena_bytes reports the block-sparse H~. */
    int solver;
    /* landmark-block storage for RBA_SOLVER_SQRTBA: RBA_STORAGE_DENSE (default;
     * the paper's (2k+3) x (9k+4) blocks) or RBA_STORAGE_FACTORED (beyond the
     * paper: Householder vectors, compact-WY T, the 6 damping Givens and the scaled J_p, 176 + 112 k
     * bytes per landmark; the reduced system is applied in O(k)).  Same results up to
     * rounding; rba_export_block is RBA_ERR_STATE in factored mode. */
    int storage;
    /* arithmetic of the landmark blocks for RBA_SOLVER_SQRTBA with dense storage (SURVEY §8f row
     * f2): RBA_PRECISION_FP32 (default, the paper's sqrt-BA-32) or RBA_PRECISION_FP64 (sqrt-BA-64:
     * the (2k+3) x (9k+4) blocks stored row-major in FP64 and every QR / product / back-substitution
     * operation in FP64; track lengths up to 1024).  sqrt-BA-64 computes the camera column norms,
     * the scaling S_p / S_l and the damping diagonals D_p^2 / D_l^2 in FP64 as well (sqrt-BA-32:
     * FP32 values, kept beside FP64 copies of S_p and D_p^2 for the FP64 PCG vectors), and every
     * kernel reads the damping lambda in FP64. */
    int precision;
    /* 1 = bitwise-reproducible camera-space sums (SURVEY §8b "no float atomics"; the paper's
     * "parallel reduce"): every landmark's contribution to a camera sum (K1 camera norms,
     * K4 block-Jacobi blocks and b~, K5 product) is written to its own slot and the slots of a
     * camera are added in a fixed order, and every scalar sum (E, model decrease) is reduced in a
     * fixed order, so two runs on the same input produce identical bits.  0 (default) = per-SM
     * FP32 slices filled by vector atomics (faster; run-to-run differences at FP32 rounding).
     * Only RBA_SOLVER_SQRTBA with dense FP32 storage supports 1 (else RBA_ERR_INVALID_ARG). */
    int deterministic;
} rba_options;

enum { RBA_PRECISION_FP32 = 0, RBA_PRECISION_FP64 = 1 };

enum { RBA_STORAGE_DENSE = 0, RBA_STORAGE_FACTORED = 1 };

enum { RBA_SOLVER_SQRTBA = 0, RBA_SOLVER_EXPLICIT_SC32 = 1, RBA_SOLVER_EXPLICIT_SC64 = 2 };

typedef struct {
    int iters;           /* PCG iterations performed                                          */
    int reason;          /* 0 tolerance reached, 1 max iterations, 2 indefinite (p^T H p <= 0) */
    double rel_residual; /* |rho_k| / |rho_0|                                                  */
} rba_pcg_stats;

typedef struct {
    int64_t iter;        /* LM iteration index; every attempt counts (reading C13)             */
    int accepted;
    int pcg_iters;
    int pcg_reason;
    double cost;         /* E at the start of the iteration                                   */
    double cost_trial;   /* E(x + dx); +inf if a point falls behind a camera (C17)            */
    double cost_after;   /* E after the accept / reject decision                              */
    double model;        /* L(0) - L(dx), reading C10                                          */
    double rho;          /* gain ratio (E - E_trial) / model                                   */
    double lambda;       /* damping used for this attempt                                     */
    double lambda_next;
    int relinearized;    /* 1: this attempt linearized + marginalized; 0: it re-damped the blocks of
                            the previous linearization (backtracking)                 */
    int status;          /* 0 running; 1 converged: this accepted step decreased E by less than ftol E
                            (rba_lm_solve); 2 error: a point is not in front of its camera at
                            the current state                                                     */
    /* per-phase device time of this attempt (ms, %globaltimer stamps taken by the kernels, so
     * valid inside the device-side loop; the paper traces time per iteration) */
    double t_linearize_ms, t_marginalize_ms, t_precond_ms, t_pcg_ms, t_trial_ms, t_total_ms;
    int64_t device_bytes; /* device memory held by the context (its peak: every buffer is allocated
                             by rba_create; the paper traces peak memory)                   */
} rba_lm_report;

/* Fill defaults: device 0, own stream, world 1, lambda0 1e-4, tol 1e-2, 500 iters, 1e-3, 1e-6, 1e32,
 * no robust loss. */
void rba_default_options(rba_options *opt);

/* Create a solver context from the full problem (host FP64, caller-owned, copied; the caller may
 * free them on return).  cameras: n_cams x 9 row-major [w0 w1 w2 t0 t1 t2 f k1 k2] (BAL order);
 * points: n_points x 3; obs_cam / obs_pt: camera / landmark index of each observation; obs_uv:
 * n_obs x 2 pixel coordinates.  Groups observations by landmark into the landmark-block arena
 * ((2k+3) x (9k+4) FP32 per landmark), uploads, and validates (see
 * RBA_ERR_BAD_PROBLEM).  *out is NULL on failure. */
rba_status rba_create(const double *cameras, int64_t n_cams, const double *points, int64_t n_points,
                      const int32_t *obs_cam, const int32_t *obs_pt, const double *obs_uv, int64_t n_obs,
                      const rba_options *opt, rba_ctx **out);
rba_status rba_destroy(rba_ctx *ctx);

/* Linearize at the current state: residuals, E, Jacobian column norms, column scaling
 * s = 1/(1+|c|) (C7) and D^2 (C8); camera norms are all-reduced across ranks.  Must precede
 * rba_marginalize_qr whenever the state changed. */
rba_status rba_linearize(rba_ctx *ctx);

/* Nullspace marginalization of every landmark block: in-place Householder QR
 * of the landmark columns (3 reflectors), with LM landmark damping sqrt(lambda) D_l folded
 * in by 6 Givens rotations.  At an unchanged linearization only the damping is
 * undone and re-applied (backtracking).  lambda >= 0 else RBA_ERR_INVALID_ARG. */
rba_status rba_marginalize_qr(rba_ctx *ctx, double lambda);

/* Solve the reduced camera system H~ dp = -b~ with block-Jacobi PCG, H~ applied
 * matrix-free as (Q^_2^T J_p)^T (Q^_2^T J_p) v + lambda D_p^2 v (Eq. cg_mult).  dp stays
 * on the device.  stats may be NULL. */
rba_status rba_pcg_solve(rba_ctx *ctx, rba_pcg_stats *stats);

/* Landmark back-substitution dl = -R^_1^-1 (Q^_1^T r + Q^_1^T J_p dp) (Eq. backsub_nm, P:222-226,
 * P:353-354); forms the trial state x + S dx and the model-decrease terms of reading C10. */
rba_status rba_backsubstitute(rba_ctx *ctx);

/* E (Eq. ba_energy) at the current state (at_trial = 0) or at the trial state (1).  Synchronizes. */
rba_status rba_cost(rba_ctx *ctx, int at_trial, double *cost);

/* One LM iteration = linearize (if the state changed) -> marginalize / re-damp -> PCG ->
 * back-substitute -> trial cost -> accept / reject and lambda update (C9, C10, C13).
 * The LM schedule (lambda, nu, current E, accept decision) lives on the device and is advanced by
 * a control kernel; on a single GPU the whole iteration is one CUDA graph (conditional nodes for
 * relinearize-vs-re-damp and the PCG loop), so the only host synchronization is the copy of the
 * report.  RBA_ERR_BAD_PROBLEM if a point is not in front of its camera at the current state.
 * report may be NULL. */
rba_status rba_lm_step(rba_ctx *ctx, rba_lm_report *report);

/* The LM loop of the paper's experiments: up to max_iters iterations (every attempt
 * counts, C13), terminating early once an accepted step decreases E by less than ftol * E
 * ("relative function tolerance"; 1e-6 in the paper).  Runs on the device without host
 * round trips (a CUDA graph `while` node around the iteration) except for the final copy of the
 * reports.  reports: caller array of max_iters entries (may be NULL); *n_done: iterations run.
 * max_iters >= 0, ftol >= 0 else RBA_ERR_INVALID_ARG. */
rba_status rba_lm_solve(rba_ctx *ctx, int max_iters, double ftol, rba_lm_report *reports, int *n_done);

/* Full state on every rank (host FP64, caller buffers n_cams x 9 and n_points x 3). */
rba_status rba_get_state(rba_ctx *ctx, double *cameras, double *points);
/* Replace the state (host FP64); the next LM step relinearizes.  LM damping state is kept. */
rba_status rba_set_state(rba_ctx *ctx, const double *cameras, const double *points);
/* Restart the LM schedule: lambda = lambda0, nu = 2, iteration counter 0. */
rba_status rba_reset_lm(rba_ctx *ctx);
/* Set / read the LM schedule (lambda > 0, nu >= 1; with the state, this replays an iteration).
 * rba_get_lm synchronizes. */
rba_status rba_set_lm(rba_ctx *ctx, double lambda, double nu);
rba_status rba_get_lm(rba_ctx *ctx, double *lambda, double *nu, int64_t *iter);
/* Change the PCG stopping rule (reading C11) for the following solves: |rho| <= rel_tol |rho_0| or
 * max_iters iterations.  rel_tol = 0 with max_iters = n runs exactly n iterations (unless the
 * system is indefinite): the replay rule of the parity protocol.  rel_tol >= 0,
 * max_iters >= 0 else RBA_ERR_INVALID_ARG. */
rba_status rba_set_pcg_limits(rba_ctx *ctx, double rel_tol, int max_iters);

/* ---- test / measurement hooks ----------------------------------------------------------- */
/* out = H~ v (incl. lambda D_p^2 v at the damping currently folded in); v, out: device FP32 9 n_cams. */
rba_status rba_matvec(rba_ctx *ctx, const float *v_dev, float *out_dev);
/* b~ = sum_j A_j^T q_j (host FP64, 9 n_cams), valid after rba_pcg_solve. */
rba_status rba_get_rhs(rba_ctx *ctx, double *b);
/* The camera-space sums of the last preconditioner pass (host FP64, n_cams x 54): the 45 upper-
 * triangle entries (row-major, i <= j) of sum_j A_j[:,i]^T A_j[:,i] (the block-Jacobi block of
 * camera i without lambda D_p^2) followed by the 9 entries of b~_i.  Valid after
 * rba_pcg_solve. */
rba_status rba_get_precond(rba_ctx *ctx, double *blocks);
/* scaled steps dp (9 n_cams) and dl (3 n_points, caller's landmark order; entries of landmarks
 * owned by other ranks are 0). */
rba_status rba_get_step(rba_ctx *ctx, double *dp, double *dl);
/* column scaling and damping diagonals (host FP64): sp, Dp2 (9 n_cams); sl, Dl2 (3 n_points). */
rba_status rba_get_scaling(rba_ctx *ctx, double *sp, double *Dp2, double *sl, double *Dl2);
/* Logical (2k+3) x (9k+4) landmark block of landmark `landmark` (caller's index) in its current
 * state, row-major, into host_buf (capacity `cap` doubles); *rows, *cols receive the shape.
 * RBA_ERR_INVALID_ARG if the landmark is not owned by this rank or cap is too small. */
rba_status rba_export_block(rba_ctx *ctx, int64_t landmark, double *host_buf, int64_t cap, int64_t *rows,
                            int64_t *cols);
/* Landmark-block bytes: logical = sum (2k+3)(9k+4)*4 + 48 per landmark (6 Givens pairs);
 * physical = bytes allocated for the arena (16-byte alignment padding included). */
rba_status rba_arena_bytes(rba_ctx *ctx, int64_t *logical, int64_t *physical);
/* Number of this library's kernel launches so far (kernel nodes executed inside CUDA graphs
 * included, counted per executed conditional branch / loop iteration). */
rba_status rba_kernel_launches(rba_ctx *ctx, int64_t *count);
/* Execution facts of a context (for tests and the benchmark line). */
typedef struct {
    int lm_graph;          /* 1: LM iterations run as one CUDA graph; 0: eager (host-driven); -1: the
                              graph failed to build / instantiate and the eager path is used     */
    int pcg_graph;         /* the same for the step-by-step rba_pcg_solve                          */
    int nccl;              /* 1: an NCCL communicator is attached (all-reduces issued)              */
    int deterministic;
    int64_t n_landmarks;   /* landmarks of this rank's shard                                       */
    int64_t n_observations;
} rba_info;
rba_status rba_get_info(rba_ctx *ctx, rba_info *info);
/* 64-bit FNV-1a checksums of the bit patterns of the camera-space vectors every rank must hold
 * identically after their all-reduces (SURVEY §8e lockstep): [0] the camera column norms^2 of the
 * last linearization, [1] the block-Jacobi partials + b~ of the last preconditioner pass, [2] the
 * last product wd, [3] the PCG solution dp.  Synchronizes. */
rba_status rba_checksums(rba_ctx *ctx, uint64_t out[4]);
/* Device memory held by the context (bytes of every buffer it allocated). */
rba_status rba_device_bytes(rba_ctx *ctx, int64_t *bytes);
/* Algorithmic bytes of one marginalization (K2: the landmark blocks written + the
 * observations read) and of one reduced-camera-system product (K5: the reduced rows read once). */
rba_status rba_plan_bytes(rba_ctx *ctx, double *marginalize_bytes, double *matvec_bytes);
/* Per-kernel CUDA-event timing on the context stream: enable (1) / disable (0) and reset. */
rba_status rba_profile(rba_ctx *ctx, int enable);
/* kernel: 0 linearize(K1), 1 marginalize(K2), 2 damp(K3), 3 precond+rhs(K4), 4 matvec(K5),
 * 5 pcg update(K6), 6 backsub(K7), 7 cost(K8).  Synchronizes.  Outputs total ms, launch count and
 * algorithmic bytes moved (per SURVEY §8d-3 / DESIGN.md §5) summed over the recorded launches.  For
 * the matvec, `launches` counts only matvecs that did work (PCG iterations run in batches and the
 * ones issued after convergence exit immediately); total_ms still includes those no-op launches. */
rba_status rba_profile_get(rba_ctx *ctx, int kernel, double *total_ms, int64_t *launches, double *bytes);
/* Deterministic LPT landmark partition (host only, no GPU): owner[j] in [0, world) for track
 * lengths k[j]; balances block bytes (2k+3)(9k+4). */
rba_status rba_plan_shards(const int32_t *k, int64_t n_landmarks, int world, int32_t *owner);
/* NCCL bootstrap helper: writes a fresh 128-byte ncclUniqueId (call on rank 0 only). */
rba_status rba_nccl_unique_id(void *id128);
/* Thread-local description of the last error. */
const char *rba_last_error(void);

/* ---- BAL ingest and the paper's preprocessing (host only, no GPU) ---------------
 * A BAL problem in host memory, FP64, arrays allocated by librba (release with rba_bal_free).
 * Layout as rba_create expects: cameras n_cams x 9 [w t f k1 k2], points n_points x 3,
 * obs_cam / obs_pt n_obs, obs_uv n_obs x 2.  Errors: RBA_ERR_BAD_PROBLEM with the offending line
 * (rba_bal_last_error), RBA_ERR_INVALID_ARG for null arguments / unreadable files. */
typedef struct {
    int64_t n_cams, n_points, n_obs;
    double *cameras, *points, *obs_uv;
    int32_t *obs_cam, *obs_pt;
} rba_bal;
/* Parse BAL text: header "n_cams n_points n_obs", n_obs lines "cam pt u v", 9 numbers per camera,
 * 3 per point.  Counts come from the header; observation order is preserved.  Reads at most
 * `len` bytes (text need not be NUL-terminated). */
rba_status rba_bal_parse(const char *text, size_t len, rba_bal *out);
/* Read a BAL file, plain text or gzip-compressed (zlib). */
rba_status rba_bal_read(const char *path, rba_bal *out);
/* Write BAL text (%.17g, so parse(write(p)) reproduces p exactly). */
rba_status rba_bal_write(const char *path, const rba_bal *p);
/* Gauge normalization: subtract the per-axis median of the points and scale so that the
 * median over points of the L1 distance to it becomes target_mad (100 in the paper; reading C25);
 * cameras follow the similarity (centre C = -R^T t moved and scaled, rotation kept), so every
 * reprojection residual is unchanged.  RBA_ERR_BAD_PROBLEM if that median is 0. */
rba_status rba_bal_normalize(rba_bal *p, double target_mad);
/* Seeded Gaussian perturbation in FP64: angle-axis += N(0, sigma_rot^2), camera
 * centre += N(0, sigma_centre^2) (translation recomputed), points += N(0, sigma_point^2); a
 * counter-based generator, so the result depends only on (problem, sigmas, seed). */
rba_status rba_bal_perturb(rba_bal *p, double sigma_rot, double sigma_centre, double sigma_point, uint64_t seed);
/* Observation filter: keep an observation iff its depth -P_z in the camera frame
 * (BAL cameras look down -z) exceeds z_min; then drop landmarks with fewer than 2 remaining
 * observations (and their observations), reindexing landmarks densely in their original order.
 * Counts of what was removed go to *removed_obs / *removed_points (may be NULL). */
rba_status rba_bal_filter(rba_bal *p, double z_min, int64_t *removed_obs, int64_t *removed_points);
void rba_bal_free(rba_bal *p);
const char *rba_bal_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* RBA_H */
