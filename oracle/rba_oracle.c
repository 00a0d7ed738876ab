/*
 * rba_oracle.c -- plain, slow, FP64 CPU oracle for the square-root bundle adjustment (sqrt-BA)
 * hot path of Demmel et al., "Square Root Bundle Adjustment for Large-Scale Reconstruction"
 * (arXiv 2103.01843; /root/reference/PAPER.md, cited as P:<line>).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header, table or helper with
 * the CUDA product path (paper_2103_01843_b200/csrc); the only common module is the seeded input
 * generator (paper_2103_01843_b200/synth.py), which holds none of the method's arithmetic.
 *
 * What it computes, in the paper's order and notation:
 *   O1 linearize        r, J_p, J_l per observation at x^0                 (Eq. linearized_residual)
 *   O2 scaling / D      Jacobian column scaling s = 1/(1+|c|), D^2 = clamp(|c|^2 s^2)  (C7, C8)
 *   O3 landmark blocks  dense (2k+3) x (9k+4) [J_p | J_l | r] per landmark  (Fig. 2)
 *   O4 QR               in-place Givens QR, 6k-6 rotations (Appendix A.1 P:550-571 with reading C5/C6)
 *   O5 damping          6 Givens rotations folding sqrt(lambda) D_l, stored; undo (Fig. 3)
 *   O6 reduced system   H~ = sum A^T A + lambda D_p^2,  b~ = sum A^T q       (Eq. cg_mult)
 *   O7 PCG              block-Jacobi preconditioned CG on H~ dp = -b~        (C11, C12)
 *   O8 back-subst.      dl = -R1^-1 (Q1^T r + Q1^T J_p dp)                   (Eq. backsub_nm)
 *   O9 LM               cost E = sum |r|^2 (Eq. ba_energy), gain ratio, lambda update (C9, C10, C13)
 * Readings of silent / garbled passages (C1..C22) are listed in DESIGN.md and SURVEY.md §8c.
 *
 * Parity pins (tests/test_oracle_*.py): golden projection values, central finite
 * differences of the Jacobians, Givens golden (3,4)->(0.6,0.8),5, Q orthogonality / nullspace
 * (P:105-119), explicit damped Schur complement computed independently in numpy,
 * dense Cholesky solve of H~ at PCG tol 1e-12, SC back-substitution, and a brute-force dense
 * least-squares solve of Eq. linearized_residual on small problems.
 * Every exported function below is pinned by at least one of those tests.
 *
 * Deterministic: OpenMP parallel-for over landmarks / cameras, every reduction in a fixed order.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define DP 9 /* pose dimensionality d_p = 9 (BAL/Snavely camera) */

typedef struct {
    int64_t n_p, n_l, n_obs;
    /* state x = (x_p, x_l) and trial state x + dx */
    double *cams, *pts, *cams_trial, *pts_trial;
    /* observations grouped by landmark: CSR, cameras ascending within a landmark */
    int64_t *lm_ptr;   /* n_l+1 */
    int32_t *o_cam;    /* n_obs, CSR order */
    double *o_uv;      /* 2 n_obs, CSR order */
    int64_t *o_src;    /* CSR position -> caller's observation index */
    int64_t *o_lm;     /* CSR position -> landmark */
    /* observations grouped by camera (for fixed-order scatter sums): list of CSR positions */
    int64_t *cam_ptr;  /* n_p+1 */
    int64_t *cam_obs;  /* n_obs: CSR positions sorted by (camera, landmark) */
    /* linearization (unscaled) */
    double *r, *Jc, *Jl; /* 2, 18, 6 per observation */
    double *sp, *Dp2, *sl, *Dl2;
    double cost;          /* E(x) */
    /* landmark blocks */
    int64_t *blk_off;     /* n_l+1, offsets in doubles */
    double *blk;
    double *giv;          /* 12 per landmark: 6 x (c, s) */
    int linearized, marginalized, damped;
    double lambda;        /* damping currently folded into the blocks */
    /* reduced system / PCG */
    double *bt;           /* b~, 9 n_p */
    double *Lp;           /* Cholesky factor of the block-Jacobi blocks, 81 n_p */
    double *dp, *rho_cg;  /* pose step (scaled), final CG residual */
    double *dl;           /* landmark step (scaled), 3 n_l */
    double *y;            /* scratch for matvec: 2k per landmark (offsets 2*lm_ptr) */
    /* model-decrease terms (C10) */
    double q1r2, damp_l;
    double cost_trial;
    /* LM */
    double lm_lambda, lm_nu;
    /* robust loss: Huber with parameter delta (pixels), 0 = squared loss */
    double huber;
    int need_linearize;
    int64_t iteration;
    /* streaming mode (SURVEY §8c "Oracle capacity"): no block arena; every operation that reads a
     * landmark block re-assembles, re-factorizes and re-damps it (O3-O5) in a per-thread scratch,
     * identical arithmetic, O(threads) memory -- for problems whose FP64 blocks do not fit in host
     * memory (config 5: 263 GB). */
    int streaming;
    int64_t max_block; /* doubles of the largest block */
} orc_ctx;

typedef struct {
    int64_t iter;
    int accepted;
    int pcg_iters;
    int pcg_reason; /* 0 tol, 1 max iters, 2 indefinite (p^T H p <= 0) */
    double cost;    /* E at the start of the iteration */
    double cost_trial;
    double cost_after; /* E after the accept/reject decision (C13) */
    double model;   /* L(0) - L(dx), C10 */
    double rho;     /* gain ratio */
    double lambda;  /* lambda used for this attempt */
    double lambda_next;
} orc_lm_report;

/* ------------------------------------------------------------------------------------------
 * Camera model: BAL / Snavely (readings C1, C2, C22).
 * cam = [w0 w1 w2 t0 t1 t2 f k1 k2],  P = R(w) X + t,  p = -P_xy / P_z,
 * d = 1 + k1 |p|^2 + k2 |p|^4,  pi = f d p,  r = pi - u.
 * ---------------------------------------------------------------------------------------- */
static void rodrigues(const double w[3], double R[9], double Jleft[9]) {
    double th2 = w[0] * w[0] + w[1] * w[1] + w[2] * w[2];
    double th = sqrt(th2);
    double K[9] = {0, -w[2], w[1], w[2], 0, -w[0], -w[1], w[0], 0};
    double K2[9];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
            double s = 0;
            for (int m = 0; m < 3; m++) s += K[3 * i + m] * K[3 * m + j];
            K2[3 * i + j] = s;
        }
    double a, b, c; /* R = I + a K + b K^2 ; Jleft = I + b K + c K^2 */
    if (th < 1e-8) {
        a = 1.0; b = 0.5; c = 1.0 / 6.0;
    } else {
        a = sin(th) / th;
        b = (1.0 - cos(th)) / th2;
        c = (th - sin(th)) / (th2 * th);
    }
    for (int i = 0; i < 9; i++) {
        double I = (i % 4 == 0) ? 1.0 : 0.0;
        R[i] = I + a * K[i] + b * K2[i];
        if (Jleft) Jleft[i] = I + b * K[i] + c * K2[i];
    }
}

/* Projection only.  Returns P_z through *Pz.  0 on success, 1 if P_z == 0. */
int orc_project(const double *cam, const double *X, double *uv, double *Pz) {
    double R[9];
    rodrigues(cam, R, NULL);
    double P[3];
    for (int i = 0; i < 3; i++) P[i] = R[3 * i] * X[0] + R[3 * i + 1] * X[1] + R[3 * i + 2] * X[2] + cam[3 + i];
    if (Pz) *Pz = P[2];
    if (P[2] == 0.0) return 1;
    double px = -P[0] / P[2], py = -P[1] / P[2];
    double n = px * px + py * py;
    double d = 1.0 + cam[7] * n + cam[8] * n * n;
    uv[0] = cam[6] * d * px;
    uv[1] = cam[6] * d * py;
    return 0;
}

/* Residual r = pi - u and analytic Jacobians J_cam (2x9, row-major) and J_lm (2x3). */
int orc_residual_jacobian(const double *cam, const double *X, const double *u, double *r, double *Jc,
                          double *Jl) {
    double R[9], JL[9];
    rodrigues(cam, R, JL);
    double RX[3], P[3];
    for (int i = 0; i < 3; i++) {
        RX[i] = R[3 * i] * X[0] + R[3 * i + 1] * X[1] + R[3 * i + 2] * X[2];
        P[i] = RX[i] + cam[3 + i];
    }
    if (P[2] == 0.0) return 1;
    double f = cam[6], k1 = cam[7], k2 = cam[8];
    double px = -P[0] / P[2], py = -P[1] / P[2];
    double n = px * px + py * py;
    double d = 1.0 + k1 * n + k2 * n * n;
    r[0] = f * d * px - u[0];
    r[1] = f * d * py - u[1];
    /* dpi/dp = f (d I + 2 (k1 + 2 k2 n) p p^T) */
    double e = 2.0 * (k1 + 2.0 * k2 * n);
    double Dpi[4] = {f * (d + e * px * px), f * e * px * py, f * e * px * py, f * (d + e * py * py)};
    /* dp/dP = -(1/P_z) [[1,0,px],[0,1,py]] */
    double iz = -1.0 / P[2];
    double DpP[6] = {iz, 0, iz * px, 0, iz, iz * py};
    double DpiP[6]; /* 2x3 */
    for (int i = 0; i < 2; i++)
        for (int j = 0; j < 3; j++) DpiP[3 * i + j] = Dpi[2 * i] * DpP[j] + Dpi[2 * i + 1] * DpP[3 + j];
    /* dP/dw = -[RX]_x Jleft(w)  (additive angle-axis update, C1) */
    double S[9] = {0, -RX[2], RX[1], RX[2], 0, -RX[0], -RX[1], RX[0], 0};
    double DPw[9];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
            double s = 0;
            for (int m = 0; m < 3; m++) s += S[3 * i + m] * JL[3 * m + j];
            DPw[3 * i + j] = -s;
        }
    for (int i = 0; i < 2; i++) {
        for (int j = 0; j < 3; j++) {
            double s = 0, sl = 0;
            for (int m = 0; m < 3; m++) {
                s += DpiP[3 * i + m] * DPw[3 * m + j];
                sl += DpiP[3 * i + m] * R[3 * m + j];
            }
            Jc[9 * i + j] = s;               /* d/dw */
            Jc[9 * i + 3 + j] = DpiP[3 * i + j]; /* d/dt, dP/dt = I */
            Jl[3 * i + j] = sl;              /* d/dX, dP/dX = R */
        }
        double pi_ = (i == 0) ? px : py;
        Jc[9 * i + 6] = d * pi_;          /* d/df  */
        Jc[9 * i + 7] = f * n * pi_;      /* d/dk1 */
        Jc[9 * i + 8] = f * n * n * pi_;  /* d/dk2 */
    }
    return 0;
}

/* Huber norm ("Huber norm with a parameter of 1 pixel ... implemented with IRLS as in
 * Ceres"), on the squared residual norm s = |r|^2:  rho(s) = s for s <= delta^2, else
 * 2 delta sqrt(s) - delta^2.  IRLS weight (Ceres' corrector with rho'' = 0): the residual and its
 * Jacobian rows are multiplied by sqrt(rho'(s)), rho'(s) = 1 for s <= delta^2, else delta/sqrt(s).
 * delta <= 0: squared loss. */
double orc_huber_rho(double s, double delta) {
    if (delta <= 0.0 || s <= delta * delta) return s;
    return 2.0 * delta * sqrt(s) - delta * delta;
}
double orc_huber_weight(double s, double delta) {
    if (delta <= 0.0 || s <= delta * delta) return 1.0;
    return sqrt(delta / sqrt(s));
}

/* Givens coefficients, reading C5 of the garbled appendix formula:
 * pivot value a (= a_pp), target value b (= a_tp);  rho = hypot(a, b), c = a/rho, s = b/rho;
 * new_pivot = c*pivot + s*target, new_target = -s*pivot + c*target  zeroes the target entry.
 * b == 0 gives the identity rotation (c=1, s=0). */
void orc_givens(double a, double b, double *c, double *s, double *rho) {
    if (b == 0.0) {
        *c = 1.0; *s = 0.0; *rho = a;
        return;
    }
    double r = hypot(a, b);
    *c = a / r; *s = b / r; *rho = r;
}

static void rot_rows(double *rp, double *rt, int64_t ncol, double c, double s) {
    for (int64_t j = 0; j < ncol; j++) {
        double p = rp[j], t = rt[j];
        rp[j] = c * p + s * t;
        rt[j] = -s * p + c * t;
    }
}

/* ------------------------------------------------------------------------------------------
 * Context
 * ---------------------------------------------------------------------------------------- */
static int cmp_i64_pair(const void *a, const void *b) {
    const int64_t *x = a, *y = b;
    if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
    if (x[1] != y[1]) return x[1] < y[1] ? -1 : 1;
    return 0;
}

void orc_destroy(orc_ctx *c);

orc_ctx *orc_create(const double *cams, int64_t n_p, const double *pts, int64_t n_l, const int32_t *obs_cam,
                    const int32_t *obs_pt, const double *obs_uv, int64_t n_obs) {
    orc_ctx *c = calloc(1, sizeof(orc_ctx));
    c->n_p = n_p; c->n_l = n_l; c->n_obs = n_obs;
    c->cams = malloc(sizeof(double) * DP * n_p);
    c->cams_trial = malloc(sizeof(double) * DP * n_p);
    c->pts = malloc(sizeof(double) * 3 * n_l);
    c->pts_trial = malloc(sizeof(double) * 3 * n_l);
    memcpy(c->cams, cams, sizeof(double) * DP * n_p);
    memcpy(c->pts, pts, sizeof(double) * 3 * n_l);
    /* CSR by landmark, cameras ascending */
    int64_t *key = malloc(sizeof(int64_t) * 3 * n_obs);
    for (int64_t i = 0; i < n_obs; i++) {
        key[3 * i] = obs_pt[i];
        key[3 * i + 1] = obs_cam[i];
        key[3 * i + 2] = i;
    }
    qsort(key, n_obs, 3 * sizeof(int64_t), cmp_i64_pair);
    c->lm_ptr = calloc(n_l + 1, sizeof(int64_t));
    c->o_cam = malloc(sizeof(int32_t) * n_obs);
    c->o_uv = malloc(sizeof(double) * 2 * n_obs);
    c->o_src = malloc(sizeof(int64_t) * n_obs);
    for (int64_t i = 0; i < n_obs; i++) {
        int64_t src = key[3 * i + 2];
        c->lm_ptr[key[3 * i] + 1]++;
        c->o_cam[i] = (int32_t)key[3 * i + 1];
        c->o_uv[2 * i] = obs_uv[2 * src];
        c->o_uv[2 * i + 1] = obs_uv[2 * src + 1];
        c->o_src[i] = src;
    }
    for (int64_t j = 0; j < n_l; j++) c->lm_ptr[j + 1] += c->lm_ptr[j];
    c->o_lm = malloc(sizeof(int64_t) * n_obs);
    for (int64_t j = 0; j < n_l; j++)
        for (int64_t o = c->lm_ptr[j]; o < c->lm_ptr[j + 1]; o++) c->o_lm[o] = j;
    /* by camera, landmarks ascending */
    for (int64_t i = 0; i < n_obs; i++) {
        key[3 * i] = c->o_cam[i];
        key[3 * i + 1] = i; /* CSR position is monotone in landmark */
        key[3 * i + 2] = 0;
    }
    qsort(key, n_obs, 3 * sizeof(int64_t), cmp_i64_pair);
    c->cam_ptr = calloc(n_p + 1, sizeof(int64_t));
    c->cam_obs = malloc(sizeof(int64_t) * n_obs);
    for (int64_t i = 0; i < n_obs; i++) {
        c->cam_ptr[key[3 * i] + 1]++;
        c->cam_obs[i] = key[3 * i + 1];
    }
    for (int64_t i = 0; i < n_p; i++) c->cam_ptr[i + 1] += c->cam_ptr[i];
    free(key);

    c->r = malloc(sizeof(double) * 2 * n_obs);
    c->Jc = malloc(sizeof(double) * 18 * n_obs);
    c->Jl = malloc(sizeof(double) * 6 * n_obs);
    c->sp = malloc(sizeof(double) * DP * n_p);
    c->Dp2 = malloc(sizeof(double) * DP * n_p);
    c->sl = malloc(sizeof(double) * 3 * n_l);
    c->Dl2 = malloc(sizeof(double) * 3 * n_l);
    c->blk_off = malloc(sizeof(int64_t) * (n_l + 1));
    c->blk_off[0] = 0;
    for (int64_t j = 0; j < n_l; j++) {
        int64_t k = c->lm_ptr[j + 1] - c->lm_ptr[j];
        c->blk_off[j + 1] = c->blk_off[j] + (2 * k + 3) * (DP * k + 4);
        if ((2 * k + 3) * (DP * k + 4) > c->max_block) c->max_block = (2 * k + 3) * (DP * k + 4);
    }
    c->blk = NULL; /* allocated by the first orc_linearize (orc_scaling needs no blocks) */
    c->giv = calloc(12 * n_l, sizeof(double));
    c->bt = malloc(sizeof(double) * DP * n_p);
    c->Lp = malloc(sizeof(double) * 81 * n_p);
    c->dp = calloc(DP * n_p, sizeof(double));
    c->rho_cg = calloc(DP * n_p, sizeof(double));
    c->dl = calloc(3 * n_l, sizeof(double));
    c->y = malloc(sizeof(double) * 2 * n_obs);
    c->lm_lambda = 1e-4;
    c->lm_nu = 2.0;
    c->need_linearize = 1;
    return c;
}

void orc_destroy(orc_ctx *c) {
    if (!c) return;
    free(c->cams); free(c->pts); free(c->cams_trial); free(c->pts_trial);
    free(c->lm_ptr); free(c->o_cam); free(c->o_uv); free(c->o_src); free(c->o_lm); free(c->cam_ptr); free(c->cam_obs);
    free(c->r); free(c->Jc); free(c->Jl); free(c->sp); free(c->Dp2); free(c->sl); free(c->Dl2);
    free(c->blk_off); free(c->blk); free(c->giv); free(c->bt); free(c->Lp); free(c->dp); free(c->rho_cg);
    free(c->dl); free(c->y);
    free(c);
}

int64_t orc_block_offset(orc_ctx *c, int64_t j) { return c->blk_off[j]; }
int64_t orc_track_length(orc_ctx *c, int64_t j) { return c->lm_ptr[j + 1] - c->lm_ptr[j]; }
int64_t orc_block_doubles(orc_ctx *c) { return c->blk_off[c->n_l]; }

static double clampd(double x, double lo, double hi) { return x < lo ? lo : (x > hi ? hi : x); }

/* E(x) = sum rho(|r_ij|^2) (Eq. ba_energy, no 1/2: C3; rho = identity unless Huber).  +inf if a point is at or
 * behind a camera (P_z >= 0, C17). */
static double cost_at(orc_ctx *c, const double *cams, const double *pts) {
    double *per = malloc(sizeof(double) * c->n_l);
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t j = 0; j < c->n_l; j++) {
        double s = 0;
        for (int64_t o = c->lm_ptr[j]; o < c->lm_ptr[j + 1]; o++) {
            double uv[2], Pz;
            orc_project(cams + DP * c->o_cam[o], pts + 3 * j, uv, &Pz);
            if (!(Pz < 0.0)) { s = INFINITY; break; }
            double dx = uv[0] - c->o_uv[2 * o], dy = uv[1] - c->o_uv[2 * o + 1];
            s += orc_huber_rho(dx * dx + dy * dy, c->huber);
        }
        per[j] = s;
    }
    double E = 0;
    for (int64_t j = 0; j < c->n_l; j++) E += per[j];
    free(per);
    return E;
}

double orc_cost(orc_ctx *c) { return cost_at(c, c->cams, c->pts); }

/* O1-O2: linearize at the current state (residuals, Jacobians, E) and compute the column scaling
 * and damping diagonals.  Needs no landmark blocks (used alone on problems whose FP64 blocks do
 * not fit in host memory). */
int orc_scaling(orc_ctx *c) {
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(| : bad)
    for (int64_t j = 0; j < c->n_l; j++)
        for (int64_t o = c->lm_ptr[j]; o < c->lm_ptr[j + 1]; o++)
            bad |= orc_residual_jacobian(c->cams + DP * c->o_cam[o], c->pts + 3 * j, c->o_uv + 2 * o,
                                         c->r + 2 * o, c->Jc + 18 * o, c->Jl + 6 * o);
    if (bad) return 1;
    /* IRLS: weight residual and Jacobian rows by sqrt(rho'(|r|^2)) */
    if (c->huber > 0.0) {
#pragma omp parallel for schedule(static)
        for (int64_t o = 0; o < c->n_obs; o++) {
            double *r = c->r + 2 * o;
            double w = orc_huber_weight(r[0] * r[0] + r[1] * r[1], c->huber);
            r[0] *= w, r[1] *= w;
            for (int q = 0; q < 18; q++) c->Jc[18 * o + q] *= w;
            for (int q = 0; q < 6; q++) c->Jl[6 * o + q] *= w;
        }
    }
    c->cost = orc_cost(c);
    /* column norms of the full Jacobian; camera columns summed over the camera's observations */
#pragma omp parallel for
    for (int64_t i = 0; i < c->n_p; i++) {
        for (int q = 0; q < DP; q++) {
            double s = 0;
            for (int64_t m = c->cam_ptr[i]; m < c->cam_ptr[i + 1]; m++) {
                int64_t o = c->cam_obs[m];
                s += c->Jc[18 * o + q] * c->Jc[18 * o + q] + c->Jc[18 * o + 9 + q] * c->Jc[18 * o + 9 + q];
            }
            double sc = 1.0 / (1.0 + sqrt(s)); /* C7 */
            c->sp[DP * i + q] = sc;
            c->Dp2[DP * i + q] = clampd(s * sc * sc, 1e-6, 1e32); /* C8 */
        }
    }
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t j = 0; j < c->n_l; j++) {
        for (int q = 0; q < 3; q++) {
            double s = 0;
            for (int64_t o = c->lm_ptr[j]; o < c->lm_ptr[j + 1]; o++)
                s += c->Jl[6 * o + q] * c->Jl[6 * o + q] + c->Jl[6 * o + 3 + q] * c->Jl[6 * o + 3 + q];
            double sc = 1.0 / (1.0 + sqrt(s));
            c->sl[3 * j + q] = sc;
            c->Dl2[3 * j + q] = clampd(s * sc * sc, 1e-6, 1e32);
        }
    }
    return 0;
}

/* O3 for one landmark: block (Fig. 2b): rows 2i,2i+1 = obs i; pose cols 9i..9i+8;
 * landmark cols 9k..9k+2; residual col 9k+3; 3 zero damping rows at the bottom. */
static void block_assemble(const orc_ctx *c, int64_t j, double *B) {
    int64_t k = c->lm_ptr[j + 1] - c->lm_ptr[j];
    int64_t W = DP * k + 4;
    memset(B, 0, sizeof(double) * (2 * k + 3) * W);
    for (int64_t i = 0; i < k; i++) {
        int64_t o = c->lm_ptr[j] + i;
        int cam = c->o_cam[o];
        for (int rr = 0; rr < 2; rr++) {
            double *row = B + (2 * i + rr) * W;
            for (int q = 0; q < DP; q++) row[DP * i + q] = c->Jc[18 * o + 9 * rr + q] * c->sp[DP * cam + q];
            for (int q = 0; q < 3; q++) row[DP * k + q] = c->Jl[6 * o + 3 * rr + q] * c->sl[3 * j + q];
            row[DP * k + 3] = c->r[2 * o + rr];
        }
    }
}

/* O4 for one landmark: in-place Givens QR of the landmark columns (Appendix A.1; C5,
 * C6): column l = 0..2, target rows i = 2k-1 down to l+1 against pivot row l: 6k-6 rotations. */
static void block_qr(int64_t k, double *B) {
    int64_t W = DP * k + 4;
    for (int l = 0; l < 3; l++)
        for (int64_t i = 2 * k - 1; i > l; i--) {
            double cs, sn, rho;
            orc_givens(B[l * W + DP * k + l], B[i * W + DP * k + l], &cs, &sn, &rho);
            if (sn == 0.0) continue;
            rot_rows(B + l * W, B + i * W, W, cs, sn);
            B[i * W + DP * k + l] = 0.0; /* exact zero below the diagonal (Fig. 2c) */
        }
}

/* O5 for one landmark (Fig. 3): damping rows 2k+q get sqrt(lambda) D_l,q in landmark
 * column q; 6 rotations (pivot,target) = (0,2k),(1,2k),(2,2k),(1,2k+1),(2,2k+1),(2,2k+2) eliminate
 * them; the (c,s) pairs go to g (12 doubles) to undo later. */
static const int DAMP_P[6] = {0, 1, 2, 1, 2, 2};
static const int DAMP_T[6] = {0, 0, 0, 1, 1, 2}; /* target = 2k + DAMP_T */
static void block_damp(const orc_ctx *c, int64_t j, double *B, double lambda, double *g) {
    int64_t k = c->lm_ptr[j + 1] - c->lm_ptr[j];
    int64_t W = DP * k + 4;
    double sl = sqrt(lambda);
    for (int q = 0; q < 3; q++) B[(2 * k + q) * W + DP * k + q] = sl * sqrt(c->Dl2[3 * j + q]);
    for (int m = 0; m < 6; m++) {
        int p = DAMP_P[m];
        double *rp = B + p * W, *rt = B + (2 * k + DAMP_T[m]) * W;
        double cs, sn, rho;
        orc_givens(rp[DP * k + p], rt[DP * k + p], &cs, &sn, &rho);
        g[2 * m] = cs;
        g[2 * m + 1] = sn;
        if (sn != 0.0) {
            rot_rows(rp, rt, W, cs, sn);
            rt[DP * k + p] = 0.0;
        }
    }
}

/* undo (Fig. 3c): transposed rotations in reverse order, then zero the damping rows */
static void block_undamp(int64_t k, double *B, const double *g) {
    int64_t W = DP * k + 4;
    for (int m = 5; m >= 0; m--) rot_rows(B + DAMP_P[m] * W, B + (2 * k + DAMP_T[m]) * W, W, g[2 * m], -g[2 * m + 1]);
    memset(B + 2 * k * W, 0, sizeof(double) * 3 * W);
}

/* The current block of landmark j: the arena's, or (streaming mode) O3-O5 recomputed into
 * `scratch` (max_block doubles) at the damping currently in force; g receives its rotations. */
static const double *lm_block(orc_ctx *c, int64_t j, double *scratch, double *g) {
    if (!c->streaming) {
        if (g) memcpy(g, c->giv + 12 * j, sizeof(double) * 12);
        return c->blk + c->blk_off[j];
    }
    int64_t k = c->lm_ptr[j + 1] - c->lm_ptr[j];
    double gl[12];
    block_assemble(c, j, scratch);
    block_qr(k, scratch);
    if (c->damped) block_damp(c, j, scratch, c->lambda, gl);
    else for (int m = 0; m < 6; m++) gl[2 * m] = 1.0, gl[2 * m + 1] = 0.0;
    if (g) memcpy(g, gl, sizeof(gl));
    return scratch;
}

/* per-thread scratch for lm_block (streaming mode); NULL otherwise */
static double *lm_scratch(orc_ctx *c) { return c->streaming ? malloc(sizeof(double) * (size_t)c->max_block) : NULL; }

/* Streaming mode on (1) / off (0).  Takes effect at the next linearization. */
void orc_set_streaming(orc_ctx *c, int on) {
    c->streaming = on;
    c->need_linearize = 1;
    c->linearized = c->marginalized = c->damped = 0;
    c->lambda = 0;
    if (on && c->blk) { free(c->blk); c->blk = NULL; }
}

/* O1-O3: orc_scaling, then assemble the (undamped, unmarginalized) landmark blocks.
 * Returns 1 on a degenerate projection, 3 if the blocks cannot be allocated. */
int orc_linearize(orc_ctx *c) {
    if (orc_scaling(c)) return 1;
    if (c->streaming) {
        c->linearized = 1;
        c->marginalized = 0;
        c->damped = 0;
        c->lambda = 0;
        return 0;
    }
    if (!c->blk) {
        c->blk = malloc(sizeof(double) * (size_t)c->blk_off[c->n_l]);
        if (!c->blk) return 3;
    }
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t j = 0; j < c->n_l; j++) block_assemble(c, j, c->blk + c->blk_off[j]);
    c->linearized = 1;
    c->marginalized = 0;
    c->damped = 0;
    c->lambda = 0;
    return 0;
}

/* O4: in-place Givens QR of the landmark columns (Appendix A.1; C5, C6):
 * column l = 0..2, target rows i = 2k-1 down to l+1 against pivot row l: 6k-6 rotations. */
int orc_marginalize(orc_ctx *c) {
    if (!c->linearized || c->marginalized) return 2;
    if (!c->streaming) {
#pragma omp parallel for schedule(dynamic, 64)
        for (int64_t j = 0; j < c->n_l; j++) block_qr(c->lm_ptr[j + 1] - c->lm_ptr[j], c->blk + c->blk_off[j]);
    }
    c->marginalized = 1;
    return 0;
}

/* O5: landmark damping (Fig. 3) of every block (block_damp); undo (block_undamp). */
int orc_undamp(orc_ctx *c) {
    if (!c->marginalized) return 2;
    if (!c->damped) return 0;
    if (!c->streaming) {
#pragma omp parallel for schedule(dynamic, 64)
        for (int64_t j = 0; j < c->n_l; j++)
            block_undamp(c->lm_ptr[j + 1] - c->lm_ptr[j], c->blk + c->blk_off[j], c->giv + 12 * j);
    }
    c->damped = 0;
    c->lambda = 0;
    return 0;
}

int orc_damp(orc_ctx *c, double lambda) {
    if (!c->marginalized) return 2;
    if (!(lambda >= 0)) return 1;
    if (c->damped) orc_undamp(c);
    if (!c->streaming) {
#pragma omp parallel for schedule(dynamic, 64)
        for (int64_t j = 0; j < c->n_l; j++) block_damp(c, j, c->blk + c->blk_off[j], lambda, c->giv + 12 * j);
    }
    c->damped = 1;
    c->lambda = lambda;
    return 0;
}

/* A_j = rows 3..2k+2 x pose columns (Q^_2^T J_p); q_j = rows 3..2k+2 of the residual column. */
#define AJ(B, W, a, col) ((B)[(3 + (a)) * (W) + (col)])

/* O6: dense reduced system (test-sized problems only): H~ = sum_j A_j^T A_j + lambda D_p^2 and
 * b~ = sum_j A_j^T q_j.  H is (9 n_p)^2 row-major. */
int orc_reduced_dense(orc_ctx *c, double *H, double *b) {
    if (!c->marginalized || c->streaming) return 2;
    int64_t N = DP * c->n_p;
    memset(H, 0, sizeof(double) * N * N);
    memset(b, 0, sizeof(double) * N);
    for (int64_t j = 0; j < c->n_l; j++) {
        int64_t k = c->lm_ptr[j + 1] - c->lm_ptr[j];
        int64_t W = DP * k + 4;
        const double *B = c->blk + c->blk_off[j];
        for (int64_t o1 = 0; o1 < k; o1++) {
            int64_t c1 = c->o_cam[c->lm_ptr[j] + o1];
            for (int q1 = 0; q1 < DP; q1++) {
                double sb = 0;
                for (int64_t a = 0; a < 2 * k; a++) sb += AJ(B, W, a, DP * o1 + q1) * AJ(B, W, a, DP * k + 3);
                b[DP * c1 + q1] += sb;
                for (int64_t o2 = 0; o2 < k; o2++) {
                    int64_t c2 = c->o_cam[c->lm_ptr[j] + o2];
                    for (int q2 = 0; q2 < DP; q2++) {
                        double s = 0;
                        for (int64_t a = 0; a < 2 * k; a++) s += AJ(B, W, a, DP * o1 + q1) * AJ(B, W, a, DP * o2 + q2);
                        H[(DP * c1 + q1) * N + DP * c2 + q2] += s;
                    }
                }
            }
        }
    }
    for (int64_t i = 0; i < N; i++) H[i * N + i] += c->lambda * c->Dp2[i];
    return 0;
}

/* O6 implicit: out = H~ v = sum_j A_j^T (A_j v_j) + lambda D_p^2 v  (Eq. cg_mult).
 * Pass 1 (per landmark): y_j = A_j v_j.  Pass 2 (per camera, landmarks ascending): gather
 * A_j[:,o]^T y_j.  Fixed summation order. */
void orc_products(orc_ctx *c, int nvec, const double *V, double *out);

void orc_matvec(orc_ctx *c, const double *v, double *out) {
    if (c->streaming) {
        orc_products(c, 1, v, out);
        return;
    }
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t j = 0; j < c->n_l; j++) {
        int64_t k = c->lm_ptr[j + 1] - c->lm_ptr[j];
        int64_t W = DP * k + 4;
        const double *B = c->blk + c->blk_off[j];
        double *y = c->y + 2 * c->lm_ptr[j];
        for (int64_t a = 0; a < 2 * k; a++) {
            double s = 0;
            for (int64_t o = 0; o < k; o++) {
                const double *vc = v + DP * c->o_cam[c->lm_ptr[j] + o];
                for (int q = 0; q < DP; q++) s += AJ(B, W, a, DP * o + q) * vc[q];
            }
            y[a] = s;
        }
    }
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t i = 0; i < c->n_p; i++) {
        double acc[DP] = {0};
        for (int64_t m = c->cam_ptr[i]; m < c->cam_ptr[i + 1]; m++) {
            int64_t pos = c->cam_obs[m];
            int64_t j = c->o_lm[pos], o = pos - c->lm_ptr[j];
            int64_t k = c->lm_ptr[j + 1] - c->lm_ptr[j];
            int64_t W = DP * k + 4;
            const double *B = c->blk + c->blk_off[j];
            const double *y = c->y + 2 * c->lm_ptr[j];
            for (int q = 0; q < DP; q++) {
                double s = 0;
                for (int64_t a = 0; a < 2 * k; a++) s += AJ(B, W, a, DP * o + q) * y[a];
                acc[q] += s;
            }
        }
        for (int q = 0; q < DP; q++) out[DP * i + q] = acc[q] + c->lambda * c->Dp2[DP * i + q] * v[DP * i + q];
    }
}

/* O6 for several vectors in one pass over the landmarks (each block read / recomputed once):
 * out[t] = sum_j A_j^T (A_j v_t) + lambda D_p^2 v_t for the nvec vectors V[t] (9 n_p each).  Every
 * thread owns a contiguous landmark range and accumulates into its own buffer; the buffers are
 * added in thread order (a fixed order for a fixed thread count).  Used by the streaming mode's
 * product and by batched probes. */
void orc_products(orc_ctx *c, int nvec, const double *V, double *out) {
    const int64_t N = DP * c->n_p;
    int T = 1;
#ifdef _OPENMP
    T = omp_get_max_threads();
#endif
    double *acc = calloc((size_t)T * nvec * N, sizeof(double));
#pragma omp parallel num_threads(T)
    {
        int t = 0;
#ifdef _OPENMP
        t = omp_get_thread_num();
#endif
        double *mine = acc + (size_t)t * nvec * N;
        double *scratch = lm_scratch(c);
        double *y = malloc(sizeof(double) * 2 * (size_t)(c->max_block > 0 ? c->max_block : 1));
        const int64_t j0 = c->n_l * t / T, j1 = c->n_l * (t + 1) / T;
        for (int64_t j = j0; j < j1; j++) {
            int64_t k = c->lm_ptr[j + 1] - c->lm_ptr[j];
            int64_t W = DP * k + 4;
            const double *B = lm_block(c, j, scratch, NULL);
            for (int v = 0; v < nvec; v++) {
                const double *vv = V + (size_t)v * N;
                for (int64_t a = 0; a < 2 * k; a++) {
                    double s = 0;
                    for (int64_t o = 0; o < k; o++) {
                        const double *vc = vv + DP * c->o_cam[c->lm_ptr[j] + o];
                        for (int q = 0; q < DP; q++) s += AJ(B, W, a, DP * o + q) * vc[q];
                    }
                    y[a] = s;
                }
                double *dst = mine + (size_t)v * N;
                for (int64_t o = 0; o < k; o++) {
                    double *oc = dst + DP * c->o_cam[c->lm_ptr[j] + o];
                    for (int q = 0; q < DP; q++) {
                        double s = 0;
                        for (int64_t a = 0; a < 2 * k; a++) s += AJ(B, W, a, DP * o + q) * y[a];
                        oc[q] += s;
                    }
                }
            }
        }
        free(scratch);
        free(y);
    }
    for (int v = 0; v < nvec; v++)
        for (int64_t i = 0; i < N; i++) {
            double s = 0;
            for (int t = 0; t < T; t++) s += acc[((size_t)t * nvec + v) * N + i];
            out[(size_t)v * N + i] = s + c->lambda * c->Dp2[i] * V[(size_t)v * N + i];
        }
    free(acc);
}

/* streaming mode: sum_j A_j[:,o]^T A_j[:,o] and A_j[:,o]^T q_j per camera (81 + 9 per camera),
 * per-thread buffers over contiguous landmark ranges, added in thread order */
static void stream_precond_sums(orc_ctx *c, double *Pall, double *ball) {
    int T = 1;
#ifdef _OPENMP
    T = omp_get_max_threads();
#endif
    const size_t per = (size_t)90 * c->n_p;
    double *acc = calloc((size_t)T * per, sizeof(double));
#pragma omp parallel num_threads(T)
    {
        int t = 0;
#ifdef _OPENMP
        t = omp_get_thread_num();
#endif
        double *mine = acc + (size_t)t * per;
        double *scratch = lm_scratch(c);
        const int64_t j0 = c->n_l * t / T, j1 = c->n_l * (t + 1) / T;
        for (int64_t j = j0; j < j1; j++) {
            int64_t k = c->lm_ptr[j + 1] - c->lm_ptr[j];
            int64_t W = DP * k + 4;
            const double *B = lm_block(c, j, scratch, NULL);
            for (int64_t o = 0; o < k; o++) {
                double *P = mine + 90 * (size_t)c->o_cam[c->lm_ptr[j] + o], *bb = P + 81;
                for (int q1 = 0; q1 < DP; q1++) {
                    double sb = 0;
                    for (int64_t a = 0; a < 2 * k; a++) sb += AJ(B, W, a, DP * o + q1) * AJ(B, W, a, DP * k + 3);
                    bb[q1] += sb;
                    for (int q2 = 0; q2 < DP; q2++) {
                        double s = 0;
                        for (int64_t a = 0; a < 2 * k; a++) s += AJ(B, W, a, DP * o + q1) * AJ(B, W, a, DP * o + q2);
                        P[DP * q1 + q2] += s;
                    }
                }
            }
        }
        free(scratch);
    }
    for (int64_t i = 0; i < c->n_p; i++)
        for (int e = 0; e < 90; e++) {
            double s = 0;
            for (int t = 0; t < T; t++) s += acc[(size_t)t * per + 90 * (size_t)i + e];
            if (e < 81) Pall[81 * i + e] = s;
            else ball[DP * i + e - 81] = s;
        }
    free(acc);
}

/* O6/O7: b~ and the block-Jacobi preconditioner P_i = sum_j A_j[:,i]^T A_j[:,i] + lambda D_p,i^2
 * (C12), factored by Cholesky.  Returns 0, or 3 if a block is not SPD. */
int orc_precond_rhs(orc_ctx *c) {
    if (!c->marginalized) return 2;
    int bad = 0;
    double *Ps = NULL, *bs = NULL;
    if (c->streaming) {
        Ps = malloc(sizeof(double) * 81 * c->n_p);
        bs = malloc(sizeof(double) * DP * c->n_p);
        stream_precond_sums(c, Ps, bs);
    }
#pragma omp parallel for schedule(dynamic, 4) reduction(| : bad)
    for (int64_t i = 0; i < c->n_p; i++) {
        double P[81] = {0}, bb[DP] = {0};
        if (c->streaming) {
            memcpy(P, Ps + 81 * i, sizeof(P));
            memcpy(bb, bs + DP * i, sizeof(bb));
        }
        for (int64_t m = c->streaming ? c->cam_ptr[i + 1] : c->cam_ptr[i]; m < c->cam_ptr[i + 1]; m++) {
            int64_t pos = c->cam_obs[m];
            int64_t j = c->o_lm[pos], o = pos - c->lm_ptr[j];
            int64_t k = c->lm_ptr[j + 1] - c->lm_ptr[j];
            int64_t W = DP * k + 4;
            const double *B = c->blk + c->blk_off[j];
            for (int q1 = 0; q1 < DP; q1++) {
                double sb = 0;
                for (int64_t a = 0; a < 2 * k; a++) sb += AJ(B, W, a, DP * o + q1) * AJ(B, W, a, DP * k + 3);
                bb[q1] += sb;
                for (int q2 = 0; q2 < DP; q2++) {
                    double s = 0;
                    for (int64_t a = 0; a < 2 * k; a++) s += AJ(B, W, a, DP * o + q1) * AJ(B, W, a, DP * o + q2);
                    P[DP * q1 + q2] += s;
                }
            }
        }
        for (int q = 0; q < DP; q++) {
            c->bt[DP * i + q] = bb[q];
            P[DP * q + q] += c->lambda * c->Dp2[DP * i + q];
        }
        /* Cholesky P = L L^T, L lower, row-major */
        double *L = c->Lp + 81 * i;
        memset(L, 0, sizeof(double) * 81);
        for (int a = 0; a < DP; a++)
            for (int bcol = 0; bcol <= a; bcol++) {
                double s = P[DP * a + bcol];
                for (int m = 0; m < bcol; m++) s -= L[DP * a + m] * L[DP * bcol + m];
                if (a == bcol) {
                    if (!(s > 0)) { bad = 1; s = 1.0; }
                    L[DP * a + a] = sqrt(s);
                } else {
                    L[DP * a + bcol] = s / L[DP * bcol + bcol];
                }
            }
    }
    free(Ps);
    free(bs);
    return bad ? 3 : 0;
}

static void precond_apply(orc_ctx *c, const double *in, double *out) {
#pragma omp parallel for
    for (int64_t i = 0; i < c->n_p; i++) {
        const double *L = c->Lp + 81 * i;
        double t[DP];
        for (int a = 0; a < DP; a++) {
            double s = in[DP * i + a];
            for (int m = 0; m < a; m++) s -= L[DP * a + m] * t[m];
            t[a] = s / L[DP * a + a];
        }
        for (int a = DP - 1; a >= 0; a--) {
            double s = t[a];
            for (int m = a + 1; m < DP; m++) s -= L[DP * m + a] * out[DP * i + m];
            out[DP * i + a] = s / L[DP * a + a];
        }
    }
}

static double dot(const double *a, const double *b, int64_t n) {
    double s = 0;
    for (int64_t i = 0; i < n; i++) s += a[i] * b[i];
    return s;
}

/* O7: PCG on H~ dp = -b~ from dp = 0 (reading C11: stop when |rho| <= tol |rho_0|,
 * or at max_iters; p^T H p <= 0 -> indefinite).  Returns iterations; reason/relres out. */
int orc_pcg(orc_ctx *c, double tol, int max_iters, int *reason, double *relres) {
    int64_t N = DP * c->n_p;
    double *rho = c->rho_cg, *z = malloc(sizeof(double) * N), *p = malloc(sizeof(double) * N),
           *w = malloc(sizeof(double) * N);
    for (int64_t i = 0; i < N; i++) { c->dp[i] = 0; rho[i] = -c->bt[i]; }
    double r0 = sqrt(dot(rho, rho, N));
    int it = 0;
    *reason = 0;
    *relres = 0;
    if (r0 == 0.0) goto done;
    precond_apply(c, rho, z);
    memcpy(p, z, sizeof(double) * N);
    double rz = dot(rho, z, N);
    for (;;) {
        if (it >= max_iters) { *reason = 1; break; }
        orc_matvec(c, p, w);
        double pw = dot(p, w, N);
        if (!(pw > 0)) { *reason = 2; break; }
        double alpha = rz / pw;
        for (int64_t i = 0; i < N; i++) { c->dp[i] += alpha * p[i]; rho[i] -= alpha * w[i]; }
        it++;
        double rn = sqrt(dot(rho, rho, N));
        *relres = rn / r0;
        if (rn <= tol * r0) { *reason = 0; break; }
        precond_apply(c, rho, z);
        double rz2 = dot(rho, z, N);
        double beta = rz2 / rz;
        rz = rz2;
        for (int64_t i = 0; i < N; i++) p[i] = z[i] + beta * p[i];
    }
done:
    free(z); free(p); free(w);
    return it;
}

/* O8: back-substitution dl_j = -R^_1^{-1}(Q^_1^T r^ + Q^_1^T J_p dp_j) and the
 * model-decrease partials sum |Q^_1^T r^|^2 and lambda sum |D_l dl|^2 (C10). */
int orc_backsub(orc_ctx *c) {
    if (!c->marginalized) return 2;
    double *q1 = malloc(sizeof(double) * c->n_l), *dd = malloc(sizeof(double) * c->n_l);
#pragma omp parallel
    {
    double *scratch = lm_scratch(c);
#pragma omp for schedule(dynamic, 256)
    for (int64_t j = 0; j < c->n_l; j++) {
        int64_t k = c->lm_ptr[j + 1] - c->lm_ptr[j];
        int64_t W = DP * k + 4;
        const double *B = lm_block(c, j, scratch, NULL);
        double rhs[3];
        double s2 = 0;
        for (int a = 0; a < 3; a++) {
            double s = B[a * W + DP * k + 3];
            s2 += s * s;
            for (int64_t o = 0; o < k; o++) {
                const double *d = c->dp + DP * c->o_cam[c->lm_ptr[j] + o];
                for (int q = 0; q < DP; q++) s += B[a * W + DP * o + q] * d[q];
            }
            rhs[a] = s;
        }
        double x[3];
        for (int a = 2; a >= 0; a--) {
            double s = rhs[a];
            for (int m = a + 1; m < 3; m++) s -= B[a * W + DP * k + m] * x[m];
            x[a] = s / B[a * W + DP * k + a];
        }
        double dsum = 0;
        for (int a = 0; a < 3; a++) {
            c->dl[3 * j + a] = -x[a];
            dsum += c->Dl2[3 * j + a] * x[a] * x[a];
        }
        q1[j] = s2;
        dd[j] = dsum;
    }
    free(scratch);
    }
    double s1 = 0, s2 = 0;
    for (int64_t j = 0; j < c->n_l; j++) { s1 += q1[j]; s2 += dd[j]; }
    c->q1r2 = s1;
    c->damp_l = c->lambda * s2;
    free(q1); free(dd);
    return 0;
}

/* C10: L(0) - L(dx) with L(dx) = |r + J dx|^2, given the back-substituted dl:
 * sum|Q^_1^T r^|^2 - b~^T dp + rho_cg^T dp + lambda |D_p dp|^2 + lambda sum |D_l dl|^2 */
double orc_model_decrease(orc_ctx *c) {
    int64_t N = DP * c->n_p;
    double m = c->q1r2 + c->damp_l;
    for (int64_t i = 0; i < N; i++)
        m += -c->bt[i] * c->dp[i] + c->rho_cg[i] * c->dp[i] + c->lambda * c->Dp2[i] * c->dp[i] * c->dp[i];
    return m;
}

/* trial state x + S dx (unscaled, additive on all 9 camera parameters and 3 point coords, C1) */
double orc_trial_cost(orc_ctx *c) {
    for (int64_t i = 0; i < DP * c->n_p; i++) c->cams_trial[i] = c->cams[i] + c->sp[i] * c->dp[i];
    for (int64_t i = 0; i < 3 * c->n_l; i++) c->pts_trial[i] = c->pts[i] + c->sl[i] * c->dl[i];
    c->cost_trial = cost_at(c, c->cams_trial, c->pts_trial);
    return c->cost_trial;
}

/* O9: one LM iteration (readings C9, C10, C13). */
int orc_lm_step(orc_ctx *c, double pcg_tol, int pcg_max_iters, orc_lm_report *rep) {
    memset(rep, 0, sizeof(*rep));
    rep->iter = c->iteration;
    if (c->need_linearize) {
        if (orc_linearize(c)) return 1;
        orc_marginalize(c);
        c->need_linearize = 0;
    }
    rep->cost = c->cost;
    rep->lambda = c->lm_lambda;
    orc_damp(c, c->lm_lambda);
    int reason = 0;
    double relres = 0;
    int pre = orc_precond_rhs(c);
    int it = 0;
    if (pre == 0) it = orc_pcg(c, pcg_tol, pcg_max_iters, &reason, &relres);
    else reason = 2;
    rep->pcg_iters = it;
    rep->pcg_reason = reason;
    int accept = 0;
    if (reason != 2) {
        orc_backsub(c);
        double model = orc_model_decrease(c);
        double Et = orc_trial_cost(c);
        double rho = (c->cost - Et) / model;
        rep->model = model;
        rep->cost_trial = Et;
        rep->rho = rho;
        accept = (model > 0) && isfinite(Et) && (rho > 1e-3);
        if (accept) {
            memcpy(c->cams, c->cams_trial, sizeof(double) * DP * c->n_p);
            memcpy(c->pts, c->pts_trial, sizeof(double) * 3 * c->n_l);
            c->cost = Et;
            double t = 2.0 * rho - 1.0;
            double fac = 1.0 - t * t * t;
            c->lm_lambda *= (fac > 1.0 / 3.0 ? fac : 1.0 / 3.0);
            c->lm_nu = 2.0;
            c->need_linearize = 1;
        }
    } else {
        rep->cost_trial = INFINITY;
    }
    if (!accept) {
        c->lm_lambda *= c->lm_nu;
        c->lm_nu *= 2.0;
    }
    c->lm_lambda = clampd(c->lm_lambda, 1e-16, 1e16);
    rep->accepted = accept;
    rep->cost_after = c->cost;
    rep->lambda_next = c->lm_lambda;
    c->iteration++;
    return 0;
}

/* ------------------------------------------------------------------------------------------
 * accessors (caller buffers)
 * ---------------------------------------------------------------------------------------- */
void orc_get_state(orc_ctx *c, double *cams, double *pts) {
    memcpy(cams, c->cams, sizeof(double) * DP * c->n_p);
    memcpy(pts, c->pts, sizeof(double) * 3 * c->n_l);
}
void orc_set_state(orc_ctx *c, const double *cams, const double *pts) {
    memcpy(c->cams, cams, sizeof(double) * DP * c->n_p);
    memcpy(c->pts, pts, sizeof(double) * 3 * c->n_l);
    c->need_linearize = 1;
    c->linearized = c->marginalized = c->damped = 0;
}
void orc_set_lm(orc_ctx *c, double lambda, double nu) { c->lm_lambda = lambda; c->lm_nu = nu; }
/* Huber parameter (pixels); 0 = squared loss.  Takes effect at the next linearization. */
void orc_set_huber(orc_ctx *c, double delta) {
    c->huber = delta;
    c->need_linearize = 1;
}
double orc_get_lambda(orc_ctx *c) { return c->lm_lambda; }
double orc_linearized_cost(orc_ctx *c) { return c->cost; }
void orc_obs_order(orc_ctx *c, int64_t *src, int64_t *lm_ptr) {
    memcpy(src, c->o_src, sizeof(int64_t) * c->n_obs);
    memcpy(lm_ptr, c->lm_ptr, sizeof(int64_t) * (c->n_l + 1));
}
void orc_get_linearization(orc_ctx *c, double *r, double *Jc, double *Jl) {
    memcpy(r, c->r, sizeof(double) * 2 * c->n_obs);
    memcpy(Jc, c->Jc, sizeof(double) * 18 * c->n_obs);
    memcpy(Jl, c->Jl, sizeof(double) * 6 * c->n_obs);
}
void orc_get_scaling(orc_ctx *c, double *sp, double *Dp2, double *sl, double *Dl2) {
    memcpy(sp, c->sp, sizeof(double) * DP * c->n_p);
    memcpy(Dp2, c->Dp2, sizeof(double) * DP * c->n_p);
    memcpy(sl, c->sl, sizeof(double) * 3 * c->n_l);
    memcpy(Dl2, c->Dl2, sizeof(double) * 3 * c->n_l);
}
void orc_get_block(orc_ctx *c, int64_t j, double *buf) {
    if (c->streaming) {  /* recomputed (O3-O5) at the damping in force */
        lm_block(c, j, buf, NULL);
        return;
    }
    memcpy(buf, c->blk + c->blk_off[j], sizeof(double) * (c->blk_off[j + 1] - c->blk_off[j]));
}
void orc_get_givens(orc_ctx *c, int64_t j, double *g) {
    if (c->streaming) {
        double *scratch = lm_scratch(c);
        lm_block(c, j, scratch, g);
        free(scratch);
        return;
    }
    memcpy(g, c->giv + 12 * j, sizeof(double) * 12);
}
void orc_get_rhs(orc_ctx *c, double *b) { memcpy(b, c->bt, sizeof(double) * DP * c->n_p); }
/* Read-only view of the landmark-block arena: *ptr = first double, offsets[j] = start of landmark j
 * (n_l + 1 entries, caller buffer); valid until the next linearization. */
void orc_block_arena(orc_ctx *c, const double **ptr, int64_t *offsets) {
    *ptr = c->blk;
    memcpy(offsets, c->blk_off, sizeof(int64_t) * (c->n_l + 1));
}
/* Cholesky factors L_i (lower, row-major, 81 per camera) of the block-Jacobi blocks of orc_precond_rhs */
void orc_get_precond_factor(orc_ctx *c, double *L) { memcpy(L, c->Lp, sizeof(double) * 81 * c->n_p); }
void orc_get_dp(orc_ctx *c, double *dp) { memcpy(dp, c->dp, sizeof(double) * DP * c->n_p); }
void orc_set_dp(orc_ctx *c, const double *dp) {
    memcpy(c->dp, dp, sizeof(double) * DP * c->n_p);
    memset(c->rho_cg, 0, sizeof(double) * DP * c->n_p);
}
void orc_get_rho_cg(orc_ctx *c, double *r) { memcpy(r, c->rho_cg, sizeof(double) * DP * c->n_p); }
void orc_get_dl(orc_ctx *c, double *dl) { memcpy(dl, c->dl, sizeof(double) * 3 * c->n_l); }
void orc_get_trial(orc_ctx *c, double *cams, double *pts) {
    memcpy(cams, c->cams_trial, sizeof(double) * DP * c->n_p);
    memcpy(pts, c->pts_trial, sizeof(double) * 3 * c->n_l);
}
double orc_get_q1r2(orc_ctx *c) { return c->q1r2; }
double orc_get_damp_l(orc_ctx *c) { return c->damp_l; }
double orc_get_block_lambda(orc_ctx *c) { return c->lambda; }
int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
