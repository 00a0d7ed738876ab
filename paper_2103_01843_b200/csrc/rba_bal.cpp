// rba_bal.cpp -- BAL problem ingest and the paper's deterministic preprocessing (host code of
// librba; NEXT row f1 of SURVEY §8f).  PAPER.md P:457-471 (Sec. "Datasets"):
//   * BAL problems (Agarwal et al.): text "n_cams n_points n_obs", n_obs lines "cam pt u v",
//     9 numbers per camera (angle-axis, translation, f, k1, k2), 3 per point (S:34 describes the
//     layout);
//   * "we center the point cloud of landmarks at the coordinate system origin and rescale to median
//     absolute deviation of 100" -- reading C25: per-axis median, MAD = median over the
//     points of the L1 distance to that median (Ceres' BAL example, which P:471 says the
//     preprocessing follows); cameras are moved with the cloud so every residual is unchanged;
//   * "Initial landmark and camera positions are then perturbed with small Gaussian noise",
//     seeded and in double precision -- angle-axis, camera centre and point coordinates
//     each get iid N(0, sigma^2) noise from a counter-based generator;
//   * "we remove all observations with a small or negative z value in the camera frame, completely
//     removing landmarks with less than two remaining observations" -- with the BAL
//     convention (camera looks down -z) the depth is -P_z; an observation is kept iff -P_z > z_min.
#include <cmath>
#include <cstdint>
#include <zlib.h>

#include <charconv>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <algorithm>

#include "../../include/rba.h"

namespace {
thread_local std::string g_bal_err;

rba_status bal_fail(rba_status s, const std::string &m) {
    g_bal_err = m;
    return s;
}

// rotation matrix of an angle-axis vector (Rodrigues), R row-major
void rotation(const double *w, double *R) {
    const double th2 = w[0] * w[0] + w[1] * w[1] + w[2] * w[2];
    double a, b;
    if (th2 < 1e-16) {
        a = 1.0 - th2 / 6.0;
        b = 0.5 - th2 / 24.0;
    } else {
        const double th = std::sqrt(th2);
        a = std::sin(th) / th;
        b = (1.0 - std::cos(th)) / th2;
    }
    const double K[9] = {0, -w[2], w[1], w[2], 0, -w[0], -w[1], w[0], 0};
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
            double k2 = 0;
            for (int m = 0; m < 3; m++) k2 += K[3 * i + m] * K[3 * m + j];
            R[3 * i + j] = (i == j ? 1.0 : 0.0) + a * K[3 * i + j] + b * k2;
        }
}

// camera centre C = -R^T t and back: t = -R C
void centre_of(const double *cam, double *C) {
    double R[9];
    rotation(cam, R);
    for (int j = 0; j < 3; j++) C[j] = -(R[j] * cam[3] + R[3 + j] * cam[4] + R[6 + j] * cam[5]);
}
void set_centre(double *cam, const double *C) {
    double R[9];
    rotation(cam, R);
    for (int i = 0; i < 3; i++) cam[3 + i] = -(R[3 * i] * C[0] + R[3 * i + 1] * C[1] + R[3 * i + 2] * C[2]);
}

double median_of(std::vector<double> v) {
    if (v.empty()) return 0.0;
    const size_t m = v.size() / 2;
    std::nth_element(v.begin(), v.begin() + m, v.end());
    double hi = v[m];
    if (v.size() % 2) return hi;
    const double lo = *std::max_element(v.begin(), v.begin() + m);
    return 0.5 * (lo + hi);
}

// counter-based N(0,1): splitmix64 of (seed, counter) -> two uniforms -> Box-Muller
uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
double gauss(uint64_t seed, uint64_t ctr) {
    const uint64_t a = splitmix64(seed ^ splitmix64(2 * ctr)), b = splitmix64(seed ^ splitmix64(2 * ctr + 1));
    const double u1 = ((a >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    const double u2 = (b >> 11) * (1.0 / 9007199254740992.0);
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
}

struct Lexer {
    const char *p, *end;
    int64_t line = 1;
    bool next_num(double *v) {
        while (p < end && (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\n')) {
            if (*p == '\n') line++;
            p++;
        }
        if (p >= end) return false;
        // bounded by `end` (the buffer need not be NUL-terminated); from_chars does not take a
        // leading '+', which BAL writers do not emit
        const std::from_chars_result res = std::from_chars(p, end, *v);
        if (res.ec != std::errc() || res.ptr == p) return false;
        p = res.ptr;
        return true;
    }
    bool next_int(int64_t *v) {
        double d;
        if (!next_num(&d) || d != std::floor(d)) return false;
        *v = (int64_t)d;
        return true;
    }
};
}  // namespace

extern "C" const char *rba_bal_last_error(void) { return g_bal_err.c_str(); }

extern "C" void rba_bal_free(rba_bal *b) {
    if (!b) return;
    std::free(b->cameras);
    std::free(b->points);
    std::free(b->obs_cam);
    std::free(b->obs_pt);
    std::free(b->obs_uv);
    std::memset(b, 0, sizeof(*b));
}

extern "C" rba_status rba_bal_parse(const char *text, size_t len, rba_bal *out) {
    if (!text || !out) return bal_fail(RBA_ERR_INVALID_ARG, "null argument");
    std::memset(out, 0, sizeof(*out));
    Lexer L{text, text + len};
    int64_t np, nl, no;
    if (!L.next_int(&np) || !L.next_int(&nl) || !L.next_int(&no) || np < 1 || nl < 0 || no < 0)
        return bal_fail(RBA_ERR_BAD_PROBLEM, "line 1: malformed header (expected \"n_cameras n_points n_observations\")");
    if (np >= (1ll << 28) || nl >= (1ll << 31) || no >= (1ll << 31))
        return bal_fail(RBA_ERR_BAD_PROBLEM, "line 1: problem too large for int32 indices");
    out->n_cams = np, out->n_points = nl, out->n_obs = no;
    out->cameras = (double *)std::malloc(sizeof(double) * 9 * np);
    out->points = (double *)std::malloc(sizeof(double) * 3 * std::max<int64_t>(nl, 1));
    out->obs_cam = (int32_t *)std::malloc(sizeof(int32_t) * std::max<int64_t>(no, 1));
    out->obs_pt = (int32_t *)std::malloc(sizeof(int32_t) * std::max<int64_t>(no, 1));
    out->obs_uv = (double *)std::malloc(sizeof(double) * 2 * std::max<int64_t>(no, 1));
    if (!out->cameras || !out->points || !out->obs_cam || !out->obs_pt || !out->obs_uv) {
        rba_bal_free(out);
        return bal_fail(RBA_ERR_OOM, "host allocation failed");
    }
    for (int64_t i = 0; i < no; i++) {
        int64_t c, j;
        double u, v;
        if (!L.next_int(&c) || !L.next_int(&j) || !L.next_num(&u) || !L.next_num(&v)) {
            const int64_t line = L.line;
            rba_bal_free(out);
            return bal_fail(RBA_ERR_BAD_PROBLEM, "line " + std::to_string(line) + ": truncated or malformed observation " +
                                                     std::to_string(i));
        }
        if (c < 0 || c >= np || j < 0 || j >= nl) {
            const int64_t line = L.line;
            rba_bal_free(out);
            return bal_fail(RBA_ERR_BAD_PROBLEM, "line " + std::to_string(line) + ": observation " + std::to_string(i) +
                                                     " index out of range");
        }
        out->obs_cam[i] = (int32_t)c, out->obs_pt[i] = (int32_t)j;
        out->obs_uv[2 * i] = u, out->obs_uv[2 * i + 1] = v;
    }
    for (int64_t i = 0; i < 9 * np; i++)
        if (!L.next_num(out->cameras + i)) {
            const int64_t line = L.line;
            rba_bal_free(out);
            return bal_fail(RBA_ERR_BAD_PROBLEM, "line " + std::to_string(line) + ": truncated camera block");
        }
    for (int64_t i = 0; i < 3 * nl; i++)
        if (!L.next_num(out->points + i)) {
            const int64_t line = L.line;
            rba_bal_free(out);
            return bal_fail(RBA_ERR_BAD_PROBLEM, "line " + std::to_string(line) + ": truncated point block");
        }
    return RBA_OK;
}

extern "C" rba_status rba_bal_read(const char *path, rba_bal *out) {
    if (!path || !out) return bal_fail(RBA_ERR_INVALID_ARG, "null argument");
    // plain text or gzip (the BAL distribution's .bz2 / .gz files are usually stored gunzipped or
    // gzipped; zlib's gzread reads both plain and gzip-compressed input transparently)
    gzFile f = gzopen(path, "rb");
    if (!f) return bal_fail(RBA_ERR_INVALID_ARG, std::string("cannot open ") + path);
    std::string buf;
    char tmp[1 << 16];
    int n;
    while ((n = gzread(f, tmp, sizeof(tmp))) > 0) buf.append(tmp, (size_t)n);
    const bool err = n < 0;
    gzclose(f);
    if (err) return bal_fail(RBA_ERR_INVALID_ARG, std::string("cannot decompress ") + path);
    return rba_bal_parse(buf.data(), buf.size(), out);
}

extern "C" rba_status rba_bal_write(const char *path, const rba_bal *b) {
    if (!path || !b) return bal_fail(RBA_ERR_INVALID_ARG, "null argument");
    FILE *f = std::fopen(path, "w");
    if (!f) return bal_fail(RBA_ERR_INVALID_ARG, std::string("cannot open ") + path);
    std::fprintf(f, "%lld %lld %lld\n", (long long)b->n_cams, (long long)b->n_points, (long long)b->n_obs);
    for (int64_t i = 0; i < b->n_obs; i++)
        std::fprintf(f, "%d %d %.17g %.17g\n", b->obs_cam[i], b->obs_pt[i], b->obs_uv[2 * i], b->obs_uv[2 * i + 1]);
    for (int64_t i = 0; i < 9 * b->n_cams; i++) std::fprintf(f, "%.17g\n", b->cameras[i]);
    for (int64_t i = 0; i < 3 * b->n_points; i++) std::fprintf(f, "%.17g\n", b->points[i]);
    std::fclose(f);
    return RBA_OK;
}

extern "C" rba_status rba_bal_normalize(rba_bal *b, double target_mad) {
    if (!b || !(target_mad > 0)) return bal_fail(RBA_ERR_INVALID_ARG, "null problem or target_mad <= 0");
    if (b->n_points < 1) return bal_fail(RBA_ERR_BAD_PROBLEM, "no landmarks to normalize");
    const int64_t nl = b->n_points;
    double med[3];
    std::vector<double> v(nl);
    for (int a = 0; a < 3; a++) {
        for (int64_t j = 0; j < nl; j++) v[j] = b->points[3 * j + a];
        med[a] = median_of(v);
    }
    for (int64_t j = 0; j < nl; j++)
        v[j] = std::fabs(b->points[3 * j] - med[0]) + std::fabs(b->points[3 * j + 1] - med[1]) +
               std::fabs(b->points[3 * j + 2] - med[2]);
    const double mad = median_of(v);
    if (!(mad > 0)) return bal_fail(RBA_ERR_BAD_PROBLEM, "degenerate point cloud (median absolute deviation 0)");
    const double s = target_mad / mad;
    for (int64_t j = 0; j < nl; j++)
        for (int a = 0; a < 3; a++) b->points[3 * j + a] = s * (b->points[3 * j + a] - med[a]);
    for (int64_t i = 0; i < b->n_cams; i++) {
        double *cam = b->cameras + 9 * i, C[3];
        centre_of(cam, C);
        for (int a = 0; a < 3; a++) C[a] = s * (C[a] - med[a]);
        set_centre(cam, C);
    }
    return RBA_OK;
}

extern "C" rba_status rba_bal_perturb(rba_bal *b, double sigma_rot, double sigma_centre, double sigma_point,
                                      uint64_t seed) {
    if (!b || !(sigma_rot >= 0) || !(sigma_centre >= 0) || !(sigma_point >= 0))
        return bal_fail(RBA_ERR_INVALID_ARG, "null problem or negative sigma");
    uint64_t ctr = 0;
    for (int64_t j = 0; j < b->n_points; j++)
        for (int a = 0; a < 3; a++) b->points[3 * j + a] += sigma_point * gauss(seed, ctr++);
    if (sigma_rot == 0.0 && sigma_centre == 0.0) return RBA_OK;  // cameras bit-identical
    for (int64_t i = 0; i < b->n_cams; i++) {
        double *cam = b->cameras + 9 * i, C[3];
        centre_of(cam, C);
        for (int a = 0; a < 3; a++) cam[a] += sigma_rot * gauss(seed, ctr++);
        for (int a = 0; a < 3; a++) C[a] += sigma_centre * gauss(seed, ctr++);
        set_centre(cam, C);
    }
    return RBA_OK;
}

extern "C" rba_status rba_bal_filter(rba_bal *b, double z_min, int64_t *removed_obs, int64_t *removed_points) {
    if (!b) return bal_fail(RBA_ERR_INVALID_ARG, "null problem");
    std::vector<char> keep(b->n_obs, 0);
    std::vector<int64_t> cnt(b->n_points, 0);
    for (int64_t i = 0; i < b->n_obs; i++) {
        const double *cam = b->cameras + 9 * (int64_t)b->obs_cam[i], *X = b->points + 3 * (int64_t)b->obs_pt[i];
        double R[9];
        rotation(cam, R);
        const double Pz = R[6] * X[0] + R[7] * X[1] + R[8] * X[2] + cam[5];
        if (-Pz > z_min) keep[i] = 1, cnt[b->obs_pt[i]]++;
    }
    std::vector<int32_t> remap(b->n_points, -1);
    int64_t nl = 0;
    for (int64_t j = 0; j < b->n_points; j++)
        if (cnt[j] >= 2) {
            remap[j] = (int32_t)nl;
            for (int a = 0; a < 3; a++) b->points[3 * nl + a] = b->points[3 * j + a];
            nl++;
        }
    int64_t no = 0;
    for (int64_t i = 0; i < b->n_obs; i++) {
        if (!keep[i] || remap[b->obs_pt[i]] < 0) continue;
        b->obs_cam[no] = b->obs_cam[i];
        b->obs_pt[no] = remap[b->obs_pt[i]];
        b->obs_uv[2 * no] = b->obs_uv[2 * i];
        b->obs_uv[2 * no + 1] = b->obs_uv[2 * i + 1];
        no++;
    }
    if (removed_obs) *removed_obs = b->n_obs - no;
    if (removed_points) *removed_points = b->n_points - nl;
    b->n_obs = no;
    b->n_points = nl;
    if (no == 0) return bal_fail(RBA_ERR_BAD_PROBLEM, "no observations left after filtering");
    return RBA_OK;
}
