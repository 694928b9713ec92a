/*
 * hsgen/gen.c — seeded, counter-based synthetic input generators (host side).
 *
 * TEST/BENCH INFRASTRUCTURE.  This module produces the *inputs* of the
 * Hierarchy-Scan (skeleton parent arrays, local poses, inverse bind poses).
 * It holds none of the method's arithmetic (no composition, no scan, no bind):
 * both the fp64 oracle (oracle/) and the CUDA path (paper_2505_06703_b200/)
 * consume what it produces, and neither shares code with the other.
 *
 * Recipe (SURVEY.md §8(d) "Synthetic inputs", restated in DESIGN.md §4):
 *   sm64(x)  = splitmix64 finaliser of x + 0x9E3779B97F4A7C15
 *   u(seed, stream, c, J, j, k) =
 *       (sm64(((c*J + j)*8 + k) ^ sm64(seed*16 + stream)) >> 11) * 2^-53
 *   stream   = 8*type + purpose
 *       purpose 0 local rotation, 1 local translation, 2 inv_bind,
 *               3 skeleton generator, 4 exact family (locals),
 *               5 label permutation, 6 exact family (inv_bind)
 *   rotation    : Shoemake quaternion from k = 0,1,2 (Haar-uniform), fp64
 *   translation : z = 2u0-1, phi = 2*pi*u1, r = u2^(1/3),
 *                 t = r*(sqrt(1-z^2)cos phi, sqrt(1-z^2) sin phi, z), fp64
 *   every transform is computed in fp64 and rounded once to fp32 (RN).
 *   Layout: [n_chars][J][3][4] fp32 row-major, element (r,c) at 4r+c,
 *   column 3 = translation, implicit bottom row (0,0,0,1).
 *
 * The device twin (hsgen/gen_cuda.cu) implements the same recipe for the
 * bench's full-size (21.5 GB) inputs; see DESIGN.md §4 for its ulp caveat.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define HSG_PI 3.14159265358979323846

uint64_t hsg_sm64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t hsg_raw(uint64_t seed, uint64_t stream, uint64_t c, uint64_t J,
                 uint64_t j, uint64_t k) {
    return hsg_sm64(((c * J + j) * 8 + k) ^ hsg_sm64(seed * 16 + stream));
}

double hsg_u(uint64_t seed, uint64_t stream, uint64_t c, uint64_t J,
             uint64_t j, uint64_t k) {
    return (double)(hsg_raw(seed, stream, c, J, j, k) >> 11) * 0x1.0p-53;
}

/* Shoemake: unit quaternion (x,y,z,w) from three uniforms -> 3x3 in fp64. */
static void rot_from_u(double u0, double u1, double u2, double R[9]) {
    double s1 = sqrt(1.0 - u0), s2 = sqrt(u0);
    double a1 = 2.0 * HSG_PI * u1, a2 = 2.0 * HSG_PI * u2;
    double x = s1 * sin(a1), y = s1 * cos(a1), z = s2 * sin(a2), w = s2 * cos(a2);
    R[0] = 1.0 - 2.0 * (y * y + z * z); R[1] = 2.0 * (x * y - w * z); R[2] = 2.0 * (x * z + w * y);
    R[3] = 2.0 * (x * y + w * z); R[4] = 1.0 - 2.0 * (x * x + z * z); R[5] = 2.0 * (y * z - w * x);
    R[6] = 2.0 * (x * z - w * y); R[7] = 2.0 * (y * z + w * x); R[8] = 1.0 - 2.0 * (x * x + y * y);
}

static void ball_from_u(double u0, double u1, double u2, double t[3]) {
    double z = 2.0 * u0 - 1.0, phi = 2.0 * HSG_PI * u1, r = cbrt(u2);
    double rho = sqrt(fmax(0.0, 1.0 - z * z));
    t[0] = r * rho * cos(phi); t[1] = r * rho * sin(phi); t[2] = r * z;
}

static void pack(const double R[9], const double t[3], float out[12]) {
    for (int r = 0; r < 3; ++r) {
        out[4 * r + 0] = (float)R[3 * r + 0];
        out[4 * r + 1] = (float)R[3 * r + 1];
        out[4 * r + 2] = (float)R[3 * r + 2];
        out[4 * r + 3] = (float)t[r];
    }
}

/* One rigid local pose: rotation on stream 8*type+0, translation on 8*type+1. */
void hsg_local_one(uint64_t seed, uint64_t type, uint64_t J, uint64_t c, uint64_t j,
                   float out[12]) {
    double R[9], t[3];
    uint64_t sr = 8 * type + 0, st = 8 * type + 1;
    rot_from_u(hsg_u(seed, sr, c, J, j, 0), hsg_u(seed, sr, c, J, j, 1),
               hsg_u(seed, sr, c, J, j, 2), R);
    ball_from_u(hsg_u(seed, st, c, J, j, 0), hsg_u(seed, st, c, J, j, 1),
                hsg_u(seed, st, c, J, j, 2), t);
    pack(R, t, out);
}

/* The 24 proper (det=+1) signed permutation matrices, lexicographic in
 * (permutation, sign bits).  Built once. */
static float g_sp24[24][9];
static int g_sp24_ready = 0;
static pthread_mutex_t g_sp24_mu = PTHREAD_MUTEX_INITIALIZER;

static void build_sp24(void) {
    pthread_mutex_lock(&g_sp24_mu);
    if (!g_sp24_ready) {
        static const int perms[6][3] = {{0,1,2},{0,2,1},{1,0,2},{1,2,0},{2,0,1},{2,1,0}};
        static const int psign[6] = {+1, -1, -1, +1, +1, -1};  /* parity of each permutation */
        int n = 0;
        for (int p = 0; p < 6; ++p)
            for (int b = 0; b < 8; ++b) {
                int sprod = 1;
                for (int r = 0; r < 3; ++r) sprod *= ((b >> r) & 1) ? -1 : 1;
                if (sprod * psign[p] != 1) continue;
                float* M = g_sp24[n++];
                memset(M, 0, 9 * sizeof(float));
                for (int r = 0; r < 3; ++r) M[3 * r + perms[p][r]] = ((b >> r) & 1) ? -1.0f : 1.0f;
            }
        g_sp24_ready = 1;
    }
    pthread_mutex_unlock(&g_sp24_mu);
}

void hsg_signed_perm(int idx, float out9[9]) {
    build_sp24();
    memcpy(out9, g_sp24[idx % 24], 9 * sizeof(float));
}

/* Exact-arithmetic family: rotation = SP24[u64 % 24], t_c = ((u64 >> (8+2c)) % 3) - 1. */
void hsg_exact_one(uint64_t seed, uint64_t stream, uint64_t J, uint64_t c, uint64_t j,
                   float out[12]) {
    build_sp24();
    uint64_t r = hsg_raw(seed, stream, c, J, j, 0);
    const float* M = g_sp24[r % 24];
    for (int row = 0; row < 3; ++row) {
        out[4 * row + 0] = M[3 * row + 0];
        out[4 * row + 1] = M[3 * row + 1];
        out[4 * row + 2] = M[3 * row + 2];
        out[4 * row + 3] = (float)((int)((r >> (8 + 2 * row)) % 3) - 1);
    }
}

/* ---- batched, multithreaded fills ---------------------------------------- */
typedef struct {
    int kind;  /* 0 local rigid, 1 exact */
    uint64_t seed, type, J, char0, c_lo, c_hi;
    float* out;
} fill_job;

static void* fill_worker(void* arg) {
    fill_job* f = (fill_job*)arg;
    for (uint64_t c = f->c_lo; c < f->c_hi; ++c)
        for (uint64_t j = 0; j < f->J; ++j) {
            float* o = f->out + ((c - f->char0) * f->J + j) * 12;
            if (f->kind == 0) hsg_local_one(f->seed, f->type, f->J, c, j, o);
            else hsg_exact_one(f->seed, 8 * f->type + 4, f->J, c, j, o);
        }
    return NULL;
}

static void fill(int kind, uint64_t seed, uint64_t type, uint64_t J, uint64_t char0,
                 uint64_t n_chars, float* out, int nthreads) {
    if (kind == 1) build_sp24();
    if (nthreads < 1) nthreads = 1;
    if ((uint64_t)nthreads > n_chars) nthreads = n_chars ? (int)n_chars : 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nthreads);
    fill_job* jobs = (fill_job*)malloc(sizeof(fill_job) * nthreads);
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].kind = kind; jobs[t].seed = seed; jobs[t].type = type; jobs[t].J = J;
        jobs[t].char0 = char0; jobs[t].out = out;
        jobs[t].c_lo = char0 + n_chars * t / nthreads;
        jobs[t].c_hi = char0 + n_chars * (t + 1) / nthreads;
        pthread_create(&th[t], NULL, fill_worker, &jobs[t]);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(th); free(jobs);
}

/* Local poses of characters [char0, char0+n_chars) of a crowd of skeleton type
 * `type` with J joints.  `out` is [n_chars][J][12]. */
void hsg_local_poses(uint64_t seed, uint64_t type, uint64_t J, uint64_t char0,
                     uint64_t n_chars, float* out, int nthreads) {
    fill(0, seed, type, J, char0, n_chars, out, nthreads);
}

void hsg_exact_poses(uint64_t seed, uint64_t type, uint64_t J, uint64_t char0,
                     uint64_t n_chars, float* out, int nthreads) {
    fill(1, seed, type, J, char0, n_chars, out, nthreads);
}

/* Per-skeleton inverse bind: rigid, |t| <= 1, stream 8*type+2,
 * rotation draws k = 0..2, translation draws k = 3..5, character index 0. */
void hsg_inv_bind(uint64_t seed, uint64_t type, uint64_t J, float* out) {
    uint64_t s = 8 * type + 2;
    for (uint64_t j = 0; j < J; ++j) {
        double R[9], t[3];
        rot_from_u(hsg_u(seed, s, 0, J, j, 0), hsg_u(seed, s, 0, J, j, 1), hsg_u(seed, s, 0, J, j, 2), R);
        ball_from_u(hsg_u(seed, s, 0, J, j, 3), hsg_u(seed, s, 0, J, j, 4), hsg_u(seed, s, 0, J, j, 5), t);
        pack(R, t, out + 12 * j);
    }
}

/* Exact-family inverse bind: stream 8*type+6, character index 0. */
void hsg_exact_inv_bind(uint64_t seed, uint64_t type, uint64_t J, float* out) {
    for (uint64_t j = 0; j < J; ++j) hsg_exact_one(seed, 8 * type + 6, J, 0, j, out + 12 * j);
}

/* SPEC random_tree (SURVEY §8(d) tree1024): joints 0..depth-1 form a
 * path; for k = depth..J-1, cand = existing joints with level < depth in index
 * order, parents[k] = cand[floor(u(seed, 8*type+3, 0, J, k, 0) * |cand|)].
 * Levels count nodes (root level 1), so max level == depth exactly.
 * Returns 0 on success, -1 on bad arguments. */
int hsg_random_tree(uint64_t seed, uint64_t type, int32_t J, int32_t depth, int32_t* parents) {
    if (J < 1 || depth < 1 || depth > J) return -1;
    int32_t* level = (int32_t*)malloc(sizeof(int32_t) * J);
    int32_t* cand = (int32_t*)malloc(sizeof(int32_t) * J);
    int32_t ncand = 0;
    for (int32_t i = 0; i < depth; ++i) {
        parents[i] = i - 1;
        level[i] = i + 1;
        if (level[i] < depth) cand[ncand++] = i;
    }
    for (int32_t k = depth; k < J; ++k) {
        double u = hsg_u(seed, 8 * type + 3, 0, (uint64_t)J, (uint64_t)k, 0);
        int32_t pick = (int32_t)floor(u * (double)ncand);
        if (pick >= ncand) pick = ncand - 1;
        int32_t p = cand[pick];
        parents[k] = p;
        level[k] = level[p] + 1;
        if (level[k] < depth) cand[ncand++] = k;  /* appended in index order */
    }
    free(level); free(cand);
    return 0;
}

/* Label permutation of n joints (Fisher-Yates, stream 8*type+5): perm[new] = old. */
void hsg_permutation(uint64_t seed, uint64_t type, int32_t n, int32_t* perm) {
    for (int32_t i = 0; i < n; ++i) perm[i] = i;
    for (int32_t i = n - 1; i > 0; --i) {
        double u = hsg_u(seed, 8 * type + 5, 0, (uint64_t)n, (uint64_t)i, 0);
        int32_t j = (int32_t)floor(u * (double)(i + 1));
        if (j > i) j = i;
        int32_t tmp = perm[i]; perm[i] = perm[j]; perm[j] = tmp;
    }
}

/* ---- Stage-1 inputs (NEXT-1): animation clips and per-character layer states ----
 * Clip keys: fp32 [n_clips][n_keys][J][10] = t(3), q = (w,x,y,z), s(3); stream
 * 8*type + 7, counter character = clip*n_keys + key; rotation draws k = 0..2
 * (Shoemake), translation k = 3..5 (unit ball), scale k = 6: s = lo + (hi-lo)*u
 * for all three axes (lo = hi = 1 gives rigid keys). */
void hsg_clips(uint64_t seed, uint64_t type, uint64_t n_clips, uint64_t n_keys, uint64_t J,
               float scale_lo, float scale_hi, float* keys) {
    const uint64_t s = 8 * type + 7;
    for (uint64_t c = 0; c < n_clips; ++c)
        for (uint64_t k = 0; k < n_keys; ++k)
            for (uint64_t j = 0; j < J; ++j) {
                const uint64_t ch = c * n_keys + k;
                double R[9], t[3];
                (void)R;
                double u0 = hsg_u(seed, s, ch, J, j, 0), u1 = hsg_u(seed, s, ch, J, j, 1),
                       u2 = hsg_u(seed, s, ch, J, j, 2);
                double s1 = sqrt(1.0 - u0), s2 = sqrt(u0);
                double a1 = 2.0 * HSG_PI * u1, a2 = 2.0 * HSG_PI * u2;
                double x = s1 * sin(a1), y = s1 * cos(a1), z = s2 * sin(a2), w = s2 * cos(a2);
                ball_from_u(hsg_u(seed, s, ch, J, j, 3), hsg_u(seed, s, ch, J, j, 4),
                            hsg_u(seed, s, ch, J, j, 5), t);
                const double sc = (double)scale_lo + ((double)scale_hi - (double)scale_lo) *
                                                         hsg_u(seed, s, ch, J, j, 6);
                float* o = keys + ((c * n_keys + k) * J + j) * 10;
                o[0] = (float)t[0]; o[1] = (float)t[1]; o[2] = (float)t[2];
                o[3] = (float)w; o[4] = (float)x; o[5] = (float)y; o[6] = (float)z;
                o[7] = o[8] = o[9] = (float)sc;
            }
}

/* Layer states of characters [char0, char0 + n_chars): int32 clip, f32 time, f32 weight,
 * int32 pad per layer; stream 8*(type + 32) + 7, counter (character, layer): clip =
 * floor(u0 * n_clips), time = u1 * time_span, weight = 0.05 + 0.95 * u2. */
void hsg_layers(uint64_t seed, uint64_t type, uint64_t char0, uint64_t n_chars, uint64_t n_layers,
                uint64_t n_clips, float time_span, void* out) {
    const uint64_t s = 8 * (type + 32) + 7;
    unsigned char* base = (unsigned char*)out;
    for (uint64_t c = 0; c < n_chars; ++c)
        for (uint64_t l = 0; l < n_layers; ++l) {
            const uint64_t ch = char0 + c;
            int32_t clip = (int32_t)floor(hsg_u(seed, s, ch, n_layers, l, 0) * (double)n_clips);
            if (clip >= (int32_t)n_clips) clip = (int32_t)n_clips - 1;
            const float tm = (float)(hsg_u(seed, s, ch, n_layers, l, 1) * (double)time_span);
            const float wt = (float)(0.05 + 0.95 * hsg_u(seed, s, ch, n_layers, l, 2));
            unsigned char* p = base + (c * n_layers + l) * 16;
            const int32_t pad = 0;
            memcpy(p, &clip, 4); memcpy(p + 4, &tm, 4); memcpy(p + 8, &wt, 4); memcpy(p + 12, &pad, 4);
        }
}

/* Synthetic skinned mesh for a skeleton (NEXT-4; "Mesh Face Number
 * 1000-3000"): V vertices, stream 8*(type + 64) + 7, counter (0, V, vertex, k).
 * Rest position uniform in [-1, 1]^3.  Influences: a home joint floor(u0 J), its
 * parent and grandparent (the joint itself at a root), and a uniform random joint;
 * weights u + 0.05 normalised in fp64 and rounded to fp32; with probability 0.3 the
 * fourth weight is 0 (fewer than four influences). */
void hsg_mesh(uint64_t seed, uint64_t type, const int32_t* parents, int32_t J, int32_t V,
              float* pos, int32_t* joints, float* weights) {
    const uint64_t s = 8 * (type + 64) + 7;
    for (int32_t v = 0; v < V; ++v) {
#define U(k) hsg_u(seed, s, 0, (uint64_t)V, (uint64_t)v, (k))
        for (int e = 0; e < 3; ++e) pos[3 * v + e] = (float)(2.0 * U(e) - 1.0);
        int32_t j0 = (int32_t)floor(U(3) * (double)J);
        if (j0 >= J) j0 = J - 1;
        const int32_t j1 = parents[j0] >= 0 ? parents[j0] : j0;
        const int32_t j2 = parents[j1] >= 0 ? parents[j1] : j1;
        int32_t j3 = (int32_t)floor(U(4) * (double)J);
        if (j3 >= J) j3 = J - 1;
        double w[4], sum = 0.0;
        for (int k = 0; k < 4; ++k) w[k] = U(5 + k) + 0.05;
        if (U(9) < 0.3) w[3] = 0.0;
        for (int k = 0; k < 4; ++k) sum += w[k];
        joints[4 * v + 0] = j0; joints[4 * v + 1] = j1; joints[4 * v + 2] = j2; joints[4 * v + 3] = j3;
        for (int k = 0; k < 4; ++k) weights[4 * v + k] = (float)(w[k] / sum);
#undef U
    }
}
