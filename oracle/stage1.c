/*
 * oracle/stage1.c — fp64 oracle for Stage 1 (Simulation) fused ahead of the
 * Hierarchy-Scan: keyframe sampling, layer blending, TRS -> 3x4 (SURVEY.md §8(f)
 * NEXT-1).  TEST INFRASTRUCTURE ONLY, like oracle.c (same library, same rules).
 *
 * Passages: PAPER.md:56-57 (§1 step 1: "Sample animation data and generate local
 * pose in local space"), PAPER.md:64 and :91 ("interpolating and blending
 * animation data").  The paper gives no formulas; the operations are SPEC.md's
 * `trs_to_matrix`, `sample_clip`, `blend` with the readings of
 * DESIGN.md §2 R19-R23:
 *   key layout   fp32 keys[clip][key][joint][10] = t(3), q = (w,x,y,z), s(3);
 *                keys uniformly spaced, key k at time k / fps; duration =
 *                (n_keys - 1) / fps                                        (R19)
 *   time         wrap, u = t * fps, k0 = floor(u), a = u - k0 computed in fp32 on
 *                both sides (a float decides an integer: same precision)   (R20)
 *   sample       a == 0 -> key k0 exactly; else lerp t and s, nlerp q with the
 *                shortest-arc sign fix                       (R21)
 *   blend        one layer -> that pose exactly; else weights normalised, t and s
 *                weighted means, quaternions sign-aligned to layer 0, summed,
 *                normalised                                   (R22)
 *   TRS          M = [R(q) diag(s) | t] (T * R * S)            (R23)
 * Then the same recurrence as oracle.c: G[j] = G[parent] (x) L[j], S = G (x) IB.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

int orc_kahn_order(const int32_t* parents, int32_t n, int32_t* order);
void orc_compose(const double* A, const double* B, double* C);

typedef struct {
    int32_t clip;
    float time;
    float weight;
    int32_t pad;
} orc_layer;   /* matches hs_layer (16 bytes) */

/* fp32 time -> (k0, a): wrap 0 = clamp, 1 = loop.  Plain fp32 ops, no contraction. */
void orc_key_index(float t, int32_t n_keys, float fps, int32_t wrap, int32_t* k0, float* a) {
    if (n_keys <= 1) { *k0 = 0; *a = 0.0f; return; }
    const float duration = (float)(n_keys - 1) / fps;
    float tt;
    if (wrap == 1) {
        const float q = floorf(t / duration);
        const float back = q * duration;
        tt = t - back;
        if (tt < 0.0f) tt = 0.0f;
    } else {
        tt = t < 0.0f ? 0.0f : (t > duration ? duration : t);
    }
    const float u = tt * fps;
    float k = floorf(u);
    float frac = u - k;
    int32_t ki = (int32_t)k;
    if (ki >= n_keys - 1) { ki = n_keys - 1; frac = 0.0f; }
    if (ki < 0) { ki = 0; frac = 0.0f; }
    *k0 = ki;
    *a = frac;
}

/* Sample joint j of one clip (keys of that clip: [n_keys][n_joints][10]). */
void orc_sample(const float* clip_keys, int32_t n_keys, int32_t n_joints, float fps, int32_t wrap,
                float t, int32_t j, double out[10]) {
    int32_t k0;
    float af;
    orc_key_index(t, n_keys, fps, wrap, &k0, &af);
    const float* p0 = clip_keys + ((size_t)k0 * n_joints + j) * 10;
    if (af == 0.0f) {
        for (int e = 0; e < 10; ++e) out[e] = (double)p0[e];
        return;
    }
    const float* p1 = clip_keys + ((size_t)(k0 + 1) * n_joints + j) * 10;
    const double a = (double)af, b = 1.0 - a;
    for (int e = 0; e < 3; ++e) out[e] = b * (double)p0[e] + a * (double)p1[e];
    for (int e = 7; e < 10; ++e) out[e] = b * (double)p0[e] + a * (double)p1[e];
    double d = 0.0;
    for (int e = 3; e < 7; ++e) d += (double)p0[e] * (double)p1[e];
    const double sg = d < 0.0 ? -1.0 : 1.0;
    double n2 = 0.0;
    for (int e = 3; e < 7; ++e) {
        out[e] = b * (double)p0[e] + a * sg * (double)p1[e];
        n2 += out[e] * out[e];
    }
    const double inv = 1.0 / sqrt(n2);
    for (int e = 3; e < 7; ++e) out[e] *= inv;
}

/* Blend n sampled poses with weights (sum > 0). */
void orc_blend(int32_t n, const double* poses, const double* weights, double out[10]) {
    if (n == 1) { memcpy(out, poses, 10 * sizeof(double)); return; }
    double W = 0.0;
    for (int i = 0; i < n; ++i) W += weights[i];
    for (int e = 0; e < 10; ++e) out[e] = 0.0;
    for (int i = 0; i < n; ++i) {
        const double w = weights[i] / W;
        const double* p = poses + (size_t)i * 10;
        double d = 0.0;
        for (int e = 3; e < 7; ++e) d += p[e] * poses[e];
        const double sg = d < 0.0 ? -1.0 : 1.0;
        for (int e = 0; e < 3; ++e) out[e] += w * p[e];
        for (int e = 3; e < 7; ++e) out[e] += w * sg * p[e];
        for (int e = 7; e < 10; ++e) out[e] += w * p[e];
    }
    double n2 = 0.0;
    for (int e = 3; e < 7; ++e) n2 += out[e] * out[e];
    const double inv = 1.0 / sqrt(n2);
    for (int e = 3; e < 7; ++e) out[e] *= inv;
}

/* T * R(q) * S as a 3x4 [R diag(s) | t]; q = (w, x, y, z) unit. */
void orc_trs_to_matrix(const double trs[10], double m[12]) {
    const double w = trs[3], x = trs[4], y = trs[5], z = trs[6];
    const double R[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                         2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                         2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
    for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c) m[4 * r + c] = R[3 * r + c] * trs[7 + c];
        m[4 * r + 3] = trs[r];
    }
}

/* Stage 1 for one (character, joint): the local 3x4 pose in fp64. */
void orc_local_pose(const float* keys, int32_t n_keys, int32_t n_joints, float fps, int32_t wrap,
                    const orc_layer* layers, int32_t n_layers, int32_t j, double m[12]) {
    double poses[8 * 10], w[8];
    const int32_t nl = n_layers > 8 ? 8 : n_layers;
    for (int32_t l = 0; l < nl; ++l) {
        const float* ck = keys + (size_t)layers[l].clip * n_keys * n_joints * 10;
        orc_sample(ck, n_keys, n_joints, fps, wrap, layers[l].time, j, poses + 10 * l);
        w[l] = (double)layers[l].weight;
    }
    double trs[10];
    orc_blend(nl, poses, w, trs);
    orc_trs_to_matrix(trs, m);
}

typedef struct {
    const int32_t* parents;
    const int32_t* order;
    int32_t n;
    const float* keys;
    int32_t n_keys;
    float fps;
    int32_t wrap;
    const orc_layer* layers;
    int32_t n_layers;
    const double* ib;
    double* global;
    double* skin;
    double* local;          /* optional [n_chars][n][12] output of Stage 1 */
    int64_t c_lo, c_hi;
} anim_job;

static void* anim_worker(void* arg) {
    anim_job* jb = (anim_job*)arg;
    const int32_t n = jb->n;
    double L[12];
    for (int64_t c = jb->c_lo; c < jb->c_hi; ++c) {
        double* G = jb->global + (size_t)c * n * 12;
        double* S = jb->skin + (size_t)c * n * 12;
        const orc_layer* lay = jb->layers + (size_t)c * jb->n_layers;
        for (int32_t k = 0; k < n; ++k) {
            const int32_t j = jb->order[k];
            orc_local_pose(jb->keys, jb->n_keys, n, jb->fps, jb->wrap, lay, jb->n_layers, j, L);
            if (jb->local) memcpy(jb->local + ((size_t)c * n + j) * 12, L, sizeof(L));
            const int32_t p = jb->parents[j];
            if (p == -1) memcpy(G + (size_t)j * 12, L, sizeof(L));
            else orc_compose(G + (size_t)p * 12, L, G + (size_t)j * 12);
            orc_compose(G + (size_t)j * 12, jb->ib + (size_t)j * 12, S + (size_t)j * 12);
        }
    }
    return NULL;
}

/* Stage 1 + Hierarchy-Scan + Bind MeshPose, all in fp64.  layers: [n_chars][n_layers]
 * (n_layers <= 8), keys: [n_clips][n_keys][n][10] fp32.  local_out may be NULL. */
int orc_animate(const int32_t* parents, int32_t n, const float* keys, int32_t n_keys, float fps,
                int32_t wrap, const orc_layer* layers, int32_t n_layers, const float* inv_bind,
                int64_t n_chars, double* global, double* skin, double* local_out, int nthreads) {
    if (n <= 0) return 2;
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    double* ib = (double*)malloc(sizeof(double) * 12 * (size_t)n);
    if (!order || !ib) { free(order); free(ib); return 6; }
    int st = orc_kahn_order(parents, n, order);
    if (st) { free(order); free(ib); return st; }
    for (int32_t j = 0; j < n; ++j)
        for (int e = 0; e < 12; ++e)
            ib[(size_t)j * 12 + e] = inv_bind ? (double)inv_bind[(size_t)j * 12 + e]
                                              : ((e == 0 || e == 5 || e == 10) ? 1.0 : 0.0);
    if (nthreads < 1) nthreads = 1;
    if (n_chars < nthreads) nthreads = n_chars > 0 ? (int)n_chars : 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
    anim_job* jobs = (anim_job*)malloc(sizeof(anim_job) * (size_t)nthreads);
    for (int t = 0; t < nthreads; ++t) {
        anim_job* jb = &jobs[t];
        jb->parents = parents; jb->order = order; jb->n = n; jb->keys = keys; jb->n_keys = n_keys;
        jb->fps = fps; jb->wrap = wrap; jb->layers = layers; jb->n_layers = n_layers; jb->ib = ib;
        jb->global = global; jb->skin = skin; jb->local = local_out;
        jb->c_lo = n_chars * t / nthreads; jb->c_hi = n_chars * (t + 1) / nthreads;
        pthread_create(&th[t], NULL, anim_worker, jb);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(th); free(jobs); free(order); free(ib);
    return 0;
}
