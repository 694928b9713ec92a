/* hs_demo.c — a plain C client of the C ABI (include/hs.h), no CUDA calls of its own:
 * builds a small skeleton, animates a crowd on the host, runs Hierarchy-Scan + Bind
 * through the host-buffer pipeline (hs_scan_host: H2D, scan, D2H inside the library)
 * and checks every result against a straightforward float64 walk of the hierarchy
 * (G_j = G_parent(j) L_j, S_j = G_j IB_j; Eq. 1 with the parent on
 * the left).  Exit status 0 on success.
 *
 *   build: gcc -std=c11 -O2 examples/hs_demo.c -Iinclude -Lpaper_2505_06703_b200 -lhs \
 *          -Wl,-rpath,'$ORIGIN/../paper_2505_06703_b200' -lm -o examples/hs_demo
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "hs.h"

#define J 13
#define N_CHARS 1000

/* a small biped: pelvis, spine chain, two arms, two legs; parents listed first */
static const int32_t kParents[J] = {-1, 0, 1, 2, 3, 2, 5, 2, 7, 0, 9, 0, 11};

static uint64_t rng_state = 0x2505067030ull;
static double urand(void) {   /* xorshift64*, uniform in [0, 1) */
    rng_state ^= rng_state >> 12;
    rng_state ^= rng_state << 25;
    rng_state ^= rng_state >> 27;
    return (double)((rng_state * 2685821657736338717ull) >> 11) * (1.0 / 9007199254740992.0);
}

/* a random rigid transform: unit quaternion -> rotation, translation in [-1, 1]^3 */
static void random_pose(float* m) {
    double q[4], n = 0.0;
    for (int i = 0; i < 4; ++i) { q[i] = 2.0 * urand() - 1.0; n += q[i] * q[i]; }
    n = sqrt(n);
    const double w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
    const double r[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                         2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                         2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
    for (int i = 0; i < 3; ++i) {
        for (int k = 0; k < 3; ++k) m[4 * i + k] = (float)r[3 * i + k];
        m[4 * i + 3] = (float)(2.0 * urand() - 1.0);
    }
}

/* c = a (x) b for 3x4 affine matrices in float64 */
static void compose64(const double* a, const double* b, double* c) {
    for (int i = 0; i < 3; ++i) {
        for (int k = 0; k < 4; ++k) {
            double s = k == 3 ? a[4 * i + 3] : 0.0;
            for (int t = 0; t < 3; ++t) s += a[4 * i + t] * b[4 * t + k];
            c[4 * i + k] = s;
        }
    }
}

int main(void) {
    const size_t per = (size_t)N_CHARS * J * 12;
    float* local = malloc(per * sizeof(float));
    float* global = malloc(per * sizeof(float));
    float* skin = malloc(per * sizeof(float));
    float inv_bind[J * 12];
    if (!local || !global || !skin) return 2;
    for (int j = 0; j < J; ++j) random_pose(inv_bind + 12 * j);
    for (size_t e = 0; e < (size_t)N_CHARS * J; ++e) random_pose(local + 12 * e);

    hs_skeleton* sk = NULL;
    hs_pipeline* pl = NULL;
    hs_status s = hs_skeleton_create(kParents, J, inv_bind, &sk);
    if (s == HS_OK) s = hs_pipeline_create(0, &pl);
    if (s == HS_OK) s = hs_scan_host(pl, sk, local, N_CHARS, global, skin);
    if (s != HS_OK) {
        fprintf(stderr, "hs_demo: %s (%s)\n", hs_status_string(s), hs_last_error());
        return 1;
    }
    int64_t rounds = 0;
    hs_skeleton_query(sk, HS_Q_ROUNDS, &rounds);

    double worst = 0.0;
    for (int c = 0; c < N_CHARS; ++c) {
        double G[J][12];
        for (int j = 0; j < J; ++j) {   /* parents come first in kParents: one pass */
            double L[12], S[12], IB[12];
            for (int e = 0; e < 12; ++e) L[e] = local[((size_t)c * J + j) * 12 + e];
            if (kParents[j] < 0) {
                for (int e = 0; e < 12; ++e) G[j][e] = L[e];
            } else {
                compose64(G[kParents[j]], L, G[j]);
            }
            for (int e = 0; e < 12; ++e) IB[e] = inv_bind[12 * j + e];
            compose64(G[j], IB, S);
            for (int e = 0; e < 12; ++e) {
                const double dg = fabs(G[j][e] - global[((size_t)c * J + j) * 12 + e]);
                const double ds = fabs(S[e] - skin[((size_t)c * J + j) * 12 + e]);
                if (dg > worst) worst = dg;
                if (ds > worst) worst = ds;
            }
        }
    }
    printf("hs_demo: %d characters x %d joints, %lld pointer-jumping rounds, max |err| %.3g\n", N_CHARS, J,
           (long long)rounds, worst);
    hs_pipeline_destroy(pl);
    hs_destroy(sk);
    free(local);
    free(global);
    free(skin);
    return worst <= 1e-4 ? 0 : 3;
}
