/*
 * oracle/lbs.c — fp64 oracle for linear-blend vertex skinning, the consumer of the
 * skin pose.  TEST INFRASTRUCTURE ONLY, like oracle.c
 * (same library, same rules: only tests/, smoke() and bench.py's baseline legs).
 *
 * Passages: PAPER.md:96 ("compute animation simulation, Hierarchy-Scan, skinning and
 * rendering in the GPU"), PAPER.md:240 (Table 1, "Mesh Face Number 1000-3000"),
 * PAPER.md:60-61 (the skin pose is what skinning consumes).  The paper gives no
 * skinning formula; reading R24 takes standard linear blend skinning:
 *     v'[c][v] = sum_k w[v][k] * ( S[c][j[v][k]] applied to (p[v], 1) )
 * i.e. the weighted sum of the four influencing skin matrices applied to the rest
 * position (weights used as given, no renormalisation), positions only.
 */
#include <stddef.h>
#include <stdint.h>

/* skin: fp64 [n_chars][J][12]; pos f32 [V][3]; joints i32 [V][4] (0 <= j < J);
 * weights f32 [V][4]; out fp64 [n_chars][V][3].  Returns 3 (out of range) on a bad
 * joint index, else 0. */
int orc_skin_vertices(const double* skin, int64_t n_chars, int32_t J, int32_t V, const float* pos,
                      const int32_t* joints, const float* weights, double* out) {
    for (int32_t v = 0; v < V; ++v)
        for (int k = 0; k < 4; ++k)
            if (joints[4 * v + k] < 0 || joints[4 * v + k] >= J) return 3;
    for (int64_t c = 0; c < n_chars; ++c)
        for (int32_t v = 0; v < V; ++v) {
            const double p[3] = {pos[3 * v], pos[3 * v + 1], pos[3 * v + 2]};
            double acc[3] = {0.0, 0.0, 0.0};
            for (int k = 0; k < 4; ++k) {
                const double* S = skin + ((size_t)c * J + joints[4 * v + k]) * 12;
                const double w = (double)weights[4 * v + k];
                for (int r = 0; r < 3; ++r) {
                    const double x = S[4 * r] * p[0] + S[4 * r + 1] * p[1] + S[4 * r + 2] * p[2] + S[4 * r + 3];
                    acc[r] += w * x;
                }
            }
            for (int r = 0; r < 3; ++r) out[((size_t)c * V + v) * 3 + r] = acc[r];
        }
    return 0;
}
