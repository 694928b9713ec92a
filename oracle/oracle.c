/*
 * oracle/oracle.c — plain, slow, obviously-correct fp64 CPU oracle for the
 * Hierarchy-Scan + Bind MeshPose path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  The
 * product path (paper_2505_06703_b200/) never links, imports or calls it, and
 * shares no code, header, table or helper with it.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md):
 *   - §1 steps 2-3: local pose -> model-space (global) pose
 *     -> skin pose "combine model space pose and bindpose".
 *   - Eq. 1 (§3.1): S_i is the product of the matrices on the
 *     root path of joint i.  Written out as the plain recurrence in a
 *     topological order, parent on the LEFT as in Alg. 1's update
 *     "M[jointID] = M[curParentID] * M[jointID]":
 *          G[j] = L[j]                 if Parent(j) == invalid (-1)
 *          G[j] = G[Parent(j)] (x) L[j] otherwise
 *     (reading R1: Eq. 1's child-left order is the row-vector
 *     transpose of the same product.)
 *   - Bind MeshPose: S[j] = G[j] (x) IB[j], IB = inverse
 *     bind pose supplied by the caller (reading R4).
 *   - (x) is affine composition of 3x4 [R|t] matrices with an implicit bottom
 *     row (0,0,0,1):  [Ra|ta] (x) [Rb|tb] = [Ra*Rb | Ra*tb + ta]
 *     (reading R2), with plain * and + in fp64, compiled with
 *     -O2 -ffp-contract=off (no FMA contraction, no fast-math).
 *
 * Deliberately independent of the CUDA path: own parent validation (iterative
 * colouring), own topological order (Kahn / BFS from roots ascending, FIFO —
 * the GPU preprocessor uses DFS preorder), own compose.
 *
 * Pins (tests/test_oracle.py, -m "not gpu"): brute force over all forests with
 * n <= 6 (count checked against Cayley's (n+1)^(n-1)), closed forms (identity,
 * dyadic translation chain == cumsum bitwise, z-rotation chain == Rz(sum),
 * planar polyline), SPEC worked values (tests/golden/), the exact-arithmetic
 * family, np.linalg.multi_dot on chains, and invariants (root, permutation,
 * forest union, bind-pose identity).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { ORC_OK = 0, ORC_EMPTY = 2, ORC_OUT_OF_RANGE = 3, ORC_CYCLE = 4, ORC_NOMEM = 6 };

/* Validate a parent array: n >= 1, -1 <= parent < n, no cycles (a self-parent
 * is a cycle).  Iterative colouring: 0 = unseen, 1 = on the current walk,
 * 2 = known to reach a root. */
int orc_validate(const int32_t* parents, int32_t n) {
    if (n <= 0) return ORC_EMPTY;
    for (int32_t i = 0; i < n; ++i)
        if (parents[i] < -1 || parents[i] >= n) return ORC_OUT_OF_RANGE;
    unsigned char* colour = (unsigned char*)calloc((size_t)n, 1);
    if (!colour) return ORC_NOMEM;
    int status = ORC_OK;
    for (int32_t s = 0; s < n && status == ORC_OK; ++s) {
        int32_t v = s;
        while (v != -1 && colour[v] == 0) { colour[v] = 1; v = parents[v]; }
        if (v != -1 && colour[v] == 1) status = ORC_CYCLE;   /* walked into itself */
        v = s;
        while (v != -1 && colour[v] == 1) { colour[v] = 2; v = parents[v]; }
    }
    free(colour);
    return status;
}

/* Kahn's algorithm: roots in ascending index order enter a FIFO; popping a node
 * appends its children in ascending index order.  order[k] = k-th node. */
int orc_kahn_order(const int32_t* parents, int32_t n, int32_t* order) {
    int st = orc_validate(parents, n);
    if (st != ORC_OK) return st;
    int32_t* first = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
    int32_t* kids = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    int32_t* fill = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
    if (!first || !kids || !fill) { free(first); free(kids); free(fill); return ORC_NOMEM; }
    memset(first, 0, sizeof(int32_t) * (size_t)(n + 1));
    for (int32_t i = 0; i < n; ++i) if (parents[i] >= 0) first[parents[i] + 1]++;
    for (int32_t i = 0; i < n; ++i) first[i + 1] += first[i];
    for (int32_t i = 0; i < n; ++i)          /* ascending i => children ascending */
        if (parents[i] >= 0) kids[first[parents[i]] + fill[parents[i]]++] = i;
    int32_t head = 0, tail = 0;
    for (int32_t i = 0; i < n; ++i) if (parents[i] == -1) order[tail++] = i;
    while (head < tail) {
        int32_t v = order[head++];
        for (int32_t e = first[v]; e < first[v + 1]; ++e) order[tail++] = kids[e];
    }
    free(first); free(kids); free(fill);
    return tail == n ? ORC_OK : ORC_CYCLE;
}

/* C = A (x) B for 3x4 affine [R|t] row-major (element (r,c) at 4r+c). */
void orc_compose(const double* A, const double* B, double* C) {
    for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c)
            C[4 * r + c] = A[4 * r + 0] * B[0 * 4 + c] + A[4 * r + 1] * B[1 * 4 + c] +
                           A[4 * r + 2] * B[2 * 4 + c];
        C[4 * r + 3] = A[4 * r + 0] * B[0 * 4 + 3] + A[4 * r + 1] * B[1 * 4 + 3] +
                       A[4 * r + 2] * B[2 * 4 + 3] + A[4 * r + 3];
    }
}

typedef struct {
    const int32_t* parents;
    const int32_t* order;
    int32_t n;
    const float* local;       /* [n_chars][n][12] */
    const double* ib;         /* [n][12] fp64 (identity when the caller passed NULL) */
    double* global;           /* [n_chars][n][12] or NULL (=> per-thread scratch) */
    double* skin;             /* idem */
    int64_t c_lo, c_hi;
    double checksum;
} scan_job;

static void* scan_worker(void* arg) {
    scan_job* jb = (scan_job*)arg;
    const int32_t n = jb->n;
    double* gs = NULL; double* ss = NULL;
    if (!jb->global) gs = (double*)malloc(sizeof(double) * 12 * (size_t)n);
    if (!jb->skin) ss = (double*)malloc(sizeof(double) * 12 * (size_t)n);
    double sum = 0.0;
    double L[12];
    for (int64_t c = jb->c_lo; c < jb->c_hi; ++c) {
        const float* lc = jb->local + (size_t)c * n * 12;
        double* G = jb->global ? jb->global + (size_t)c * n * 12 : gs;
        double* S = jb->skin ? jb->skin + (size_t)c * n * 12 : ss;
        for (int32_t k = 0; k < n; ++k) {
            int32_t j = jb->order[k];
            for (int e = 0; e < 12; ++e) L[e] = (double)lc[(size_t)j * 12 + e];  /* exact promotion */
            int32_t p = jb->parents[j];
            if (p == -1) memcpy(G + (size_t)j * 12, L, sizeof(L));
            else orc_compose(G + (size_t)p * 12, L, G + (size_t)j * 12);
            orc_compose(G + (size_t)j * 12, jb->ib + (size_t)j * 12, S + (size_t)j * 12);
        }
        if (gs || ss) sum += G[12 * (size_t)(n - 1) + 3] + S[12 * (size_t)(n - 1) + 3];
    }
    jb->checksum = sum;
    free(gs); free(ss);
    return NULL;
}

/* The oracle scan.  local: [n_chars][n][12] fp32 (host), inv_bind: [n][12] fp32
 * or NULL (identity), outputs [n_chars][n][12] fp64 or NULL (then results are
 * computed into per-thread scratch and discarded — the timed-baseline mode).
 * Characters are split over `nthreads` POSIX threads.  *checksum (optional)
 * receives a value depending on the scratch results so the work is observable. */
int orc_scan(const int32_t* parents, int32_t n, const float* local, const float* inv_bind,
             int64_t n_chars, double* global, double* skin, int nthreads, double* checksum) {
    if (n <= 0) return ORC_EMPTY;
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    double* ib = (double*)malloc(sizeof(double) * 12 * (size_t)n);
    if (!order || !ib) { free(order); free(ib); return ORC_NOMEM; }
    int st = orc_kahn_order(parents, n, order);
    if (st != ORC_OK) { free(order); free(ib); return st; }
    for (int32_t j = 0; j < n; ++j)
        for (int e = 0; e < 12; ++e)
            ib[(size_t)j * 12 + e] = inv_bind ? (double)inv_bind[(size_t)j * 12 + e]
                                              : ((e == 0 || e == 5 || e == 10) ? 1.0 : 0.0);
    if (nthreads < 1) nthreads = 1;
    if (n_chars < nthreads) nthreads = n_chars > 0 ? (int)n_chars : 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
    scan_job* jobs = (scan_job*)malloc(sizeof(scan_job) * (size_t)nthreads);
    for (int t = 0; t < nthreads; ++t) {
        scan_job* jb = &jobs[t];
        jb->parents = parents; jb->order = order; jb->n = n; jb->local = local; jb->ib = ib;
        jb->global = global; jb->skin = skin; jb->checksum = 0.0;
        jb->c_lo = n_chars * t / nthreads; jb->c_hi = n_chars * (t + 1) / nthreads;
        pthread_create(&th[t], NULL, scan_worker, jb);
    }
    double sum = 0.0;
    for (int t = 0; t < nthreads; ++t) { pthread_join(th[t], NULL); sum += jobs[t].checksum; }
    if (checksum) *checksum = sum;
    free(th); free(jobs); free(order); free(ib);
    return ORC_OK;
}
