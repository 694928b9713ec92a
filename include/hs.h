/*
 * hs.h — C ABI of the B200-native Hierarchy-Scan + Bind MeshPose library
 * (libhs.so, built from paper_2505_06703_b200/csrc/).
 *
 * The operation (PAPER.md = arxiv 2505.06703, "A GPU-based solution for
 * large-scale skeletal animation simulation"):
 *   - Hierarchy-Scan, §1 step 2 and Eq. 1 (PAPER.md:101-105,
 *     §3.1): for every character c and joint j, the model-space ("global") pose
 *          G[c][j] = L[c][j]                    if Parent(j) == -1
 *          G[c][j] = G[c][Parent(j)] (x) L[c][j] otherwise,
 *     i.e. the product of the local matrices on j's root path, parent on the
 *     LEFT as in Algs. 1-4's update M[joint] = M[parent] * M[joint]
 *     (reading R1).
 *   - Bind MeshPose, §1 step 3: S[c][j] = G[c][j] (x) IB[j],
 *     IB = the skeleton's inverse bind pose (reading R4), fused as the
 *     scan's epilogue.
 *   - (x) = composition of 3x4 affine transforms [R|t] with an implicit bottom
 *     row (0,0,0,1): [Ra|ta](x)[Rb|tb] = [Ra Rb | Ra tb + ta] (reading R2).
 *
 * Data layout (all pose arrays): float32 [n_chars][n_joints][3][4], row-major,
 * element (r,c) of joint j of character ch at ((ch*n_joints + j)*12 + 4r + c);
 * column 3 is the translation.  Joint indices are the USER's labels, in any
 * order (parents may have larger indices than children); outputs are in the
 * same user order.  Forests (several roots) are allowed.
 *
 * Errors: every function returns hs_status (HS_OK = 0) and never throws or
 * aborts across the ABI; hs_last_error() returns a thread-local detail string.
 * CUDA launch errors are reported via cudaGetLastError (no device sync).
 * NaN/Inf inputs are not validated; they propagate.
 */
#ifndef HS_H_
#define HS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    HS_OK = 0,
    HS_ERR_INVALID_ARG = 1,   /* null pointer, n < 0, misaligned (16 B), size overflow, aliasing */
    HS_ERR_EMPTY = 2,         /* n_joints == 0                                  (SPEC Empty)      */
    HS_ERR_OUT_OF_RANGE = 3,  /* parent < -1 or parent >= n_joints              (SPEC OutOfRange) */
    HS_ERR_CYCLE = 4,         /* a parent chain loops, self-parent included     (SPEC CycleDetected) */
    HS_ERR_CUDA = 5,          /* CUDA runtime error (detail in hs_last_error)   */
    HS_ERR_OOM = 6,           /* host or device allocation failed               */
    HS_ERR_WRONG_DEVICE = 7,  /* handle used on a device other than its own     */
    HS_ERR_UNSUPPORTED = 8    /* n_joints above HS_MAX_JOINTS, or an option this build lacks */
} hs_status;

#define HS_MAX_JOINTS (1 << 20)

typedef struct hs_skeleton hs_skeleton;   /* opaque; immutable after create */

/* Build a skeleton handle on the CURRENT CUDA device.
 *   parents  : host, [n_joints], parents[j] = parent label or -1 (root); any order.
 *   inv_bind : host, [n_joints][3][4] fp32, or NULL (identity).  Copied.
 *   out      : receives the handle (unchanged on error).
 * Runs the host topology preprocessor once (validation, levels, internal
 * topological order, pointer-jumping schedule, chunk/anchor program;
 * PAPER.md:126-130 Eq. 2, :146-175 blocks / MaxParentOutBlock, :154 in-order
 * list) and uploads its tables.  Errors: HS_ERR_EMPTY, HS_ERR_OUT_OF_RANGE,
 * HS_ERR_CYCLE, HS_ERR_INVALID_ARG (null parents/out, n_joints < 0),
 * HS_ERR_UNSUPPORTED (n_joints > HS_MAX_JOINTS), HS_ERR_OOM, HS_ERR_CUDA. */
hs_status hs_skeleton_create(const int32_t* parents, int32_t n_joints, const float* inv_bind,
                             hs_skeleton** out);

/* Creation options (hs_skeleton_create uses all-zero = automatic). */
typedef struct {
    int32_t chunk;        /* K, joints per thread chunk: odd in 3..11; 0 = auto (5)            */
    int32_t tile_joints;  /* target joints per CTA tile (chars per tile = max(1, this / n));
                             0 = auto (1024)                                                  */
    int32_t force_split;  /* 1 = use the multi-CTA program even when one CTA would fit          */
    int32_t stages;       /* TMA load stages of the chunked kernel (2 or 3); 0 = auto           */
    int32_t sbufs;        /* skin staging buffers (1 or 2); 0 = auto                            */
    int32_t pbuf;         /* anchor buffer P: 2 = ping-pong (one barrier per round), 1 = single
                             buffer (two barriers per round, half the shared memory); 0 = auto */
    int32_t chunking;     /* thread chunks: 1 = runs of K consecutive internal positions (the
                             paper's index blocks), 2 = heavy-path pieces packed per thread
                             (fewer anchors), 3 = heavy paths longer than K on consecutive
                             lanes joined by a warp-shuffle scan (fewest anchors, shallow
                             anchor forest); 0 = auto: 3 for one-character tiles when it at
                             least halves the pointer-jumping work, else 2 when it cuts that
                             work without adding threads per character, else 1              */
    int32_t reserved[1];  /* must be zero                                                      */
} hs_create_opts;

/* hs_skeleton_create with explicit options (opts == NULL: automatic).
 * Extra errors: HS_ERR_INVALID_ARG for an invalid option value. */
hs_status hs_skeleton_create_ex(const int32_t* parents, int32_t n_joints, const float* inv_bind,
                                const hs_create_opts* opts, hs_skeleton** out);

/* Hierarchy-Scan + fused Bind MeshPose for n_chars characters sharing `sk`.
 *   local      : device, [n_chars][n_joints][3][4] fp32, 16-byte aligned, read-only.
 *   n_chars    : >= 0; 0 is a no-op.
 *   global_out : device, same shape; receives G.  Must not alias local or skin_out.
 *   skin_out   : device, same shape; receives S = G (x) IB.  Must not alias.
 *                NULL skips the Bind MeshPose epilogue (global pose only).
 *   cuda_stream: cudaStream_t (NULL = legacy default stream).
 * Asynchronous and stream-ordered: no device synchronisation and no host<->
 * device copies.  Skeletons beyond one CTA's shared memory (the multi-CTA
 * path) take a stream-ordered workspace from a library-owned CUDA memory pool
 * (cudaMallocFromPoolAsync; the pool keeps its memory for the next call).  Buffers must
 * stay valid until the stream work completes.  Errors: HS_ERR_INVALID_ARG,
 * HS_ERR_WRONG_DEVICE, HS_ERR_CUDA, HS_ERR_OOM. */
hs_status hs_scan(const hs_skeleton* sk, const float* local, int64_t n_chars, float* global_out,
                  float* skin_out, void* cuda_stream);

/* Algorithms selectable through hs_scan_ex (tests / comparisons). */
typedef enum {
    HS_ALGO_AUTO = 0,       /* = CHUNKED when the skeleton fits one CTA; else TILES for crowds
                               of at least as many characters as the GPU has SMs (one CTA per
                               character at a time), SPLIT for smaller crowds               */
    HS_ALGO_CHUNKED = 1,    /* persistent TMA tile kernel: per-thread serial chunks + pointer
                               jumping over chunk anchors                       */
    HS_ALGO_DOUBLING = 2,   /* Alg. 2: radix-2 pointer jumping, one thread per
                               joint, ceil(log2 L) rounds; honours max_rounds                    */
    HS_ALGO_SPLIT = 3,      /* multi-CTA path (PAPER.md:145-175 generalised): phase-1 kernel,
                               recursive anchor scan, phase-3 kernel.  Available when the
                               skeleton does not fit one CTA or was created with force_split  */
    HS_ALGO_GATEAU = 4,     /* Alg. 1: thread per joint walks every ancestor   */
    HS_ALGO_LEAF = 5,       /* KIYA leaf walk: thread per leaf fills its root path */
    HS_ALGO_BLOCKED = 6,    /* Alg. 3 literally: 64-joint blocks, in-block
                               doubling clamped to the block, then the MaxParentOutBlock walk;
                               n_joints <= 1024                                                */
    HS_ALGO_TILES = 7,      /* multi-tile path for skeletons beyond one CTA (
                               Alg. 3's cross-block carry): the topological
                               order cut into CTA tiles; a persistent CTA runs a character's
                               tiles in order, importing the final global poses of earlier
                               tiles' joints from a per-CTA workspace (L2), so each joint is
                               read and written once (144 B/joint).  Available when the
                               skeleton does not fit one CTA or was created with force_split   */
    HS_ALGO_COMPRESSED = 8  /* Alg. 4 literally: 64-joint groups, 7 serial
                               composes with in-group ancestors at distance 1..7, a barrier,
                               7 stride-8 composes on that snapshot, a barrier, then the
                               MaxParentOutBlock walk; n_joints <= 1024                        */
} hs_algo;

typedef struct {
    int32_t algo;        /* hs_algo                                                          */
    int32_t max_rounds;  /* DOUBLING only: stop after this many rounds (< 0 = all); the
                            round-induction test                          */
    int32_t tile_ctas;   /* CHUNKED: CTAs per SM for the persistent grid (0 = occupancy max)  */
    int32_t reserved[5]; /* must be zero                                                     */
} hs_scan_opts;

/* hs_scan with explicit options; opts == NULL behaves as hs_scan. */
hs_status hs_scan_ex(const hs_skeleton* sk, const float* local, int64_t n_chars, float* global_out,
                     float* skin_out, void* cuda_stream, const hs_scan_opts* opts);

/* ---------------------------------------------------------------------------
 * Heterogeneous single launch ("varied
 * hierarchies"): several crowds, each with its own skeleton, scanned by ONE kernel
 * launch.  Their tiles form one global tile space over the persistent CTAs, which
 * switch programs at segment boundaries, so the per-launch pipeline fill/drain and
 * tails of separate hs_scan calls disappear.  Results are bitwise identical to
 * calling hs_scan on each item in order (characters are chunked per character and
 * the per-skeleton tile size is kept).  Measured on B200: 2.9x
 * faster than per-type hs_scan for 8 types x 64 characters, break-even near 32 tiles
 * per SM per type; above that separate hs_scan calls are ~3 % faster.
 *   items     host array of n_items descriptors (read during the call only); each
 *             item's buffers follow hs_scan's rules (device, 16-byte aligned, no
 *             aliasing); distinct items must not overlap in memory.
 *   n_items   0..HS_MAX_BATCH; items with n_chars == 0 are skipped.
 * Every skeleton must be on the single-CTA path (HS_Q_PATH == HS_ALGO_CHUNKED), use
 * the same chunk size (HS_Q_CHUNK) and live on the current device; otherwise
 * HS_ERR_UNSUPPORTED / HS_ERR_WRONG_DEVICE and nothing is launched.
 * ------------------------------------------------------------------------- */
#define HS_MAX_BATCH 8
typedef struct {
    const hs_skeleton* skeleton;
    const float* local;     /* device [n_chars][n_joints][3][4]                          */
    int64_t n_chars;
    float* global_out;      /* device, same shape                                        */
    float* skin_out;        /* device, same shape, or NULL (no bind epilogue)             */
} hs_batch_item;
hs_status hs_scan_batch(const hs_batch_item* items, int32_t n_items, void* cuda_stream);

/* Per-character topology ("and/or per-character topology"):
 * every character has its own skeleton, so nothing is planned ahead.  Pointer jumping
 * with the parent pointers themselves (Alg. 2, with the Eq. 2 lift
 * built on the fly): ceil(log2 L) rounds per character group.
 *   parents   device int32 [n_chars][n_joints], character-local labels, -1 = root,
 *             any order; an entry outside [-1, n_joints) is treated as a root; a cycle
 *             gives undefined values but the launch terminates (bounded rounds).
 *   local     device fp32 [n_chars][n_joints][3][4] (16-byte aligned)
 *   inv_bind  device fp32 [n_chars][n_joints][3][4] per-character inverse binds, or
 *             NULL (skin = global)
 *   n_joints  1..1024 (HS_ERR_UNSUPPORTED above); outputs as hs_scan. */
hs_status hs_scan_varied(const int32_t* parents, const float* local, const float* inv_bind, int32_t n_joints,
                         int64_t n_chars, float* global_out, float* skin_out, void* cuda_stream);

/* ---------------------------------------------------------------------------
 * Linear blend skinning fused after the bind epilogue (
 * PAPER.md:96 "compute animation simulation, Hierarchy-Scan, skinning and rendering
 * in the GPU", PAPER.md:240 meshes of 1000-3000 faces).  The paper gives no formula;
 * DESIGN.md reading R24: per character c and vertex v,
 *     verts[c][v] = sum_{k<4} w[v][k] * S[c][j[v][k]] (p[v], 1)
 * with S = G (x) IB the skin pose, weights used as given, positions only.  The skin
 * palette of a tile never leaves shared memory (skin_out may be NULL).
 * ------------------------------------------------------------------------- */
typedef struct hs_mesh hs_mesh;

/* pos: host fp32 [n_vertices][3] rest positions (bind space); joints: host int32
 * [n_vertices][4] influencing joints (user labels, each in [0, n_joints)); weights:
 * host fp32 [n_vertices][4] (a 0 weight disables an influence).  Copied to the
 * current device.  Errors: HS_ERR_INVALID_ARG (null, n_vertices outside 1..2^24),
 * HS_ERR_OUT_OF_RANGE (a joint index), HS_ERR_UNSUPPORTED (n_joints > 65535). */
hs_status hs_mesh_create(const hs_skeleton* sk, int32_t n_vertices, const float* pos, const int32_t* joints,
                         const float* weights, hs_mesh** out);
hs_status hs_mesh_destroy(hs_mesh* mesh);

/* hs_scan (G, and S when skin_out != NULL) plus skinned vertex positions:
 *   verts_out  device fp32 [n_chars][n_vertices][3], 4-byte aligned, not aliasing
 *              the other buffers.
 * The mesh must have been created for this skeleton (HS_ERR_INVALID_ARG).  Same as
 * hs_scan_skin_ex with opts == NULL. */
hs_status hs_scan_skin(const hs_skeleton* sk, const hs_mesh* mesh, const float* local, int64_t n_chars,
                       float* global_out, float* skin_out, float* verts_out, void* cuda_stream);

/* Where skinning runs.  FUSED: in the scan kernel after the bind epilogue, the
 * palette never leaves shared memory (single-CTA skeletons only).  TWO_PASS: the
 * scan writes S (to skin_out, or to a stream-ordered pooled workspace of
 * workspace_bytes, default 1 GiB, in batches) and a skinning kernel with several
 * CTAs per SM reads it back (+48 B/joint of HBM; any skeleton whose palette fits
 * shared memory with the character's vertices: 48 n_joints + 12 n_vertices <= 227 KB).
 * The two-pass kernel processes vertices in joint-sorted order (palette reads become
 * shared-memory broadcasts) and stages them in smem to write them out in the caller's
 * order.  AUTO = TWO_PASS when n_vertices >= 2 n_joints or the skeleton is multi-CTA,
 * else FUSED.  Both compute each vertex with the same device code:
 * bitwise equal results. */
typedef enum { HS_SKIN_AUTO = 0, HS_SKIN_FUSED = 1, HS_SKIN_TWO_PASS = 2 } hs_skin_mode;
typedef struct {
    int32_t mode;             /* hs_skin_mode                                            */
    int32_t reserved0;        /* must be 0                                               */
    int64_t workspace_bytes;  /* TWO_PASS with skin_out == NULL (0 = 1 GiB)             */
    int64_t reserved[2];      /* must be 0                                               */
} hs_skin_opts;
hs_status hs_scan_skin_ex(const hs_skeleton* sk, const hs_mesh* mesh, const float* local, int64_t n_chars,
                          float* global_out, float* skin_out, float* verts_out, void* cuda_stream,
                          const hs_skin_opts* opts);

/* Skinning alone, from skin poses already on the device (e.g. hs_animate's skin_out):
 *   skin     device fp32 [n_chars][n_joints][3][4] (16-byte aligned), n_joints = the
 *            mesh's skeleton
 *   verts_out device fp32 [n_chars][n_vertices][3] (4-byte aligned)
 * The two-pass LBS kernel (joint-sorted vertices, smem-staged output; the palette and
 * the vertices must fit shared memory: HS_ERR_UNSUPPORTED otherwise).  Together with
 * hs_animate this runs the paper's whole GPU pipeline: simulation,
 * Hierarchy-Scan, bind, skinning. */
hs_status hs_skin_vertices(const hs_mesh* mesh, const float* skin, int64_t n_chars, float* verts_out,
                           void* cuda_stream);

/* ---------------------------------------------------------------------------
 * Stage 1 fused ahead of the scan ("Sample
 * animation data and generate local pose in local space").
 * Per character and joint: sample each animation layer's clip at its time (keys
 * uniformly spaced at `fps`; linear t/s, normalised-lerp rotation with the
 * shortest-arc sign fix; an exact key time returns the key), blend the layers
 * (weights normalised; quaternions sign-aligned to layer 0; one layer = its
 * sample), build L = [R(q) diag(s) | t], then Hierarchy-Scan + Bind as hs_scan.
 * The local poses never touch HBM (96 instead of 144 bytes per joint).
 * ------------------------------------------------------------------------- */
typedef struct hs_clipset hs_clipset;

/* keys: host fp32 [n_clips][n_keys][n_joints][10] = t(3), q(w,x,y,z), s(3), for the
 * skeleton `sk` (same n_joints); key k of a clip is at time k / fps; wrap: 0 = clamp,
 * 1 = loop (duration = (n_keys - 1) / fps).  Copied to the handle's device. */
hs_status hs_clipset_create(const hs_skeleton* sk, const float* keys, int32_t n_clips, int32_t n_keys,
                            float fps, int32_t wrap, hs_clipset** out);
hs_status hs_clipset_destroy(hs_clipset* cs);

/* One animation layer of one character (16 bytes). */
typedef struct {
    int32_t clip;      /* clip index in the clip set; values outside [0, n_clips) are
                          clamped to the nearest valid clip on the device (no error:
                          layers are device data and are not validated per call)   */
    float time;        /* seconds                                                     */
    float weight;      /* blend weight; the weights of a character must have a
                          positive sum (SPEC.md WeightSumZero): a sum <= 0 is not
                          detected on the device and yields non-finite poses        */
    int32_t reserved;  /* ignored                                                     */
} hs_layer;

/* layers: device [n_chars][n_layers] hs_layer (n_layers 1..8), 16-byte aligned; outputs
 * as hs_scan.  Same as hs_animate_ex with opts == NULL (two-pass: any skeleton). */
hs_status hs_animate(const hs_skeleton* sk, const hs_clipset* cs, const void* layers, int32_t n_layers,
                     int64_t n_chars, float* global_out, float* skin_out, void* cuda_stream);

/* How Stage 1 meets the scan.  FUSED: computed in shared memory inside the scan
 * kernel (96 B/joint of HBM traffic).  TWO_PASS: a streaming Stage-1 kernel writes the
 * local poses of a batch of characters to a workspace (stream-ordered cudaMallocAsync,
 * workspace_bytes, default 1 GiB) and the plain scan reads them back (192 B/joint),
 * which hides the key-load latency better, and works for multi-CTA skeletons too
 * (FUSED needs a single-CTA skeleton: HS_ERR_UNSUPPORTED otherwise).  AUTO = TWO_PASS
 * (measured faster on B200).  Both produce bitwise the same local
 * poses, hence the same output. */
typedef enum { HS_ANIMATE_AUTO = 0, HS_ANIMATE_FUSED = 1, HS_ANIMATE_TWO_PASS = 2 } hs_animate_mode;
typedef struct {
    int32_t mode;             /* hs_animate_mode                                        */
    int32_t reserved0;        /* must be 0                                              */
    int64_t workspace_bytes;  /* TWO_PASS batch workspace (0 = 1 GiB; >= one character) */
    int64_t reserved[2];      /* must be 0                                              */
} hs_animate_opts;
hs_status hs_animate_ex(const hs_skeleton* sk, const hs_clipset* cs, const void* layers, int32_t n_layers,
                        int64_t n_chars, float* global_out, float* skin_out, void* cuda_stream,
                        const hs_animate_opts* opts);

/* The paper's whole GPU pipeline in one call: Stage 1 (two-pass
 * placement), Hierarchy-Scan, bind and linear blend skinning of `mesh` (hs_mesh
 * below; the scan + skinning of each Stage-1 batch runs as hs_scan_skin with AUTO
 * placement).  Outputs as hs_animate plus verts_out [n_chars][n_vertices][3]. */
hs_status hs_animate_skin(const hs_skeleton* sk, const hs_clipset* cs, const void* layers, int32_t n_layers,
                          int64_t n_chars, const hs_mesh* mesh, float* global_out, float* skin_out,
                          float* verts_out, void* cuda_stream);

/* Destroy a handle (NULL-safe).  The caller guarantees no hs_scan using it is
 * still in flight.  Frees its device tables with cudaFree (device-synchronising). */
hs_status hs_destroy(hs_skeleton* sk);

/* Queries (integer results). */
typedef enum {
    HS_Q_N_JOINTS = 0,
    HS_Q_MAX_LEVEL = 1,      /* L: node count of the longest root path (root level = 1)      */
    HS_Q_ROUNDS = 2,         /* R = ceil(log2 L): Alg. 2 rounds                               */
    HS_Q_PATH = 3,           /* algo HS_ALGO_AUTO resolves to for a large crowd (HS_ALGO_CHUNKED,
                                or HS_ALGO_TILES beyond one CTA; SPLIT if TILES is unavailable) */
    HS_Q_CHUNK = 4,          /* K: joints per thread chunk                                     */
    HS_Q_TILE_CHARS = 5,     /* characters per CTA tile (chunked path)                         */
    HS_Q_ANCHORS = 6,        /* anchor slots per tile (chunked) / per character (split)        */
    HS_Q_ANCHOR_ROUNDS = 7,  /* pointer-jumping rounds over anchors                            */
    HS_Q_IDENTITY_ORDER = 8, /* 1 if the user order is already topological (no gather)         */
    HS_Q_SMEM_BYTES = 9,     /* dynamic shared memory per CTA of the chunked kernel            */
    HS_Q_THREADS = 10,       /* threads per CTA of the chunked kernel (incl. producer warp)    */
    HS_Q_STAGES = 11,        /* TMA load stages                                                */
    HS_Q_DEVICE = 12,        /* CUDA device ordinal the handle lives on                        */
    HS_Q_SPLIT_LEVELS = 13,  /* recursion depth of the multi-CTA path (0 if single-CTA)         */
    HS_Q_PBUFS = 15,         /* anchor buffers of the chunked kernel (2 ping-pong, 1 single)    */
    HS_Q_SBUFS = 16,         /* skin staging buffers of the chunked kernel                      */
    HS_Q_CHUNKING = 17,      /* chunk construction in use (1 consecutive, 2 heavy-path pieces)  */
    HS_Q_TILE_SLOTS = 18,    /* plan only: P slots of the one-character tile program            */
    HS_Q_TILE_ROUNDS_ENTRIES = 19, /* plan only: phase-2 descriptors of that program           */
    HS_Q_TILE_R2 = 20,       /* plan only: its pointer-jumping rounds                           */
    HS_Q_SMALL_TILE_CHARS = 21, /* characters per tile of the small-crowd twin program (0 = none):
                                  hs_scan runs it when the default tiles would not cover the SMs */
    HS_Q_SEQ_TILES = 22,     /* HS_ALGO_TILES: tiles per character (0 = not available)         */
    HS_Q_SEQ_TILE_JOINTS = 23, /* HS_ALGO_TILES: joints per tile (F)                            */
    HS_Q_SEQ_EXPORTS = 24,   /* HS_ALGO_TILES: joints with a child in a later tile (workspace
                                slots per CTA)                                                 */
    HS_Q_SEQ_SMEM_BYTES = 25, /* HS_ALGO_TILES: dynamic shared memory per CTA                 */
    HS_Q_SEQ_THREADS = 26,   /* plan only: compute threads of the multi-tile program (T)        */
    HS_Q_SEQ_SLOTS = 27,     /* plan only: anchor slots per P buffer (S)                       */
    HS_Q_SEQ_R2MAX = 28,     /* plan only: most pointer-jumping rounds of a tile               */
    HS_Q_SEQ_ENTRIES = 29,   /* plan only: phase-2 descriptors of all tiles                    */
    HS_Q_SEQ_IMPORTS = 30,   /* plan only: import pairs of all tiles                           */
    HS_Q_SEQ_RUNS = 31,      /* plan only: TMA runs of all tiles                               */
    HS_Q_SEQ_QSLOTS = 32,    /* plan only: Q locations (most imports of a tile)                */
    HS_Q_SEQ_CHUNK = 33,     /* HS_ALGO_TILES: chunk K of the multi-tile program                */
    HS_Q_SEQ_SBUFS = 34      /* HS_ALGO_TILES: skin / inverse-bind buffers                      */
} hs_query;

hs_status hs_skeleton_query(const hs_skeleton* sk, int32_t what, int64_t* value);

const char* hs_status_string(hs_status s);
const char* hs_last_error(void);

/* Workspaces (two-pass hs_animate / hs_scan_skin, the multi-CTA path) come from a
 * library-owned stream-ordered pool per device that keeps its memory between calls,
 * so steady-state frames allocate nothing.  hs_workspace_trim returns the pool's
 * unused memory of the CURRENT device to the driver (outstanding work keeps what it
 * holds); *held_bytes (may be NULL) receives what the pool still reserves.  Safe to
 * call at any time; HS_OK if the pool was never created. */
hs_status hs_workspace_trim(int64_t* held_bytes);

/* ---------------------------------------------------------------------------
 * Host-only topology plan (no CUDA calls): the preprocessor hs_skeleton_create
 * runs, exposed for tests and tools.  Exports are in USER labels unless noted.
 * ------------------------------------------------------------------------- */
typedef struct hs_plan hs_plan;

/* parents as in hs_skeleton_create; chunk = K (odd, 3..11; 0 = auto); the plan's
 * chunk program uses chunking 3 (runs); block_size = the paper's block size for the
 * MaxParentOutBlock export (0 = 64). */
hs_status hs_plan_create(const int32_t* parents, int32_t n_joints, int32_t chunk,
                         int32_t block_size, hs_plan** out);
/* The same with the creation options that shape the program (chunk K, chunking). */
hs_status hs_plan_create_ex(const int32_t* parents, int32_t n_joints, const hs_create_opts* opts,
                            int32_t block_size, hs_plan** out);
hs_status hs_plan_query(const hs_plan* p, int32_t what, int64_t* value);

typedef enum {
    HS_X_LEVELS = 0,       /* int32 [n]   level of each joint (root = 1)                         */
    HS_X_ORDER = 1,        /* int32 [n]   internal position -> user label (topological order)     */
    HS_X_LIFT = 2,         /* int32 [R][n] anc[r][u] = 2^r-th ancestor of u (user labels), -1     */
    HS_X_BLOCK_OF = 3,     /* int32 [n]   block of each INTERNAL position (position / block_size) */
    HS_X_MPOB = 4,         /* int32 [n]   MaxParentOutBlock of each INTERNAL position, internal
                                          position of the nearest ancestor in another block, -1   */
    HS_X_CHUNK_SRC = 5,    /* int32 [n]   per INTERNAL position: -1 root, -2 previous joint of the
                                          same chunk list, >= 0 anchor = internal position of parent */
    HS_X_ANCHOR_LINK = 6,  /* int32 [A]   per anchor slot (ascending internal position): link to
                                          the anchor slot of its segment head's parent, or -1     */
    HS_X_CHUNK_LISTS = 7,  /* int32 [T][K] internal positions of each thread's chunk, -1 padded
                                          (T = HS_Q_THREADS of the plan)                           */
    /* The chunked kernel's tile program for ONE character (ping-pong P), as uploaded: */
    HS_X_TILE_META = 8,    /* uint64 [T][K]: user joint | ibu<<16 | int16 src<<32 | int16 own<<48;
                              src: -1 root, -2 previous, -3 none, >= 0 P location of the parent */
    HS_X_TILE_P1LEN = 9,   /* int32 [T]: phase-1 length of each thread                          */
    HS_X_TILE_ROUND_OFF = 10, /* int32 [R2+1]: start of each pointer-jumping round              */
    HS_X_TILE_ROUNDS = 11, /* uint32 [E]: slot | dst buffer<<14 | self buffer<<15 | link loc<<16 */
    /* The multi-tile program (HS_ALGO_TILES) as uploaded (sizes from the HS_Q_SEQ_* queries;
       built for the plan's options with F = tile_joints or 1024, shrunk until it fits): */
    HS_X_SEQ_TILES = 12,   /* int32 [KT][12]: first, nj, R2, entries, rounds_off, n_imp, imp_off,
                              n_runs, runs_off, T, 0, 0                                       */
    HS_X_SEQ_META = 13,    /* uint64 [KT][T][K]: smem offset (10 bits) | (src + 8)<<10 (13) |
                              (own + 1)<<23 (13) | (workspace export slot + 1)<<36 (16) |
                              (next tile's Q index + 1)<<52 (12); src >= 2S: a Q location
                              (2S + (k & 1) nQ + index)                                        */
    HS_X_SEQ_P1LEN = 14,   /* int32 [KT][T]                                                     */
    HS_X_SEQ_ROUND_OFF = 15, /* int32 [KT][R2max+1 rounded up to 4], relative to rounds_off      */
    HS_X_SEQ_ROUNDS = 16,  /* uint32 [E] (all tiles; each tile's records padded to 4)           */
    HS_X_SEQ_IMP = 17,     /* int32 [I][2]: workspace slot, Q location (parents two or more
                              tiles back; a parent in the previous tile is forwarded); each
                              tile's pairs padded to an even count                              */
    HS_X_SEQ_RUNS = 18,    /* int32 [R][4]: user start, smem offset, length, 0                  */
    HS_X_SEQ_IB_USER = 19  /* int32 [KT][F]: user label at each smem offset (-1 = none)          */
} hs_plan_export_what;

/* Copy an export into buf (buf_bytes must be >= the export's size). */
hs_status hs_plan_export(const hs_plan* p, int32_t what, void* buf, int64_t buf_bytes);
hs_status hs_plan_destroy(hs_plan* p);

/* ---------------------------------------------------------------------------
 * Host-buffer entry point (end-to-end): H2D of local, scan, D2H of global and
 * skin, pipelined over character batches on the pipeline's own streams.
 * Synchronous: returns when h_global / h_skin hold the results.  Host buffers
 * should be page-locked (cudaHostAlloc / torch pin_memory) for full PCIe rate.
 * ------------------------------------------------------------------------- */
typedef struct hs_pipeline hs_pipeline;

/* batch_bytes: device staging per buffer set (0 = 256 MiB); created on the
 * current device with 3 buffer sets and 3 streams. */
hs_status hs_pipeline_create(int64_t batch_bytes, hs_pipeline** out);
hs_status hs_scan_host(hs_pipeline* pl, const hs_skeleton* sk, const float* h_local,
                       int64_t n_chars, float* h_global, float* h_skin);

/* The same over several crowds (any skeletons): items hold HOST pointers here
 * (local, global_out and skin_out all required), n_items >= 0.  One pipeline runs
 * through every item's characters, so the copy engines do not drain between skeleton
 * types.  Errors as hs_scan_host. */
hs_status hs_scan_host_batch(hs_pipeline* pl, const hs_batch_item* items, int32_t n_items);

/* Stage 1 + scan + bind from HOST buffers: h_layers [n_chars][n_layers] hs_layer (host),
 * outputs as hs_scan_host.  Per batch: layers up, hs_animate (two-pass) on the device,
 * global and skin poses back. */
hs_status hs_animate_host(hs_pipeline* pl, const hs_skeleton* sk, const hs_clipset* cs, const void* h_layers,
                          int32_t n_layers, int64_t n_chars, float* h_global, float* h_skin);
hs_status hs_pipeline_destroy(hs_pipeline* pl);

#ifdef __cplusplus
}
#endif
#endif /* HS_H_ */
