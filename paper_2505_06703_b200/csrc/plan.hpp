// plan.hpp — host topology preprocessor for the Hierarchy-Scan (runs once per
// skeleton, never per frame; no CUDA).  See DESIGN.md §5.
//
// What it builds, and the passages it implements:
//   * validation: range / cycle / empty (SPEC.md:63-72 errors; a forward parent
//     is accepted and reordered — DESIGN.md reading R17);
//   * levels, L and R = ceil(log2 L) (Table 1 "hierarchy layer");
//   * internal topological order: the user order when it is already topological
//     (parent < child), else DFS preorder with roots/children ascending
//     ("traversing the skeleton tree in order ... the parent node of any tree node
//     must have a smaller sequence number");
//   * Eq. 2 MultiParent lift table anc[r][j] = 2^r-th ancestor,
//     used by the Alg. 2 doubling kernel;
//   * the paper's block layout / MaxParentOutBlock — exported
//     for tests; the B200 kernels use the chunk/anchor program below instead;
//   * the CHUNK/ANCHOR program (this build's generalisation of Alg. 3,
//     PAPER.md:145-175, with per-thread chunks of K consecutive internal positions
//     as the "blocks", serial in-chunk composition instead of in-block doubling,
//     and pointer jumping (Alg. 2) over the chunks' anchor joints instead of the
//     serial MaxParentOutBlock walk).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace hs {

enum : int32_t { SRC_ROOT = -1, SRC_PREV = -2, SRC_NONE = -3, SRC_RUN = -4 };
enum : int { CHUNK_CONSECUTIVE = 0, CHUNK_HEAVY = 1, CHUNK_RUNS = 2 };

// Chunk decomposition of a flat forest given in topological order (par[f] < f):
// per-thread lists of at most K nodes; a node's parent is either the previous node
// of its list (PREV), absent (ROOT), or an ANCHOR elsewhere.
//   CHUNK_CONSECUTIVE  lists = runs of K consecutive positions (the paper's index
//                      blocks, at thread granularity)
//   CHUNK_HEAVY        lists = heavy-path pieces (<= K joints) packed first-fit
//                      decreasing, then ordered for conflict-free smem access
//   CHUNK_RUNS         heavy paths longer than K on consecutive lanes (RUNS, joined
//                      by a warp-shuffle segmented scan: src SRC_RUN on a lane's first
//                      joint), the other paths packed as in CHUNK_HEAVY
struct ChunkDecomp {
    int K = 0;
    std::vector<std::vector<int32_t>> lists;
    std::vector<int32_t> run_back; // per list (lane): preceding lanes of its run in the warp
    std::vector<int32_t> src;      // per node: SRC_ROOT, SRC_PREV, SRC_RUN, or anchor node (>= 0)
    std::vector<int32_t> slot_of;  // per node: anchor slot or -1
    std::vector<int32_t> slots;    // slot -> node (ascending node index => topological)
    std::vector<int32_t> link0;    // slot -> slot of anchor(seghead(node)), or -1
    std::vector<int32_t> head;     // per node: first joint of its segment (through PREV / RUN)
};
ChunkDecomp decompose(const std::vector<int32_t>& par, int K, int mode,
                      const std::vector<int32_t>* smem_pos, bool pad_to_warp);

// Persistent-tile program for the single-CTA chunked kernel.
struct TileProgram {
    int K = 0, C = 0, F = 0, T = 0;     // chunk, chars per tile, joints per tile, compute threads
    int nslots = 0, R2 = 0;             // anchor slots per tile, pointer-jumping rounds
    bool pingpong = true;               // P double-buffered (else: 2 barriers per round)
    int max_round_entries = 0;          // largest round (single buffer needs <= 4 per thread)
    int lists_nonempty = 0;             // chunks with work per character (T may include padding)
    std::vector<uint64_t> meta;         // [T][K]: off | ibu<<16 | (u16)src<<32 | (u16)own<<48
    std::vector<int32_t> p1len;         // [T]: phase-1 length (bits 0..7) | run_back << 8 |
                                        //      (run anchor P location + 1) << 16
    bool has_runs = false;              // some lanes are joined by the warp-shuffle scan
    std::vector<int32_t> round_off;     // [R2 + 1] offsets into rounds
    std::vector<uint32_t> rounds;       // slot | dst buf<<14 | self buf<<15 | link location<<16
};

// Multi-CTA (split) program: the same decomposition over ONE character with
// unbounded size; slots index a global workspace [n_chars][nslots][12].
struct SplitProgram {
    int K = 0, nchunks = 0, nslots = 0;
    std::vector<int32_t> meta;          // [nchunks][K][4]: off(user j), src, own, pad
    std::vector<int32_t> anchor_parents;// [nslots]: link0 (the anchor skeleton, topological)
};

// Multi-tile program for skeletons beyond one CTA: the internal
// (topological) order is cut into tiles of <= F consecutive positions; a CTA walks a
// character's tiles in order, so every cross-tile parent is FINAL when its child's
// tile runs (Alg. 3's cross-block carry, with the carry resolved
// before the block instead of walked after it).  Per tile: the chunk/anchor program
// of the tile's sub-forest, where a joint whose parent lies in an earlier tile reads
// that parent's global pose from an imported slot Q (a final root of the anchor
// forest); joints with a child in a later tile export their global pose to a
// per-CTA workspace slot in phase 3.
constexpr int kSeqInboxPiecesPerThread = 9;    // = kernels.cuh kSeqInboxPieces
constexpr int kSeqInboxLatePerThread = 4;      // = kernels.cuh kSeqInboxLate
struct SeqTile {
    int32_t n_early, nj;          // inbox rows from tiles <= k - 3 (a prefix); joints [k F, k F + nj)
    int32_t R2, n_entries;        // pointer-jumping rounds and phase-2 descriptors
    int32_t rounds_off;           // offset into rounds; round_off rows are per tile
    int32_t n_imp, imp_off;       // inbox: workspace rows [imp_off, imp_off + n_imp) -> Q 0..n_imp
    int32_t n_runs, runs_off;     // TMA runs: (user start, smem offset, length)
    int32_t T;                    // compute threads with work
    int32_t n_exl, exl_off;       // export list: pairs [exl_off, exl_off + n_exl) of exl
};
struct SeqProgram {
    int K = 0, F = 0, T = 0, KT = 0;   // chunk, joints per tile (max), threads (max), tiles
    int S = 0;                          // anchor slots per buffer (uniform over tiles)
    int nQ = 0;                         // Q slots per buffer (max imports of a tile); tile k's Q
                                        // buffer is 2S + (k & 1) nQ .. + nQ
    int R2max = 0, max_entries = 0, max_imp = 0, max_runs = 0;
    int max_exl = 0;                    // largest export list of a tile (pairs, padded to 2)
    int n_exp = 0;                      // workspace rows per CTA: all tiles' inboxes
    bool has_runs = false;
    std::vector<SeqTile> tiles;
    std::vector<uint64_t> meta;         // [KT][T][K]: off 10 | src + 8 13 | own + 1 13 | ws slot + 1 16 | fwd + 1 12
    std::vector<int32_t> p1len;         // [KT][T] as TileProgram::p1len
    // per-tile records are 16-byte aligned and sized (the producer warp loads them by TMA)
    std::vector<int32_t> round_off;     // [KT][R2max + 1 rounded up to 4], relative to rounds_off
    std::vector<uint32_t> rounds;       // per tile, padded to 4: phase-2 descriptors (TileProgram encoding)
    std::vector<int32_t> exl;           // export lists: (smem offset in the tile, workspace row)
                                        // pairs, each tile's list padded to 2 pairs (TMA)
    std::vector<int32_t> runs;          // [..][4]: user start, smem offset, length, 0
    std::vector<int32_t> ib_user;       // [KT][F]: user label at each smem offset (-1 = none)
};
struct Plan {
    int32_t n = 0;
    std::vector<int32_t> parents;       // user labels
    std::vector<int32_t> level;         // user labels, root = 1
    int32_t L = 0, R = 0;
    bool identity = true;
    std::vector<int32_t> order;         // internal -> user
    std::vector<int32_t> rank;          // user -> internal
    std::vector<int32_t> ipar;          // internal parents
    std::vector<int32_t> lift;          // [R][n] user labels (Eq. 2 powers of two)
    std::vector<int32_t> leaves;        // user labels of leaves (KIYA kernel)
};

// Returns 0 (HS_OK) or an hs_status code; err gets a message.
int build_plan(const int32_t* parents, int32_t n, Plan& out, std::string& err);

TileProgram build_tile_program(const Plan& p, int K, int C, bool pingpong, int mode);
SplitProgram build_split_program(const Plan& p, int K);
// Returns false when a tile does not fit (more than max_threads compute threads or a
// field overflows its 16-bit encoding): the caller retries with a smaller F.
bool build_seq_program(const Plan& p, int K, int F, int mode, int max_threads, SeqProgram& out);
int64_t seq_smem_bytes(const SeqProgram& sp, int stages, int sbufs);
int64_t seq_max_tile_entries(const SeqProgram& sp);   // phase-2 descriptors of the largest tile
int64_t seq_prog_words(const SeqProgram& sp);         // 4-byte words of one program buffer

// The paper's block layout for block size B over INTERNAL positions (exports).
void block_layout(const Plan& p, int B, std::vector<int32_t>& block_of, std::vector<int32_t>& mpob);

// Tables of the literal Alg. 3 comparison kernel, in USER labels:
// lb[r][u] = 2^r-th ancestor of u along in-block parents (stage A, clamped to u's
// block: DESIGN.md reading R8), mpob[u] = MaxParentOutBlock(u) (stage B walk,
// reading R9); RB = ceil(log2 B) stage-A rounds.
void blocked_tables(const Plan& p, int B, std::vector<int32_t>& lb, std::vector<int32_t>& mpob, int& RB);

// Tables of the literal Alg. 4 comparison kernel, in USER labels:
// lp[u] = in-block parent (stage A hops, clamped: R8), l8[u] = in-block 8th ancestor
// (stage B's MultiParent(., 8)), -1 when the hop leaves u's B-block.
void compressed_tables(const Plan& p, int B, std::vector<int32_t>& lp, std::vector<int32_t>& l8);

// Shared-memory bytes of the chunked kernel for a tile program and stage counts
// (tiles, skin buffers, anchor buffers, and the phase-2 tables staged in smem).
int64_t tile_smem_bytes(const TileProgram& tp, int stages, int sbufs);

}  // namespace hs
