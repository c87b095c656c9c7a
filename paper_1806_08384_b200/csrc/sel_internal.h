// sel_internal.h — libsel internals shared by the host planner (canon.cpp, host.h units) and the
// sm_100a kernels (kernels.cu). Not part of the ABI (include/sel.h is).
//
// A validated predicate program (include/sel.h format) is canonicalised on the host into
//   * leaves: one column compared against a UNION OF CLOSED INTERVALS in that column's
//     order-preserving unsigned "key space" (every =,<,>,<=,>=,BETWEEN,IN leaf and every NOT of
//     one is exactly such a set, see canon.cpp), and
//   * postfix AND/OR over leaf masks (NOT is pushed into the leaves by complementing their
//     interval sets, which is exact in key space including NaN keys for FLOAT32).
// The device evaluates a leaf as   ((key(v) - lo) mod 2^w) <= span   per interval, where the
// host pre-biases `lo` so that key() is the identity for every type but FLOAT32 (signed ints:
// key(v) = v ^ signbit, so key(v) - lo == v - (lo ^ signbit) mod 2^w).
#pragma once
#include <stdint.h>

namespace sel {

constexpr int kWarpsPerCta = 8;              // 256 threads
constexpr int kThreads = kWarpsPerCta * 32;
constexpr int kRowsPerThread = 32;           // one 32-bit row mask per thread per chunk
constexpr int kChunkRows = 32 * kRowsPerThread;        // 1024 rows per warp-chunk
// Push-down: one warp tile = one 1024-row chunk. Dynamic shared memory per warp holds the
// compacted chunk-local row indices (u16 x 1024) and captures of projected predicate columns.
constexpr uint32_t kIdxBytes = 2 * kChunkRows;
constexpr uint32_t kCaptureBudget = 8 * kChunkRows;     // <= 8 bytes/row of captured columns
constexpr uint32_t kMaxPushdownSmem = kWarpsPerCta * (kIdxBytes + kCaptureBudget);  // 80 KB
constexpr uint16_t kNoCapture = 0xFFFF;
constexpr uint16_t kKeptBase = 0xFF00;  // push-down from a selection: proj_cap_off = kKeptBase + slot
// proj_cap_off = kConstProj: every selected row has the same value in this column (the
// conjunction pins it with a single-value leaf), raw bits in (uintptr_t)proj_src: a fill.
constexpr uint16_t kConstProj = 0xFFFE;
// proj_cap_off = kCodedProj (push-down from a selection): the conjunction pins the column to two
// values (an IN of two points on a 1- or 4-byte column) and the keeping count recorded, per row,
// which one matched (SelectionBufs::which); the staged row numbers carry that bit (kCodeBit) and
// the value is (uintptr_t)proj_src >> (w * bit), w = 8 or 32 — the column is never read by the
// push-down.
constexpr uint16_t kCodedProj = 0xFFFD;
constexpr uint16_t kCodeBit = 1u << 12;          // staged block-relative rows are < 4096
constexpr int kMaxDeviceStack = 32;

enum WidthClass : uint8_t { W1 = 0, W2 = 1, W4 = 2, W8 = 3 };
enum DevOpcode : uint8_t { DOP_LEAF = 0, DOP_AND = 1, DOP_OR = 2 };
enum Path : int { PATH_INTERP = 0, PATH_CONJ = 1, PATH_CONST = 2 };
// Leaf kinds of the count kernel's conjunctive fast path (width in bytes, key-space test):
//   FK_E4  4-byte column, one point           v == lo
//   FK_R4  4-byte column, one interval        v - lo <= span
//   FK_S4  4-byte column, 2..4 intervals      OR of the above
//   FK_R8  8-byte column, one interval        v - lo <= span (64-bit)
//   FK_S1  1-byte column, 1..4 points         SWAR byte compare, 4 rows per instruction group
enum FastKind : uint8_t { FK_E4 = 0, FK_R4 = 1, FK_S4 = 2, FK_R8 = 3, FK_S1 = 4 };
constexpr int kMaxFastLeaves = 4;

struct DevLeaf {
  uint8_t slot;      // index into DevProgram::col
  uint8_t wclass;    // WidthClass of the column
  uint8_t fkey;      // 1: FLOAT32 — apply the sortable-key transform before the interval test
  uint8_t cap;       // push-down: 1 = store the loaded raw values to shared memory at cap_off
  uint16_t iv_begin; // first interval in lo[]/span[]
  uint16_t iv_count; // >= 1
  uint16_t cap_off;  // byte offset of the capture within the warp's shared-memory area
  uint16_t pad;      // kLeafBitmap | kLeafNegate: an IN_BITMAP leaf (lo[iv_begin] = words,
                     // span[iv_begin] = nbits | smem offset << 32; test: v < nbits && bit v, raw v)
};
constexpr uint16_t kLeafBitmap = 1, kLeafNegate = 2, kLeafStaged = 4;  // staged: in shared memory

// Kernel parameter block (passed by value as a __grid_constant__; no H2D copy per probe).
template <int MAXOPS, int MAXLEAVES, int MAXIV, int MAXSLOTS, int MAXPROJ>
struct DevProgramT {
  static constexpr int kMaxOps = MAXOPS, kMaxLeaves = MAXLEAVES, kMaxIv = MAXIV,
                       kMaxSlots = MAXSLOTS, kMaxProj = MAXPROJ;
  uint32_t n_ops;        // postfix length; 0 means "always true"
  uint32_t n_leaves;
  uint32_t conj;         // 1: ops are leaf0 AND leaf1 AND ... (no stack needed)
  uint32_t n_proj;
  uint32_t warp_smem;    // push-down: dynamic shared memory bytes per warp
  uint32_t prefetch;     // 1: L2 bulk-prefetch each warp's next chunk (SEL_PREFETCH=0 disables)
  uint32_t chunk_stride; // count kernel: scan chunks phase, phase + stride, ... (1: all)
  uint32_t chunk_phase;
  uint32_t gate;         // push-down from a selection: 1 = write nothing if the global count
                         // (Scratch::result[kGateSlot]) exceeds gate_max (Algorithm 1's throw)
  uint32_t bm_bytes;     // IN_BITMAP key sets: total bytes (16-byte aligned each)
  uint32_t bm_smem;      // count kernel: bytes of the sets staged in shared memory (leaves with
                         // kLeafStaged; offset = span[iv_begin] >> 32), 0 = none
  uint32_t n_direct;     // push-down from a selection: projections that are kept or constant
  uint32_t coded;        // push-down from a selection: a projection is kCodedProj
  uint32_t dense_split;  // push-down from a selection: fully selected chunks are left to
                         // dense_chunks_kernel (whole-chunk copies)
  uint32_t global_out;   // push-down from a selection: the outputs are the GLOBAL result
                         // (sel_execute_to): positions start at Scratch::result[kOffsetSlot]
  // Count kernel fast path (template-specialised conjunctive forms): when
  // fast_n > 0 the program is leaf 0 AND ... AND leaf fast_n-1 and leaf s has kind fast_kind[s]
  // (FastKind); the kernel instantiated for fast_n evaluates it as straight-line code with the
  // leaf parameters hoisted out of the chunk loop. FK_S1 compares against fast_pts[s][0..npts)
  // (the point keys, each byte-replicated).
  uint32_t fast_n;
  int32_t fast_code;     // keeping count: slot whose point-1 matches are kept as `which`, or -1
  uint8_t fast_kind[4];
  uint8_t fast_npts[4];
  uint32_t fast_pts[4][4];
  uint64_t row_offset;   // global id of local row 0 (push-down ids)
  uint64_t capacity;     // push-down capacity in rows
  uint64_t gate_max;
  uint8_t op[MAXOPS];
  uint8_t arg[MAXOPS];   // leaf index for DOP_LEAF
  DevLeaf leaf[MAXLEAVES];
  const void* col[MAXSLOTS];
  uint64_t lo[MAXIV];
  uint64_t span[MAXIV];
  const void* proj_src[MAXPROJ];
  void* proj_dst[MAXPROJ];
  uint16_t proj_cap_off[MAXPROJ];  // kNoCapture: gather from proj_src; else smem capture offset
  uint8_t proj_wclass[MAXPROJ];
};

// Small block for the common case (≤ 32 leaves/64 ops/64 intervals/16 projections, ~2.6 KB);
// large block for anything the validator admits (128 instructions, 512 constants, 255 projections).
using DevProgramSmall = DevProgramT<64, 32, 64, 32, 16>;
using DevProgramLarge = DevProgramT<256, 128, 1024, 128, 256>;

// Batch of programs over one scan (sel_count_batch): distinct leaves of all
// programs grouped by column (each column loaded once per chunk, each leaf evaluated once into a
// shared-memory leaf-mask table), then each program's postfix over leaf masks, DOP_EMIT(k) ending
// program k.
constexpr int kBatchMaxLeaves = 32, kBatchMaxProgs = 32, kBatchMaxCols = 32;
constexpr uint8_t DOP_EMIT = 3;
struct BatchColumn {
  const void* data;
  uint8_t wclass, fkey;
  uint16_t leaf_begin, leaf_count;  // its leaves are [leaf_begin, leaf_begin + leaf_count)
  uint8_t swar;                     // 1-byte column whose every leaf is 1..4 points (leaf_pts)
  uint8_t pad;
};
struct BatchProgram {
  uint32_t n_cols, n_leaves, n_ops, n_progs;
  // every program a conjunction of leaves (or TRUE/FALSE): program k counts the rows in all
  // leaves of conj_set[k] (bit l = leaf l; 0 = TRUE) when bit k of prog_live is set — no postfix
  // walk, no stack
  uint32_t all_conj, prog_live;
  uint32_t conj_set[kBatchMaxProgs];
  BatchColumn col[kBatchMaxCols];
  uint16_t leaf_iv_begin[kBatchMaxLeaves];
  uint16_t leaf_iv_count[kBatchMaxLeaves];
  // a leaf on a 1-byte column whose intervals are 1..4 single points: their count; 0 otherwise
  uint8_t leaf_pts[kBatchMaxLeaves];
  uint8_t op[512];
  uint8_t arg[512];
  uint64_t lo[1024];
  uint64_t span[1024];
};
int launch_count_batch(const BatchProgram& p, uint64_t n, int grid, uint64_t* out_counts,
                       void* stream);
int occupancy_count_batch();

// A kept selection (sel_count_ex with SEL_KEEP_SELECTION): per chunk of 1024 rows, 32 row-major
// mask words (word L, bit b = row 32L + b of the chunk) and the chunk's count; per superblock of
// 64 chunks the sum of its chunk counts (atomics during the count); per hyperblock of 4096
// chunks the exclusive prefix of those sums, which the count's last CTA forms (<= 1024
// hyperblocks for 2^32 rows). A push-down block's output position is the hyperblock prefix + the
// superblock sums before it within its hyperblock + the chunk counts before it within its
// superblock (two loads per lane each). No memset, no scan kernel per probe: the superblock sums
// alternate between two halves by the parity of the device's keeping-count epoch (state[0]), and
// a count zeroes the other half (the previous, now dead, selection's) while it runs.
// Push-down from a selection: chunks per warp block. 4 on large shards (A/B 2/4/8: C5 push-down
// 0.233 -> 0.206 ms, C3 0.240 -> 0.232, C2 equal, 8 slower); fewer below kSmallBlockRows local
// rows, where a 4-chunk grid runs too few rounds to balance (step A/B: 75M rows 0.2261 -> 0.2220
// ms with 2, 150M equal, 300M 0.7556 -> 0.7681 with 2; then 1 against 2: 75M async step 0.2159
// -> 0.2125 ms, 37.5M equal).
constexpr int kSelBlockChunks = 4;
#ifndef SEL_SMALL_BLOCK_ROWS
#define SEL_SMALL_BLOCK_ROWS (150ull << 20)
#endif
constexpr uint64_t kSmallBlockRows = SEL_SMALL_BLOCK_ROWS;
#ifndef SEL_SMALL_BC
#define SEL_SMALL_BC 1   // chunks per block below kSmallBlockRows (1 or 2)
#endif
inline int pushdown_block_chunks(uint64_t local_rows) {
  return local_rows < kSmallBlockRows ? SEL_SMALL_BC : kSelBlockChunks;
}
constexpr int kSbShift = 6;
constexpr uint64_t kSbChunks = 1ull << kSbShift;
constexpr int kHbShift = 12;                          // chunks per hyperblock: 4096
constexpr uint64_t kHbChunks = 1ull << kHbShift;
constexpr int kMaxKeep = 8;
struct SelectionBufs {
  uint32_t* bits;        // [nchunks * 32]
  uint32_t* which;       // [nchunks * 32] row-major: row matched point 1 of the coded leaf
  int32_t code_col;      // table column coded by `which` (host bookkeeping), -1 = none
  uint64_t code_pts;     // its two raw values: 1-byte column point 0 | point 1 << 8; 4-byte
                         // column point 0 | point 1 << 32
  uint16_t* chunk_cnt;   // [nchunks]
  uint32_t* sb_sum;      // two halves of sb_stride words (a multiple of 4), zero beyond nsb; the
                         // selection's half is (state[0] - 1) & 1
  uint32_t sb_stride;
  uint32_t* hb_prefix;   // [nhb + 2]: exclusive prefix, [nhb] the local count, [nhb + 1] the flag
                         // (a fully selected chunk was kept: dense_chunks_kernel has work)
  uint32_t* state;       // [4]: [0] keeping counts so far, [1 + h] words of half h to zero,
                         // [3] the full-chunk flag while a count runs
  // Kept values of projected predicate columns: chunk c's selected values, compacted in row
  // order, at keep_slot[k] + c * 1024 * width (written by the count, copied by the push-down).
  uint32_t n_keep;
  uint32_t warp_smem;            // count kernel: dynamic shared memory per warp (0 without keep)
  uint8_t keep_col[kMaxKeep];    // table column index (host bookkeeping)
  uint8_t keep_wclass[kMaxKeep];
  uint16_t keep_cap_off[kMaxKeep];
  void* keep_slot[kMaxKeep];
};

// Result slots: [0] local count, [1 .. kMaxRanks] gathered per-rank counts / batch counts,
// [kGateSlot] the global count sel_execute's device-side gate reads.
constexpr int kMaxRanks = 1024;
constexpr int kGateSlot = 1 + kMaxRanks;
constexpr int kOffsetSlot = 2 + kMaxRanks;   // this rank's global output offset (sel_execute_to)
constexpr int kResultSlots = 3 + kMaxRanks;
// One word past the result slots: the device-gated Execute's sequence number. finish_execute
// bumps result[kSeqSlot] and stores it to the pinned mirror after the mirror's other words
// (fence at system scope in between), so that a host spinning on it (sel_prepared_execute_async)
// knows the count is final without waiting for the materialisation.
constexpr int kSeqSlot = kResultSlots;
constexpr int kResultAlloc = kResultSlots + 1;
constexpr int kMirrorMax = 512;  // read-back mirror below kGateSlot (ExecFinish)

// The library's own exchange over peer memory (sel_ctx_set_peers; SURVEY §8e "a one-shot peer
// write of each rank's count into a symmetric buffer over NVLink plus a flag"). Every rank owns a
// symmetric buffer `mine` of 2 x kMaxPeers x kMaxXchgVals u64 (two halves by exchange parity)
// that every peer maps (CUDA IPC). An exchange of k values: the rank bumps its device epoch e,
// stores (e << 32 | value) for each value into half e&1, row `rank`, of EVERY rank's buffer
// (P2P stores over NVLink, release at system scope), then waits until all n rows of its own
// half e&1 carry epoch e (acquire loads). Values are < 2^32 (per-rank counts). A rank can run at
// most one exchange ahead of another (it cannot finish e+1 before every rank has written e+1,
// which each does only after finishing e), so the parity halves never mix two exchanges. A wait
// that exceeds timeout_ns (10 s unless sel_ctx_set_peer_timeout) sets *err (host-mapped) and gives
// up instead of hanging: every gathered value and sum of that exchange becomes kXchgFailed, so the
// gated push-down kernels that follow write nothing (a global count of kXchgFailed exceeds every
// maxSize and they also test for it), and the host fails the call and every later probe of the
// context (SEL_E_STATE) until the peers are dropped and set again.
constexpr uint64_t kXchgFailed = ~0ull;
constexpr int kMaxPeers = 32;
constexpr int kMaxXchgVals = 32;
struct PeerXchg {
  uint64_t* const* peers;  // device array [n]: rank r's buffer as mapped here (peers[rank] = mine)
  uint64_t* mine;
  uint32_t* epoch;         // device counter, bumped once per exchange
  uint32_t* err;           // host-mapped flag: nonzero after a timed-out wait
  int n, rank;
  uint64_t timeout_ns;     // a wait longer than this is a failed exchange
};

// The result words of a device-gated Execute (sel_execute), finished by ONE CTA right after the
// count: with peers the exchange of the local count in result[kGateSlot] (gathered into
// result[1..n], their sum into result[kGateSlot]); with gate_ranks > 0 (NCCL: result[1..gate_ranks]
// all-gathered before) their sum into result[kGateSlot]; the words the host reads back mirrored
// right below result[kGateSlot] (the gathered counts at [kGateSlot - nr, kGateSlot), or the local
// count at kGateSlot - 1) and this rank's offset in the rank-ordered result at
// result[kOffsetSlot]; with `host` (the context's pinned mirror, device-accessible) the mirror and
// the gate stored there as well, so that no copy follows. result == nullptr: nothing to finish
// (a count with host != nullptr stores its count, after the exchange, to host[0]).
struct ExecFinish {
  uint64_t* result;
  uint64_t* host;
  int gate_ranks;
  int rank;
};

// Device-side scratch owned by a context.
struct Scratch {
  uint64_t* partials;      // per-CTA partial counts (count kernel)
  unsigned int* done;      // CTA completion counter, self-resetting
  uint64_t* result;        // [0] = count of the last probe, [1..] = gathered per-rank counts
  unsigned long long* ticket;  // monotone tile ticket counter (push-down)
  uint64_t* status;        // push-down tile status words (epoch | flag | value)
  uint64_t status_cap;     // entries in status
  PeerXchg xg;             // count kernel: n > 0 = its last CTA exchanges the count over peer
                           // memory and leaves the global sum in *result (sel_count with peers)
};

// Gather k (<= kMaxXchgVals) values src[0..k) of every rank: out[r * k + j] = rank r's src[j]
// (out may be null); sums[j] = sum over ranks (sums may be null). One CTA, on `stream`.
int launch_peer_exchange(const PeerXchg& x, const uint64_t* src, int k, uint64_t* out,
                         uint64_t* sums, void* stream);

// Equi-depth histogram of a block sample (sel_histogram): sample keys -> radix sort -> bucket
// statistics, all on `stream`; histogram_temp_bytes sizes the sort's scratch for m keys.
int launch_histogram(const void* col, int wclass, uint32_t flip, uint64_t n, uint64_t stride,
                     uint64_t phase, uint64_t nsamp, uint64_t m, uint32_t nb, uint32_t* keys,
                     uint32_t* sorted, void* temp, size_t temp_bytes, uint32_t* lo, uint32_t* hi,
                     uint64_t* rows, uint64_t* distinct, void* stream);
size_t histogram_temp_bytes(uint64_t m);

// *p = v on `stream` (one thread; sel_count_async's constant and empty cases).
int launch_set_u64(uint64_t* p, uint64_t v, void* stream);

// Launch entry points (kernels.cu). Return cudaError_t as int.
// keep != nullptr: also keep the selection (and, with keep->n_keep > 0, the selected values of
// projected predicate columns; the leaves carry the capture offsets and keep->warp_smem is set).
// nw: warps per CTA, kWarpsPerCta or 32 (one 1024-thread CTA per SM when staged key sets fill
// the shared memory; keep->warp_smem must then be 0).
// fin (keeping counts of a device-gated Execute): the count's last CTA also finishes the
// Execute's result words (ExecFinish; with s.xg.n > 0 through the peer exchange) — no kernel, no
// copy between the count and the gated materialisation.
int launch_count_small(const DevProgramSmall& p, uint64_t n, int grid, const Scratch& s,
                       const SelectionBufs* keep, void* stream, int nw = kWarpsPerCta,
                       const ExecFinish* fin = nullptr);
int launch_count_large(const DevProgramLarge& p, uint64_t n, int grid, const Scratch& s,
                       const SelectionBufs* keep, void* stream, int nw = kWarpsPerCta,
                       const ExecFinish* fin = nullptr);
// Push-down from a kept selection (the count left the superblock prefix): unless `finished` (the
// count finished the Execute's result words, fin above), a 1-CTA kernel first writes the kept
// local count to s.result[0] and finishes the result words (ExecFinish with gate_ranks, rank,
// host; xg != nullptr: through the peer exchange); then the compaction/gather kernel and, with
// p.dense_split, the whole-chunk copy kernel.
// block_chunks: chunks per warp block of the compaction kernel, 1, 2 or 4 (pushdown_block_chunks).
int launch_pushdown_sel_small(const DevProgramSmall& p, uint64_t n, uint32_t* out_ids, int grid,
                              const Scratch& s, const SelectionBufs& sb, void* stream,
                              int gate_ranks = 0, const PeerXchg* xg = nullptr, int rank = 0,
                              bool finished = false, uint64_t* host = nullptr,
                              int block_chunks = kSelBlockChunks);
int launch_pushdown_sel_large(const DevProgramLarge& p, uint64_t n, uint32_t* out_ids, int grid,
                              const Scratch& s, const SelectionBufs& sb, void* stream,
                              int gate_ranks = 0, const PeerXchg* xg = nullptr, int rank = 0,
                              bool finished = false, uint64_t* host = nullptr,
                              int block_chunks = kSelBlockChunks);
int launch_pushdown_small(const DevProgramSmall& p, uint64_t n, uint32_t* out_ids, int grid,
                          const Scratch& s, uint64_t ticket_base, uint32_t epoch, void* stream);
int launch_pushdown_large(const DevProgramLarge& p, uint64_t n, uint32_t* out_ids, int grid,
                          const Scratch& s, uint64_t ticket_base, uint32_t epoch, void* stream);
// One-time kernel attributes (dynamic shared memory limit of the push-down kernels).
int prepare_kernels();
// Occupancy (CTAs per SM) of each kernel, for persistent-grid sizing.
int occupancy_count_small();
int occupancy_count_large();
int occupancy_count_keep_small(size_t dyn_smem);
int occupancy_count_fast(int fast_n, bool keep, size_t dyn_smem);  // fast path (small block)
int occupancy_count_keep_large(size_t dyn_smem);
int occupancy_count_dyn_small(size_t dyn_smem);   // plain count with staged key sets
int occupancy_count_dyn_large(size_t dyn_smem);
constexpr uint32_t kMaxCountSmem = 200 * 1024;    // dynamic shared memory cap of the count kernel
int occupancy_pushdown_small(size_t dyn_smem);
int occupancy_pushdown_sel_small();
int occupancy_pushdown_sel_large();
int occupancy_pushdown_large(size_t dyn_smem);

}  // namespace sel
