// sel_internal.h — libsel internals shared by the host planner (canon.cpp, api.cpp) and the
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
constexpr int kPdChunks = 2;                            // push-down: chunks per warp tile
constexpr int kPdTileRows = kPdChunks * kChunkRows;     // 2048 rows per push-down warp tile
constexpr int kMaxDeviceStack = 32;

enum WidthClass : uint8_t { W1 = 0, W2 = 1, W4 = 2, W8 = 3 };
enum DevOpcode : uint8_t { DOP_LEAF = 0, DOP_AND = 1, DOP_OR = 2 };
enum Path : int { PATH_INTERP = 0, PATH_CONJ = 1, PATH_CONST = 2 };

struct DevLeaf {
  uint8_t slot;      // index into DevProgram::col
  uint8_t wclass;    // WidthClass of the column
  uint8_t fkey;      // 1: FLOAT32 — apply the sortable-key transform before the interval test
  uint8_t pad;
  uint16_t iv_begin; // first interval in lo[]/span[]
  uint16_t iv_count; // >= 1
};

// Kernel parameter block (passed by value as a __grid_constant__; no H2D copy per probe).
template <int MAXOPS, int MAXLEAVES, int MAXIV, int MAXSLOTS, int MAXPROJ>
struct DevProgramT {
  static constexpr int kMaxOps = MAXOPS, kMaxLeaves = MAXLEAVES, kMaxIv = MAXIV,
                       kMaxSlots = MAXSLOTS, kMaxProj = MAXPROJ;
  uint32_t n_ops;        // postfix length; 0 means "always true"
  uint32_t n_leaves;
  uint32_t conj;         // 1: ops are leaf0 AND leaf1 AND ... (no stack needed)
  uint32_t n_proj;
  uint64_t row_offset;   // global id of local row 0 (push-down ids)
  uint64_t capacity;     // push-down capacity in rows
  uint8_t op[MAXOPS];
  uint8_t arg[MAXOPS];   // leaf index for DOP_LEAF
  DevLeaf leaf[MAXLEAVES];
  const void* col[MAXSLOTS];
  uint64_t lo[MAXIV];
  uint64_t span[MAXIV];
  const void* proj_src[MAXPROJ];
  void* proj_dst[MAXPROJ];
  uint8_t proj_wclass[MAXPROJ];
};

// Small block for the common case (≤ 32 leaves/64 ops/64 intervals/16 projections, ~2.6 KB);
// large block for anything the validator admits (128 instructions, 512 constants, 255 projections).
using DevProgramSmall = DevProgramT<64, 32, 64, 32, 16>;
using DevProgramLarge = DevProgramT<256, 128, 1024, 128, 256>;

// Device-side scratch owned by a context.
struct Scratch {
  uint64_t* partials;      // per-CTA partial counts (count kernel)
  unsigned int* done;      // CTA completion counter, self-resetting
  uint64_t* result;        // [0] = count of the last probe, [1..] = gathered per-rank counts
  unsigned long long* ticket;  // monotone tile ticket counter (push-down)
  uint64_t* status;        // push-down tile status words (epoch | flag | value)
  uint64_t status_cap;     // entries in status
};

// Launch entry points (kernels.cu). Return cudaError_t as int.
int launch_count_small(const DevProgramSmall& p, uint64_t n, int grid, const Scratch& s,
                       void* stream);
int launch_count_large(const DevProgramLarge& p, uint64_t n, int grid, const Scratch& s,
                       void* stream);
int launch_pushdown_small(const DevProgramSmall& p, uint64_t n, uint32_t* out_ids, int grid,
                          const Scratch& s, uint64_t ticket_base, uint32_t epoch, void* stream);
int launch_pushdown_large(const DevProgramLarge& p, uint64_t n, uint32_t* out_ids, int grid,
                          const Scratch& s, uint64_t ticket_base, uint32_t epoch, void* stream);
// Occupancy (CTAs per SM) of each kernel, for persistent-grid sizing.
int occupancy_count_small();
int occupancy_count_large();
int occupancy_pushdown_small();
int occupancy_pushdown_large();

}  // namespace sel
