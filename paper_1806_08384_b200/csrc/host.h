// host.h — internals shared by the host-side units of libsel (not part of the ABI; include/sel.h
// is): error state, the dlopen'd NCCL, the context / table / prepared-execute objects, and the
// planning, memory and enqueue helpers each unit uses.
//   context.cpp   contexts, communicators, the peer exchange's buffers, tables, key sets
//   plan.cpp      program -> canonical plan -> kernel parameter block (and the host-only ABI)
//   probe.cpp     count / push-down / Execute enqueue and their ABI entry points
//   synopsis.cpp  batch and sampled counts, histograms, the synopsis estimators
//   graph.cpp     prepared executes (CUDA graphs)
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "sel.h"
#include "canon.h"
#include "sel_internal.h"

namespace sel {

constexpr uint64_t kTwoPassMinRows = 3ull << 20;  // sel_pushdown: two passes from here
constexpr uint64_t kDenseSplitMinRows = 8ull << 20;  // whole-chunk copy kernel from here (§6)
constexpr int kMaxGrid = 148 * 32;
constexpr size_t kMaxBitmaps = 65536;  // ids fit the instruction's u16 `a`

// ---- thread-local error state (context.cpp) ----------------------------------------------------
extern thread_local sel_status g_status;
extern thread_local std::string g_message;
sel_status set_error(sel_status st, const std::string& msg);
void clear_error();
uint64_t fail64(sel_status st, const std::string& msg);
// sync_stream's report of a failed communicator (not a CUDA code).
constexpr cudaError_t kNcclAsyncFailed = (cudaError_t)0x7FFF0001;
std::string cuda_msg(const char* what, cudaError_t e);
// wait_result_seq's report of a stream that drained without the Execute's result words.
constexpr cudaError_t kSeqMissing = (cudaError_t)0x7FFF0002;
inline sel_status sync_code(cudaError_t e) {
  return e == kNcclAsyncFailed ? SEL_E_NCCL : e == kSeqMissing ? SEL_E_STATE : SEL_E_CUDA;
}

struct DeviceGuard {
  int prev = -1;
  bool ok = false;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// ---- NCCL via dlopen (torch's bundled libnccl.so.2 is normally already loaded) ----------------
struct NcclApi {
  bool loaded = false;
  std::string error;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;  // optional
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;                         // optional
};

NcclApi& nccl();
std::string nccl_msg(const char* what, ncclResult_t r);

inline int width_of(int type) {
  switch (type) {
    case SEL_INT64: return 8;
    case SEL_DICT8: return 1;
    case SEL_DICT16: return 2;
    default: return 4;
  }
}
inline uint8_t wclass_of(int type) {
  switch (width_of(type)) {
    case 1: return W1;
    case 2: return W2;
    case 4: return W4;
    default: return W8;
  }
}
inline bool known_type(int t) { return t >= SEL_INT32 && t <= SEL_DICT32; }

}  // namespace sel

using namespace sel;   // the objects below and every unit use the kernels' types unqualified

// ---- objects ------------------------------------------------------------------------------------
struct sel_ctx_s {
  int device = 0;
  int num_sms = 148;
  int occ_count_small = 1, occ_count_large = 1;
  int occ_small_max = 1, occ_large_max = 1;   // the occupancy calculator's (ctas_per_sm caps it)
  Scratch s{};
  uint64_t* h_result = nullptr;   // pinned mirror of Scratch::result (kResultSlots), mapped:
  uint64_t* h_result_dev = nullptr;   // its device address (kernels store the Execute's words)
  uint64_t ticket_base = 0;
  uint32_t epoch = 0;
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  bool timing = false;
  // the last sel_prepared_execute_async: its materialisation may still be running on
  // async_stream; calls on another stream wait for this event first (ordered_stream)
  cudaEvent_t async_ev = nullptr;
  cudaStream_t async_stream = nullptr;
  bool async_pending = false;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;   // count kernel
  cudaEvent_t ev2 = nullptr, ev3 = nullptr;   // push-down kernels (sel_execute times both)
  float last_ms = 0.f;
  int live_tables = 0;
  bool destroyed = false;
  // kept selection (sel_count_ex + SEL_KEEP_SELECTION)
  SelectionBufs sel{};
  uint64_t sel_cap_chunks = 0;
  sel_table kept_table = nullptr;
  std::string kept_prog;
  std::vector<int> kept_cols;        // columns with kept values (slot k holds kept_cols[k])
  void* slot_buf[kMaxKeep] = {};     // value slots, nchunks * 1024 * width bytes each
  uint64_t slot_cap[kMaxKeep] = {};  // bytes allocated per slot
  int last_pd_path = -1;
  int last_pd_flags = 0;   // SEL_PD_* of the last materialisation from a kept selection
  bool force_single = false;
  // sel_pushdown without a kept selection: two passes (keeping count -> materialise from it) at
  // >= two_pass_min_rows local rows, else the single pass (SEL_PUSHDOWN_PATH=single|two forces)
  uint64_t two_pass_min_rows = kTwoPassMinRows;
  bool fast_enabled = true;  // count fast path (SEL_FAST=0: interpreter only)
  bool code_enabled = true;  // coded projections (SEL_CODED=0: gather them)
  bool dense_split = true;   // fully selected chunks copied whole (SEL_DENSE_SPLIT=0: not)
  bool graph_comm = true;    // prepared executes with a communicator are captured (SEL_GRAPH_COMM=0: not)
  int prefetch_mode = -1;   // -1 auto, 0 off, 1 on
  bool keep_values = false;  // SEL_KEEP_VALUES=1: executes also keep projected predicate values
  float last_count_ms = 0.f, last_push_ms = 0.f;
  // IN_BITMAP key sets (sel_bitmap_register): id -> device words / nbits; words null = free id
  std::vector<const uint64_t*> bm_words;
  std::vector<uint64_t> bm_nbits;
  // generations: bumped when device buffers are reallocated / the bitmap registry changes, so
  // that prepared executes (captured CUDA graphs) re-capture instead of using stale pointers
  uint64_t alloc_gen = 0, bm_gen = 0;
  cudaStream_t cap_stream = nullptr;  // stream-capture source for prepared executes
  bool capturing = false;             // timing events become graph event-record nodes
  int count_nw = 0;                   // SEL_COUNT_NW: 8 forces 8-warp count CTAs
  // the library's own exchange over peer memory (sel_ctx_set_peers; sel_internal.h PeerXchg)
  bool comm_failed = false;          // an asynchronous NCCL error aborted the communicator
  bool peers = false;
  bool peer_failed = false;           // a peer exchange timed out: probes fail until re-set
  uint64_t peer_timeout_ns = 10000000000ull;  // sel_ctx_set_peer_timeout
  uint64_t* peer_buf = nullptr;       // this rank's symmetric buffer (exported by CUDA IPC)
  uint64_t** peer_ptrs = nullptr;     // device array of the n buffers as mapped here
  std::vector<void*> peer_opened;     // IPC mappings to close
  uint32_t* peer_epoch = nullptr;     // device exchange counter
  uint32_t* h_peer_err = nullptr;     // host-mapped timeout flag
  std::map<std::string, void*> imported;  // sel_ctx_import_buffer: IPC handle -> mapped base
  char* hist_buf = nullptr;           // sel_histogram scratch (keys, sorted keys, sort temp, stats)
  size_t hist_cap = 0;
  PeerXchg xg{};
};

struct sel_table_s {
  sel_ctx ctx;
  std::vector<sel_column> cols;
  std::vector<int> types;
  uint64_t local_rows, row_offset, global_rows;
  std::vector<sel_prepared> prepared;  // orphaned (table = nullptr) when the table is released
};

struct sel_prepared_s {
  sel_table t = nullptr;
  std::string prog;
  std::vector<uint32_t> proj;
  std::vector<void*> out_cols;
  uint32_t* out_rowids = nullptr;
  uint64_t max_size = 0, capacity = 0;
  bool graph = false;                 // false: each run is a plain sel_execute
  cudaGraphExec_t exec = nullptr;
  uint64_t alloc_gen = ~0ull, bm_gen = ~0ull;
  bool timing = false;
  ncclComm_t comm = nullptr;
  std::vector<int> kept_cols;         // the kept selection a run leaves in the context
  SelectionBufs sel{};
};

namespace sel {

// Cross-rank combination needed: a communicator (NCCL) or peers (the library's own exchange).
inline bool multi(sel_ctx c) { return c->comm != nullptr || c->peers; }
cudaError_t sync_stream(sel_ctx c, cudaStream_t s);
cudaError_t wait_result_seq(sel_ctx c, cudaStream_t s, uint64_t seq0);
// The caller's stream of a probe, ordered after an async Execute still running on another stream.
cudaStream_t ordered_stream(sel_ctx c, void* cuda_stream);
sel_status peer_status(sel_ctx c);
sel_status ensure_status(sel_ctx c, uint64_t ntiles, cudaStream_t stream);
sel_status ensure_selection(sel_ctx c, uint64_t nchunks);
sel_status ensure_slot(sel_ctx c, int k, uint64_t bytes);

// ---- planning (plan.cpp; the templates here) ----------------------------------------------------
template <class P>
bool fits_block(const Plan& plan, size_t nslots, uint32_t nproj) {
  return plan.op.size() <= (size_t)P::kMaxOps && plan.leaves.size() <= (size_t)P::kMaxLeaves &&
         plan.n_intervals <= (size_t)P::kMaxIv && nslots <= (size_t)P::kMaxSlots &&
         nproj <= (uint32_t)P::kMaxProj;
}

int fast_kinds(const Plan& plan, const int* types, uint8_t (&kind)[kMaxFastLeaves],
               uint32_t (&pts)[kMaxFastLeaves][4], uint8_t (&npts)[kMaxFastLeaves]);

template <class P>
void classify_fast(const Plan& plan, const sel_table_s* t, P* p) {
  p->fast_n = 0;
  p->fast_code = -1;
  if (!t->ctx->fast_enabled) return;
  p->fast_n = (uint32_t)fast_kinds(plan, t->types.data(), p->fast_kind, p->fast_pts, p->fast_npts);
}

// Plan -> kernel parameter block. TRUE (PATH_CONST with value true) packs as an empty conjunction.
template <class P>
void pack(const Plan& plan, const sel_table_s* t, P* p) {
  std::memset(p, 0, sizeof(P));
  std::vector<int> slot_of(t->cols.size(), -1);
  std::vector<int> bm_ids;
  std::vector<uint32_t> bm_off;
  uint32_t nslots = 0, iv = 0;
  p->n_ops = (uint32_t)plan.op.size();
  p->n_leaves = (uint32_t)plan.leaves.size();
  p->prefetch = t->ctx->prefetch_mode == 1 ? 1u : 0u;
  p->chunk_stride = 1;
  p->chunk_phase = 0;
  p->conj = plan.path != PATH_INTERP ? 1u : 0u;
  for (size_t i = 0; i < plan.op.size(); ++i) {
    p->op[i] = plan.op[i];
    p->arg[i] = plan.arg[i];
  }
  for (size_t l = 0; l < plan.leaves.size(); ++l) {
    const PlanLeaf& L = plan.leaves[l];
    if (slot_of[L.col] < 0) {
      slot_of[L.col] = (int)nslots;
      p->col[nslots++] = t->cols[L.col].data;
    }
    const int type = t->types[L.col];
    DevLeaf& d = p->leaf[l];
    d.slot = (uint8_t)slot_of[L.col];
    d.wclass = wclass_of(type);
    d.fkey = type == SEL_FLOAT32 ? 1 : 0;
    d.iv_begin = (uint16_t)iv;
    if (L.bitmap >= 0) {  // IN_BITMAP: one table entry = (words pointer, nbits | smem offset)
      d.iv_count = 1;
      d.pad = (uint16_t)(kLeafBitmap | (L.negate ? kLeafNegate : 0));
      const uint64_t nbits = t->ctx->bm_nbits[L.bitmap];
      uint32_t off = p->bm_bytes;
      for (size_t q = 0; q < bm_ids.size(); ++q)
        if (bm_ids[q] == L.bitmap) off = bm_off[q];
      if (off == p->bm_bytes) {  // first leaf on this set: lay it out (16-byte aligned)
        bm_ids.push_back(L.bitmap);
        bm_off.push_back(off);
        const uint64_t bytes = ((nbits + 127) / 128) * 16;
        p->bm_bytes = (uint32_t)std::min<uint64_t>(off + bytes, 0xFFFFFFFFull);
      }
      p->lo[iv] = (uint64_t)(uintptr_t)t->ctx->bm_words[L.bitmap];
      p->span[iv] = nbits | ((uint64_t)off << 32);
      ++iv;
      continue;
    }
    d.iv_count = (uint16_t)L.iv.size();
    const uint64_t bias = key_sign_bias(type);
    for (const Interval& x : L.iv) {
      p->lo[iv] = x.lo ^ bias;
      p->span[iv] = x.hi - x.lo;
      ++iv;
    }
  }
  classify_fast(plan, t, p);
}

// Stage key sets in the count kernel's shared memory, smallest first, while they fit beside `dyn`
// bytes of warp areas (a staged lookup costs ~conflict-degree cycles per warp; a global one an
// L1 wavefront per distinct 128-byte line). Staged sets are re-laid out contiguously.
template <class P>
void choose_bitmap_staging(P* p, size_t dyn) {
  p->bm_smem = 0;
  if (p->bm_bytes == 0) return;
  struct Set { uint64_t words; uint32_t nbits, bytes, off; };
  std::vector<Set> sets;
  for (uint32_t l = 0; l < p->n_leaves; ++l) {
    const DevLeaf& L = p->leaf[l];
    if (!(L.pad & kLeafBitmap)) continue;
    const uint64_t w = p->lo[L.iv_begin];
    bool seen = false;
    for (auto& s : sets) seen = seen || s.words == w;
    if (!seen) {
      const uint32_t nb = (uint32_t)p->span[L.iv_begin];
      sets.push_back({w, nb, (uint32_t)(((uint64_t)nb + 127) / 128 * 16), 0xFFFFFFFFu});
    }
  }
  std::sort(sets.begin(), sets.end(), [](const Set& x, const Set& y) { return x.bytes < y.bytes; });
  uint32_t used = 0;
  for (auto& s : sets) {
    if (dyn + used + s.bytes > kMaxCountSmem) break;
    s.off = used;
    used += s.bytes;
  }
  for (uint32_t l = 0; l < p->n_leaves; ++l) {
    DevLeaf& L = p->leaf[l];
    if (!(L.pad & kLeafBitmap)) continue;
    for (auto& s : sets) {
      if (s.words != p->lo[L.iv_begin] || s.off == 0xFFFFFFFFu) continue;
      L.pad |= kLeafStaged;
      p->span[L.iv_begin] = s.nbits | ((uint64_t)s.off << 32);
    }
  }
  p->bm_smem = used;
}

// Warps per count CTA: when staged key sets leave room for a single 8-warp CTA per SM, run one
// 32-warp CTA instead (4x the loads in flight; the sets are staged once per SM either way).
// Needs no per-warp areas (no kept values). SEL_COUNT_NW=8 disables it.
template <class P>
int pick_count_warps(sel_ctx c, const P& p, size_t dyn, int occ8) {
  if (!p.bm_smem || dyn != 0 || occ8 > 1 || c->count_nw == kWarpsPerCta) return kWarpsPerCta;
  return 32;
}

uint64_t plan_bitmap_bytes(sel_ctx c, const Plan& plan);
size_t count_slots(const Plan& plan);
sel_status plan_for(sel_table t, const void* prog, size_t bytes, Plan* plan);
int grid_for(sel_ctx c, uint64_t units, int occ);
std::vector<std::pair<int, uint64_t>> const_columns(sel_table t, const Plan& plan);
bool is_const_col(const std::vector<std::pair<int, uint64_t>>& cc, int col, uint64_t* raw);
std::vector<std::pair<int, uint32_t>> choose_kept(sel_table t, const Plan& plan,
                                                  const uint32_t* keep_cols, uint32_t nkeep,
                                                  uint32_t* off);

// ---- enqueue (probe.cpp) -------------------------------------------------------------------------
void record(sel_ctx c, cudaEvent_t ev, cudaStream_t s);
sel_status reserve_selection(sel_table t, uint64_t nchunks,
                             const std::vector<std::pair<int, uint32_t>>& chosen);
sel_status enqueue_count(sel_table t, const Plan& plan, uint32_t flags, const uint32_t* keep_cols,
                         uint32_t nkeep, cudaStream_t stream, uint64_t* d_out,
                         bool allreduce = true, const uint32_t* code_cols = nullptr,
                         uint32_t ncode = 0, const ExecFinish* fin = nullptr);
sel_status enqueue_pushdown_sel(sel_table t, const Plan& plan, const uint32_t* proj_cols,
                                uint32_t nproj, uint32_t* out_rowids, void* const* out_cols,
                                uint64_t capacity_rows, bool gate, uint64_t gate_max,
                                cudaStream_t stream, int gate_ranks = 0,
                                const PeerXchg* xg = nullptr, bool global_out = false,
                                bool finished = false, uint64_t* host = nullptr);
sel_status gather_counts(sel_ctx c, uint64_t local, void* cuda_stream);
sel_status enqueue_execute(sel_table t, const Plan& plan, const uint32_t* proj, uint32_t nproj,
                           uint32_t nkeep, uint64_t max_size, uint32_t* out_rowids,
                           void* const* outs, uint64_t capacity, cudaStream_t s,
                           bool global_out = false);
uint64_t execute_outputs(sel_ctx c, uint64_t max_size, uint64_t* out_local_count,
                         uint64_t* out_global_offset, int* out_materialized);
sel_status check_projection(sel_table t, const uint32_t* proj_cols, uint32_t nproj,
                            uint32_t* out_rowids, void* const* out_cols, uint64_t capacity_rows);

}  // namespace sel
