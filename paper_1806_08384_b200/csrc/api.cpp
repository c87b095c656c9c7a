// api.cpp — the C ABI of libsel (include/sel.h): contexts, table registry, probe orchestration,
// NCCL (dlopen'd) for the cross-GPU count all-reduce and push-down offset all-gather.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <map>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "sel.h"
#include "canon.h"
#include "sel_internal.h"

using namespace sel;

// ---- thread-local error state ----------------------------------------------------------------
namespace {
constexpr uint64_t kTwoPassMinRows = 3ull << 20;  // sel_pushdown: two passes from here
constexpr uint64_t kDenseSplitMinRows = 8ull << 20;  // whole-chunk copy kernel from here (§6)
thread_local sel_status g_status = SEL_OK;
thread_local std::string g_message;

sel_status set_error(sel_status st, const std::string& msg) {
  g_status = st;
  g_message = msg;
  return st;
}
void clear_error() {
  g_status = SEL_OK;
  g_message.clear();
}
uint64_t fail64(sel_status st, const std::string& msg) {
  set_error(st, msg);
  return SEL_ERR;
}
// sync_stream's report of a failed communicator (not a CUDA code).
constexpr cudaError_t kNcclAsyncFailed = (cudaError_t)0x7FFF0001;
std::string cuda_msg(const char* what, cudaError_t e) {
  if (e == kNcclAsyncFailed)
    return std::string(what) + ": NCCL asynchronous error (a rank failed; communicator aborted)";
  return std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
}
sel_status sync_code(cudaError_t e) { return e == kNcclAsyncFailed ? SEL_E_NCCL : SEL_E_CUDA; }

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

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
#ifdef SEL_NCCL_FALLBACK
    if (!h) h = dlopen(SEL_NCCL_FALLBACK, RTLD_NOW | RTLD_GLOBAL);
#endif
    if (!h) {
      a.error = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
      return a;
    }
    a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))dlsym(h, "ncclCommInitRank");
    a.AllReduce = (decltype(a.AllReduce))dlsym(h, "ncclAllReduce");
    a.AllGather = (decltype(a.AllGather))dlsym(h, "ncclAllGather");
    a.CommDestroy = (decltype(a.CommDestroy))dlsym(h, "ncclCommDestroy");
    a.GetErrorString = (decltype(a.GetErrorString))dlsym(h, "ncclGetErrorString");
    a.CommGetAsyncError = (decltype(a.CommGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
    a.CommAbort = (decltype(a.CommAbort))dlsym(h, "ncclCommAbort");
    a.loaded = a.GetUniqueId && a.CommInitRank && a.AllReduce && a.AllGather && a.CommDestroy &&
               a.GetErrorString;
    if (!a.loaded) a.error = "libnccl.so.2 lacks a required symbol";
    return a;
  }();
  return api;
}

std::string nccl_msg(const char* what, ncclResult_t r) {
  return std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "?");
}

int width_of(int type) {
  switch (type) {
    case SEL_INT64: return 8;
    case SEL_DICT8: return 1;
    case SEL_DICT16: return 2;
    default: return 4;
  }
}
uint8_t wclass_of(int type) {
  switch (width_of(type)) {
    case 1: return W1;
    case 2: return W2;
    case 4: return W4;
    default: return W8;
  }
}
bool known_type(int t) { return t >= SEL_INT32 && t <= SEL_DICT32; }

}  // namespace

// ---- objects ------------------------------------------------------------------------------------
struct sel_ctx_s {
  int device = 0;
  int num_sms = 148;
  int occ_count_small = 1, occ_count_large = 1;
  Scratch s{};
  uint64_t* h_result = nullptr;   // pinned mirror of Scratch::result (kResultSlots), mapped:
  uint64_t* h_result_dev = nullptr;   // its device address (kernels store the Execute's words)
  uint64_t ticket_base = 0;
  uint32_t epoch = 0;
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  bool timing = false;
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

namespace {

constexpr int kMaxGrid = 148 * 32;
constexpr size_t kMaxBitmaps = 65536;  // ids fit the instruction's u16 `a`

// Cross-rank combination needed: a communicator (NCCL) or peers (the library's own exchange).
bool multi(sel_ctx c) { return c->comm != nullptr || c->peers; }

// Wait for stream `s`. With a communicator, poll instead of blocking so that an asynchronous NCCL
// failure (a rank died) aborts the communicator and fails the call instead of hanging
// (SURVEY §5 failure detection; the peer exchange bounds its own waits).
cudaError_t sync_stream(sel_ctx c, cudaStream_t s) {
  if (!c->comm || !nccl().CommGetAsyncError) return cudaStreamSynchronize(s);
  for (unsigned spin = 0;; ++spin) {
    const cudaError_t q = cudaStreamQuery(s);
    if (q != cudaErrorNotReady) return q;
    ncclResult_t st = ncclSuccess;
    if (nccl().CommGetAsyncError(c->comm, &st) == ncclSuccess && st != ncclSuccess &&
        st != ncclInProgress) {
      if (nccl().CommAbort) nccl().CommAbort(c->comm);
      c->comm = nullptr;
      c->comm_failed = true;   // every later probe of this context fails (plan_for)
      return kNcclAsyncFailed;
    }
    if (spin > 64) std::this_thread::yield();
  }
}

// After a synchronisation that followed peer exchanges: a timed-out wait (a rank missing) is an
// error of the call, and sticky: the ranks' exchange epochs are out of step, so every later probe
// of the context fails (plan_for) until the peers are dropped and set again (like comm_failed).
sel_status peer_status(sel_ctx c) {
  if (c->peers && c->h_peer_err && *(volatile uint32_t*)c->h_peer_err) {
    c->peer_failed = true;
    return set_error(SEL_E_STATE, "peer exchange timed out (a rank did not take part)");
  }
  return SEL_OK;
}

template <class P>
bool fits_block(const Plan& plan, size_t nslots, uint32_t nproj) {
  return plan.op.size() <= (size_t)P::kMaxOps && plan.leaves.size() <= (size_t)P::kMaxLeaves &&
         plan.n_intervals <= (size_t)P::kMaxIv && nslots <= (size_t)P::kMaxSlots &&
         nproj <= (uint32_t)P::kMaxProj;
}

// Count fast path (sel_internal.h FastKind): a conjunction of 1..4 leaves, each a point or
// interval(s) on a 4-byte column, one interval on an 8-byte column, or up to 4 points on a
// 1-byte column. Anything else (FLOAT32 keys, 2-byte columns, key sets, OR/NOT structure, wider
// sets) runs the interpreter. Returns the number of fast leaves (0 = interpreter); fills kind[]
// and, for FK_S1 leaves, the byte-replicated point keys. SEL_FAST=0 disables it (pack()).
int fast_kinds(const Plan& plan, const int* types, uint8_t (&kind)[kMaxFastLeaves],
               uint32_t (&pts)[kMaxFastLeaves][4], uint8_t (&npts)[kMaxFastLeaves]) {
  if (plan.path != PATH_CONJ || plan.leaves.empty() || plan.leaves.size() > (size_t)kMaxFastLeaves)
    return 0;
  for (size_t i = 0; i < plan.op.size(); ++i)   // a conjunction evaluates leaves in index order
    if (plan.op[i] == DOP_LEAF && plan.arg[i] >= plan.leaves.size()) return 0;
  for (size_t l = 0; l < plan.leaves.size(); ++l) {
    const PlanLeaf& L = plan.leaves[l];
    const int type = types[L.col];
    if (L.bitmap >= 0 || type == SEL_FLOAT32 || L.iv.empty()) return 0;
    const uint8_t w = wclass_of(type);
    npts[l] = 0;
    if (w == W4) {
      if (L.iv.size() == 1) kind[l] = L.iv[0].lo == L.iv[0].hi ? FK_E4 : FK_R4;
      else if (L.iv.size() <= 4) kind[l] = FK_S4;
      else return 0;
    } else if (w == W8) {
      if (L.iv.size() != 1) return 0;
      kind[l] = FK_R8;
    } else if (w == W1) {
      uint64_t n = 0;
      for (const Interval& x : L.iv) n += x.hi - x.lo + 1;
      if (n > 4) return 0;
      uint32_t k = 0;
      for (const Interval& x : L.iv)
        for (uint64_t v = x.lo; v <= x.hi; ++v) pts[l][k++] = (uint32_t)v * 0x01010101u;
      npts[l] = (uint8_t)n;
      kind[l] = FK_S1;
    } else {
      return 0;
    }
  }
  return (int)plan.leaves.size();
}

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

// Shared-memory bytes of the distinct key sets a plan's IN_BITMAP leaves use.
uint64_t plan_bitmap_bytes(sel_ctx c, const Plan& plan) {
  std::vector<int> ids;
  uint64_t total = 0;
  for (auto& L : plan.leaves) {
    if (L.bitmap < 0 || std::find(ids.begin(), ids.end(), L.bitmap) != ids.end()) continue;
    ids.push_back(L.bitmap);
    total += (c->bm_nbits[L.bitmap] + 127) / 128 * 16;
  }
  return total;
}

size_t count_slots(const Plan& plan) {
  std::vector<int> cols;
  for (auto& L : plan.leaves) cols.push_back(L.col);
  std::sort(cols.begin(), cols.end());
  return (size_t)(std::unique(cols.begin(), cols.end()) - cols.begin());
}

sel_status plan_for(sel_table t, const void* prog, size_t bytes, Plan* plan) {
  if (t->ctx->comm_failed)
    return set_error(SEL_E_NCCL, "the communicator failed earlier (a rank was lost); context unusable");
  if (t->ctx->peer_failed)
    return set_error(SEL_E_STATE, "a peer exchange failed earlier (a rank did not take part); "
                                  "drop the peers and set them again on every rank");
  Program P;
  std::string msg;
  const int st = decode_program(prog, bytes, t->types.data(), (uint32_t)t->types.size(), &P, &msg);
  if (st != SEL_OK) return set_error((sel_status)st, msg);
  const sel_ctx c = t->ctx;
  for (const Instr& in : P.ins)
    if (in.op == 0x31 && (in.a >= c->bm_words.size() || c->bm_words[in.a] == nullptr))
      return set_error(SEL_E_ARG, "IN_BITMAP id " + std::to_string(in.a) + " is not registered");
  plan_program(P, t->types.data(), plan);
  if (plan->max_depth > kMaxDeviceStack)
    return set_error(SEL_E_PROGRAM, "program too deep after canonicalisation");
  return SEL_OK;
}

int grid_for(sel_ctx c, uint64_t units, int occ) {
  const uint64_t persistent = (uint64_t)c->num_sms * (uint64_t)std::max(1, occ);
  return (int)std::max<uint64_t>(1, std::min<uint64_t>({persistent, units, (uint64_t)kMaxGrid}));
}

sel_status ensure_status(sel_ctx c, uint64_t ntiles, cudaStream_t stream) {
  if (c->s.status_cap >= ntiles) return SEL_OK;
  cudaError_t e = sync_stream(c, stream);
  if (e != cudaSuccess) return set_error(sync_code(e), cuda_msg("cudaStreamSynchronize", e));
  if (c->s.status) cudaFree(c->s.status);
  c->s.status = nullptr;
  c->s.status_cap = 0;
  const uint64_t cap = std::max<uint64_t>(ntiles, 1024) * 2;
  e = cudaMalloc(&c->s.status, cap * sizeof(uint64_t));
  if (e != cudaSuccess) return set_error(SEL_E_CUDA, cuda_msg("cudaMalloc(status)", e));
  e = cudaMemsetAsync(c->s.status, 0, cap * sizeof(uint64_t), stream);
  if (e != cudaSuccess) return set_error(SEL_E_CUDA, cuda_msg("cudaMemsetAsync(status)", e));
  c->s.status_cap = cap;
  c->epoch = 0;
  return SEL_OK;
}

sel_status ensure_selection(sel_ctx c, uint64_t nchunks) {
  if (c->sel_cap_chunks >= nchunks) return SEL_OK;
  if (c->sel.bits) cudaFree(c->sel.bits);
  if (c->sel.which) cudaFree(c->sel.which);
  if (c->sel.chunk_cnt) cudaFree(c->sel.chunk_cnt);
  if (c->sel.sb_sum) cudaFree(c->sel.sb_sum);   // the base of the sums / prefix / state block
  c->sel = SelectionBufs{};
  c->sel.code_col = -1;
  c->sel_cap_chunks = 0;
  c->kept_table = nullptr;
  ++c->alloc_gen;
  const uint64_t cap = std::max<uint64_t>(nchunks, 1024);
  const uint64_t nsb = (cap + kSbChunks - 1) / kSbChunks;
  const uint64_t nhb = (cap + kHbChunks - 1) / kHbChunks;
  c->kept_cols.clear();
  cudaError_t e = cudaMalloc(&c->sel.bits, cap * 32 * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMalloc(&c->sel.which, cap * 32 * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMalloc(&c->sel.chunk_cnt, cap * sizeof(uint16_t));
  // one block: superblock sums (two halves) | hyperblock prefix (+ local count, flag) | state;
  // all zero to start with (sel_internal.h SelectionBufs)
  const uint64_t stride = (nsb + 3) & ~3ull;
  const uint64_t words = 2 * stride + ((nhb + 2 + 3) & ~3ull) + 4;
  if (e == cudaSuccess) e = cudaMalloc(&c->sel.sb_sum, words * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemset(c->sel.sb_sum, 0, words * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess) {
    c->sel.sb_stride = (uint32_t)stride;
    c->sel.hb_prefix = c->sel.sb_sum + 2 * stride;
    c->sel.state = c->sel.hb_prefix + ((nhb + 2 + 3) & ~3ull);
  }
  if (e != cudaSuccess) return set_error(SEL_E_CUDA, cuda_msg("cudaMalloc(selection)", e));
  c->sel_cap_chunks = cap;
  return SEL_OK;
}

sel_status ensure_slot(sel_ctx c, int k, uint64_t bytes) {
  if (c->slot_cap[k] >= bytes) return SEL_OK;
  ++c->alloc_gen;
  if (c->slot_buf[k]) cudaFree(c->slot_buf[k]);
  c->slot_buf[k] = nullptr;
  c->slot_cap[k] = 0;
  cudaError_t e = cudaMalloc(&c->slot_buf[k], bytes);
  if (e != cudaSuccess) return set_error(SEL_E_CUDA, cuda_msg("cudaMalloc(kept values)", e));
  c->slot_cap[k] = bytes;
  return SEL_OK;
}

}  // namespace

// ---- ABI -------------------------------------------------------------------------------------------
extern "C" {

int sel_abi_version(void) { return SEL_ABI_VERSION; }
sel_status sel_last_error(void) { return g_status; }
const char* sel_last_error_message(void) { return g_message.c_str(); }

sel_status sel_ctx_create(int cuda_device, sel_ctx* out) {
  clear_error();
  if (!out) return set_error(SEL_E_ARG, "null out");
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess) return set_error(SEL_E_CUDA, cuda_msg("cudaGetDeviceCount", e));
  if (cuda_device < 0 || cuda_device >= ndev) return set_error(SEL_E_CUDA, "no such CUDA device");
  DeviceGuard g(cuda_device);
  if (!g.ok) return set_error(SEL_E_CUDA, "cudaSetDevice failed");
  sel_ctx c = new sel_ctx_s();
  c->device = cuda_device;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, cuda_device);
  c->occ_count_small = occupancy_count_small();
  c->occ_count_large = occupancy_count_large();
  if (prepare_kernels() != cudaSuccess) {
    delete c;
    return set_error(SEL_E_CUDA, "cudaFuncSetAttribute(push-down shared memory) failed");
  }
  // L2 bulk prefetch of the next chunk: measured to help the count that keeps values (extra
  // per-chunk compaction) and to hurt the plain streaming count; SEL_PREFETCH=0/1 forces it.
  const char* pf = std::getenv("SEL_PREFETCH");
  c->prefetch_mode = pf ? (std::strcmp(pf, "1") == 0 ? 1 : 0) : -1;
  const char* kv = std::getenv("SEL_KEEP_VALUES");
  c->keep_values = kv && std::strcmp(kv, "1") == 0;
  const char* ds = std::getenv("SEL_DENSE_SPLIT");
  c->dense_split = !(ds && std::strcmp(ds, "0") == 0);
  const char* cd = std::getenv("SEL_CODED");
  c->code_enabled = !(cd && std::strcmp(cd, "0") == 0);
  const char* gc = std::getenv("SEL_GRAPH_COMM");
  c->graph_comm = !(gc && std::strcmp(gc, "0") == 0);
  const char* fe = std::getenv("SEL_FAST");
  c->fast_enabled = !(fe && std::strcmp(fe, "0") == 0);
  const char* cnw = std::getenv("SEL_COUNT_NW");
  c->count_nw = cnw ? std::atoi(cnw) : 0;
  const char* pp = std::getenv("SEL_PUSHDOWN_PATH");
  c->force_single = pp && std::strcmp(pp, "single") == 0;
  if (pp && std::strcmp(pp, "two") == 0) c->two_pass_min_rows = 0;
  const char* tpm = std::getenv("SEL_TWO_PASS_MIN_ROWS");
  if (tpm && !c->force_single && !(pp && std::strcmp(pp, "two") == 0))
    c->two_pass_min_rows = std::strtoull(tpm, nullptr, 10);
  const char* env = std::getenv("SEL_CTAS_PER_SM");
  if (env && std::atoi(env) > 0) {
    const int v = std::atoi(env);
    c->occ_count_small = std::min(c->occ_count_small, v);
    c->occ_count_large = std::min(c->occ_count_large, v);
  }
  bool okay = cudaMalloc(&c->s.partials, kMaxGrid * sizeof(uint64_t)) == cudaSuccess &&
              cudaMalloc(&c->s.done, sizeof(unsigned int)) == cudaSuccess &&
              cudaMalloc(&c->s.result, kResultSlots * sizeof(uint64_t)) == cudaSuccess &&
              cudaMalloc(&c->s.ticket, sizeof(unsigned long long)) == cudaSuccess &&
              cudaHostAlloc(&c->h_result, kResultSlots * sizeof(uint64_t), cudaHostAllocMapped) == cudaSuccess &&
              cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->h_result_dev), c->h_result, 0) == cudaSuccess &&
              cudaMemset(c->s.done, 0, sizeof(unsigned int)) == cudaSuccess &&
              cudaMemset(c->s.ticket, 0, sizeof(unsigned long long)) == cudaSuccess &&
              cudaMemset(c->s.result, 0, kResultSlots * sizeof(uint64_t)) == cudaSuccess &&
              cudaEventCreate(&c->ev0) == cudaSuccess && cudaEventCreate(&c->ev1) == cudaSuccess &&
              cudaEventCreate(&c->ev2) == cudaSuccess && cudaEventCreate(&c->ev3) == cudaSuccess &&
              cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking) == cudaSuccess &&
              cudaDeviceSynchronize() == cudaSuccess;
  if (!okay) {
    cudaError_t le = cudaGetLastError();
    sel_ctx_destroy(c);  // no tables yet: frees the struct
    return set_error(SEL_E_CUDA, cuda_msg("context allocation", le));
  }
  *out = c;
  return SEL_OK;
}

sel_status sel_nccl_unique_id(void* out128) {
  clear_error();
  if (!out128) return set_error(SEL_E_ARG, "null out");
  NcclApi& n = nccl();
  if (!n.loaded) return set_error(SEL_E_NCCL, n.error);
  ncclUniqueId id;
  ncclResult_t r = n.GetUniqueId(&id);
  if (r != ncclSuccess) return set_error(SEL_E_NCCL, nccl_msg("ncclGetUniqueId", r));
  std::memcpy(out128, &id, sizeof(id));
  return SEL_OK;
}

sel_status sel_ctx_set_comm(sel_ctx ctx, int nranks, int rank, const void* nccl_unique_id) {
  clear_error();
  if (!ctx || !nccl_unique_id || nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks)
    return set_error(SEL_E_ARG, "bad communicator arguments");
  if (ctx->comm) return set_error(SEL_E_STATE, "communicator already set");
  if (ctx->peers && (ctx->nranks != nranks || ctx->rank != rank))
    return set_error(SEL_E_ARG, "communicator ranks differ from the peers'");
  NcclApi& n = nccl();
  if (!n.loaded) return set_error(SEL_E_NCCL, n.error);
  DeviceGuard g(ctx->device);
  ncclUniqueId id;
  std::memcpy(&id, nccl_unique_id, sizeof(id));
  ncclComm_t comm = nullptr;
  ncclResult_t r = n.CommInitRank(&comm, nranks, id, rank);
  if (r != ncclSuccess) return set_error(SEL_E_NCCL, nccl_msg("ncclCommInitRank", r));
  ctx->comm = comm;
  ctx->nranks = nranks;
  ctx->rank = rank;
  return SEL_OK;
}

sel_status sel_ctx_peer_handle(sel_ctx ctx, void* out64) {
  clear_error();
  if (!ctx || !out64) return set_error(SEL_E_ARG, "null argument");
  if (ctx->destroyed) return set_error(SEL_E_STATE, "context destroyed");
  DeviceGuard g(ctx->device);
  if (!g.ok) return set_error(SEL_E_CUDA, "cudaSetDevice failed");
  if (!ctx->peer_buf) {
    const size_t bytes = 2 * (size_t)kMaxPeers * kMaxXchgVals * sizeof(uint64_t);
    cudaError_t e = cudaMalloc(&ctx->peer_buf, bytes);
    if (e == cudaSuccess) e = cudaMemset(ctx->peer_buf, 0, bytes);
    if (e == cudaSuccess) e = cudaMalloc(&ctx->peer_epoch, sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMemset(ctx->peer_epoch, 0, sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaHostAlloc(&ctx->h_peer_err, sizeof(uint32_t), cudaHostAllocMapped);
    if (e == cudaSuccess) *ctx->h_peer_err = 0;
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return set_error(SEL_E_CUDA, cuda_msg("peer buffer", e));
  }
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, ctx->peer_buf);
  if (e != cudaSuccess) return set_error(SEL_E_CUDA, cuda_msg("cudaIpcGetMemHandle", e));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(out64, &h, sizeof(h));
  return SEL_OK;
}

// The base of the allocation holding `p` (driver API, through the runtime's loaded libcuda).
static cudaError_t allocation_base(const void* p, uintptr_t* base) {
  typedef int (*range_fn)(unsigned long long*, size_t*, unsigned long long);
  static range_fn fn = [] {
    void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libcuda.so.1", RTLD_NOW);
    return h ? (range_fn)dlsym(h, "cuMemGetAddressRange_v2") : (range_fn) nullptr;
  }();
  if (!fn) return cudaErrorNotSupported;
  unsigned long long b = 0;
  size_t size = 0;
  if (fn(&b, &size, (unsigned long long)(uintptr_t)p) != 0) return cudaErrorInvalidValue;
  *base = (uintptr_t)b;
  return cudaSuccess;
}

sel_status sel_ctx_export_buffer(sel_ctx ctx, const void* dev_ptr, void* out72) {
  clear_error();
  if (!ctx || !dev_ptr || !out72) return set_error(SEL_E_ARG, "null argument");
  DeviceGuard g(ctx->device);
  if (!g.ok) return set_error(SEL_E_CUDA, "cudaSetDevice failed");
  uintptr_t base = 0;
  cudaError_t e = allocation_base(dev_ptr, &base);
  cudaIpcMemHandle_t h;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return set_error(SEL_E_CUDA, cuda_msg("exporting the buffer", e));
  const uint64_t off = (uint64_t)((uintptr_t)dev_ptr - base);
  std::memcpy(out72, &h, 64);
  std::memcpy(static_cast<char*>(out72) + 64, &off, 8);
  return SEL_OK;
}

sel_status sel_ctx_import_buffer(sel_ctx ctx, const void* handle72, void** out_dev_ptr) {
  clear_error();
  if (!ctx || !handle72 || !out_dev_ptr) return set_error(SEL_E_ARG, "null argument");
  DeviceGuard g(ctx->device);
  if (!g.ok) return set_error(SEL_E_CUDA, "cudaSetDevice failed");
  const std::string key(static_cast<const char*>(handle72), 64);
  uint64_t off = 0;
  std::memcpy(&off, static_cast<const char*>(handle72) + 64, 8);
  auto it = ctx->imported.find(key);
  void* base = nullptr;
  if (it != ctx->imported.end()) {
    base = it->second;
  } else {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle72, 64);
    cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return set_error(SEL_E_CUDA, cuda_msg("cudaIpcOpenMemHandle", e));
    ctx->imported[key] = base;
  }
  *out_dev_ptr = static_cast<char*>(base) + off;
  return SEL_OK;
}

sel_status sel_ctx_set_peers(sel_ctx ctx, int nranks, int rank, const void* handles) {
  clear_error();
  if (ctx && nranks == 0) {  // drop the peers: unmap the others' buffers, keep this rank's
    DeviceGuard g(ctx->device);
    for (void* p : ctx->peer_opened) cudaIpcCloseMemHandle(p);
    ctx->peer_opened.clear();
    for (auto& kv : ctx->imported) cudaIpcCloseMemHandle(kv.second);
    ctx->imported.clear();
    if (ctx->peer_ptrs) cudaFree(ctx->peer_ptrs);
    ctx->peer_ptrs = nullptr;
    ctx->xg = PeerXchg{};
    // a new group starts in step: epoch 0, an empty buffer, no failure, no stale gate word
    // (every rank drops before any rank sets its peers again, as for the first set)
    bool clean = true;
    if (ctx->peer_buf)
      clean = cudaMemset(ctx->peer_buf, 0, 2 * (size_t)kMaxPeers * kMaxXchgVals * sizeof(uint64_t)) ==
                  cudaSuccess &&
              cudaMemset(ctx->peer_epoch, 0, sizeof(uint32_t)) == cudaSuccess;
    clean = clean && cudaMemset(ctx->s.result + kGateSlot, 0, 2 * sizeof(uint64_t)) == cudaSuccess &&
            cudaDeviceSynchronize() == cudaSuccess;
    if (ctx->h_peer_err) *(volatile uint32_t*)ctx->h_peer_err = 0;
    ctx->peer_failed = false;
    if (ctx->peers && !ctx->comm) ctx->nranks = 1, ctx->rank = 0;
    ctx->peers = false;
    ++ctx->alloc_gen;
    return clean ? SEL_OK : set_error(SEL_E_CUDA, "resetting the exchange buffer failed");
  }
  if (!ctx || !handles || nranks < 1 || nranks > kMaxPeers || rank < 0 || rank >= nranks)
    return set_error(SEL_E_ARG, "bad peer arguments");
  if (ctx->peers) return set_error(SEL_E_STATE, "peers already set");
  if (!ctx->peer_buf) return set_error(SEL_E_STATE, "export this rank's handle (sel_ctx_peer_handle) first");
  if (ctx->comm && (ctx->nranks != nranks || ctx->rank != rank))
    return set_error(SEL_E_ARG, "peer ranks differ from the communicator's");
  DeviceGuard g(ctx->device);
  if (!g.ok) return set_error(SEL_E_CUDA, "cudaSetDevice failed");
  std::vector<uint64_t*> ptrs(nranks, nullptr);
  std::vector<void*> opened;
  cudaError_t e = cudaSuccess;
  for (int r = 0; r < nranks && e == cudaSuccess; ++r) {
    if (r == rank) {
      ptrs[r] = ctx->peer_buf;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const char*>(handles) + 64 * (size_t)r, sizeof(h));
    void* p = nullptr;
    e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e == cudaSuccess) {
      opened.push_back(p);
      ptrs[r] = static_cast<uint64_t*>(p);
    }
  }
  uint64_t** dptrs = nullptr;
  if (e == cudaSuccess) e = cudaMalloc(&dptrs, nranks * sizeof(uint64_t*));
  if (e == cudaSuccess)
    e = cudaMemcpy(dptrs, ptrs.data(), nranks * sizeof(uint64_t*), cudaMemcpyHostToDevice);
  uint32_t* derr = nullptr;
  if (e == cudaSuccess) e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&derr), ctx->h_peer_err, 0);
  if (e != cudaSuccess) {
    for (void* p : opened) cudaIpcCloseMemHandle(p);
    if (dptrs) cudaFree(dptrs);
    return set_error(SEL_E_CUDA, cuda_msg("opening the peers' buffers", e));
  }
  ctx->peer_opened = opened;
  ctx->peer_ptrs = dptrs;
  ctx->xg = PeerXchg{dptrs, ctx->peer_buf, ctx->peer_epoch, derr, nranks, rank, ctx->peer_timeout_ns};
  ctx->peers = true;
  ctx->nranks = nranks;
  ctx->rank = rank;
  ++ctx->alloc_gen;   // prepared executes re-capture with the exchange
  return SEL_OK;
}

namespace {
void release_ctx_resources(sel_ctx c) {
  DeviceGuard g(c->device);
  if (c->comm && nccl().loaded) nccl().CommDestroy(c->comm);
  c->comm = nullptr;
  for (void* p : c->peer_opened) cudaIpcCloseMemHandle(p);
  c->peer_opened.clear();
  for (auto& kv : c->imported) cudaIpcCloseMemHandle(kv.second);
  c->imported.clear();
  if (c->hist_buf) cudaFree(c->hist_buf);
  c->hist_buf = nullptr;
  c->hist_cap = 0;
  if (c->peer_ptrs) cudaFree(c->peer_ptrs);
  if (c->peer_buf) cudaFree(c->peer_buf);
  if (c->peer_epoch) cudaFree(c->peer_epoch);
  if (c->h_peer_err) cudaFreeHost(c->h_peer_err);
  c->peer_ptrs = nullptr;
  c->peer_buf = nullptr;
  c->peer_epoch = nullptr;
  c->h_peer_err = nullptr;
  c->peers = false;
  if (c->s.partials) cudaFree(c->s.partials);
  if (c->s.done) cudaFree(c->s.done);
  if (c->s.result) cudaFree(c->s.result);
  if (c->s.ticket) cudaFree(c->s.ticket);
  if (c->s.status) cudaFree(c->s.status);
  if (c->h_result) cudaFreeHost(c->h_result);
  if (c->sel.bits) cudaFree(c->sel.bits);
  if (c->sel.which) cudaFree(c->sel.which);
  if (c->sel.chunk_cnt) cudaFree(c->sel.chunk_cnt);
  if (c->sel.sb_sum) cudaFree(c->sel.sb_sum);
  c->sel = SelectionBufs{};
  c->sel_cap_chunks = 0;
  c->kept_table = nullptr;
  for (int k = 0; k < kMaxKeep; ++k) {
    if (c->slot_buf[k]) cudaFree(c->slot_buf[k]);
    c->slot_buf[k] = nullptr;
    c->slot_cap[k] = 0;
  }
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->ev2) cudaEventDestroy(c->ev2);
  if (c->ev3) cudaEventDestroy(c->ev3);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  c->cap_stream = nullptr;
  c->s = Scratch{};
  c->h_result = nullptr;
  c->ev0 = c->ev1 = c->ev2 = c->ev3 = nullptr;
}
}  // namespace

// Destroying a context that still has registered tables releases its device resources at once;
// the struct itself lives until the last table is released (so a late sel_table_release is safe),
// and probes on those tables fail with SEL_E_STATE.
void sel_ctx_destroy(sel_ctx c) {
  if (!c || c->destroyed) return;
  release_ctx_resources(c);
  c->destroyed = true;
  if (c->live_tables == 0) delete c;
}

sel_status sel_ctx_set_peer_timeout(sel_ctx ctx, uint64_t timeout_ms) {
  clear_error();
  if (!ctx || timeout_ms == 0 || timeout_ms > 3600000ull)
    return set_error(SEL_E_ARG, "timeout must be 1 ms .. 1 h");
  ctx->peer_timeout_ns = timeout_ms * 1000000ull;
  ctx->xg.timeout_ns = ctx->peer_timeout_ns;
  ++ctx->alloc_gen;   // prepared executes bake the exchange parameters: re-capture
  return SEL_OK;
}

sel_status sel_ctx_set_timing(sel_ctx ctx, int enable) {
  clear_error();
  if (!ctx) return set_error(SEL_E_ARG, "null ctx");
  ctx->timing = enable != 0;
  ctx->last_ms = 0.f;
  return SEL_OK;
}

sel_status sel_ctx_set_pushdown_path(sel_ctx ctx, int mode) {
  clear_error();
  if (!ctx) return set_error(SEL_E_ARG, "null ctx");
  if (mode != -1 && mode != 0 && mode != 2) return set_error(SEL_E_ARG, "mode must be -1, 0 or 2");
  ctx->force_single = mode == 0;
  ctx->two_pass_min_rows = mode == 2 ? 0 : (mode == 0 ? ~0ull : kTwoPassMinRows);
  return SEL_OK;
}

sel_status sel_ctx_last_kernel_ms(sel_ctx ctx, float* ms) {
  clear_error();
  if (!ctx || !ms) return set_error(SEL_E_ARG, "null argument");
  *ms = ctx->timing ? ctx->last_ms : 0.f;
  return SEL_OK;
}

sel_status sel_table_register(sel_ctx ctx, const sel_column* cols, uint32_t ncols,
                              uint64_t local_rows, uint64_t global_row_offset,
                              uint64_t global_rows, sel_table* out) {
  clear_error();
  if (!ctx || !cols || !out) return set_error(SEL_E_ARG, "null argument");
  *out = nullptr;
  if (ctx->destroyed) return set_error(SEL_E_STATE, "context destroyed");
  if (ncols == 0 || ncols > 255) return set_error(SEL_E_ARG, "ncols must be 1..255");
  if (global_rows >= (1ull << 32)) return set_error(SEL_E_TOO_LARGE, "global_rows must be < 2^32");
  if (global_row_offset > global_rows || local_rows > global_rows - global_row_offset)
    return set_error(SEL_E_ARG, "shard [offset, offset + local_rows) exceeds global_rows");
  for (uint32_t c = 0; c < ncols; ++c) {
    const sel_column& col = cols[c];
    if (!known_type(col.type)) return set_error(SEL_E_TYPE, "unknown column type at " + std::to_string(c));
    if (local_rows > 0 && col.data == nullptr) return set_error(SEL_E_ARG, "null column data at " + std::to_string(c));
    if (((uintptr_t)col.data & 15u) != 0) return set_error(SEL_E_ALIGN, "column data not 16-byte aligned at " + std::to_string(c));
    const uint64_t code_range = col.type == SEL_DICT8 ? (1ull << 8) : col.type == SEL_DICT16 ? (1ull << 16) : (1ull << 32);
    if ((col.type == SEL_DICT8 || col.type == SEL_DICT16) && col.dict_size > code_range)
      return set_error(SEL_E_ARG, "dict_size above the code range at " + std::to_string(c));
  }
  sel_table t = new sel_table_s();
  t->ctx = ctx;
  t->cols.assign(cols, cols + ncols);
  for (uint32_t c = 0; c < ncols; ++c) t->types.push_back((int)cols[c].type);
  t->local_rows = local_rows;
  t->row_offset = global_row_offset;
  t->global_rows = global_rows;
  ctx->live_tables++;
  *out = t;
  return SEL_OK;
}

void sel_table_release(sel_table t) {
  if (!t) return;
  sel_ctx c = t->ctx;
  if (c->kept_table == t) c->kept_table = nullptr;
  for (sel_prepared q : t->prepared) q->t = nullptr;
  delete t;
  if (--c->live_tables == 0 && c->destroyed) delete c;
}

sel_status sel_program_check(const void* prog, size_t prog_bytes, const sel_type* types,
                             uint32_t ncols) {
  clear_error();
  std::vector<int> ty(ncols);
  for (uint32_t c = 0; c < ncols; ++c) {
    if (!types || !known_type(types[c])) return set_error(SEL_E_TYPE, "unknown column type");
    ty[c] = (int)types[c];
  }
  Program P;
  std::string msg;
  const int st = decode_program(prog, prog_bytes, ty.data(), ncols, &P, &msg);
  if (st != SEL_OK) return set_error((sel_status)st, msg);
  return SEL_OK;
}

int sel_program_path(const void* prog, size_t prog_bytes, const sel_type* types, uint32_t ncols) {
  const sel_status st = sel_program_check(prog, prog_bytes, types, ncols);
  if (st != SEL_OK) return -(int)st;
  std::vector<int> ty(types, types + ncols);
  Program P;
  decode_program(prog, prog_bytes, ty.data(), ncols, &P, nullptr);
  Plan plan;
  plan_program(P, ty.data(), &plan);
  return plan.path;
}

long sel_program_plan_json(const void* prog, size_t prog_bytes, const sel_type* types,
                           uint32_t ncols, char* buf, size_t cap) {
  const sel_status st = sel_program_check(prog, prog_bytes, types, ncols);
  if (st != SEL_OK) return -(long)st;
  std::vector<int> ty(types, types + ncols);
  Program P;
  decode_program(prog, prog_bytes, ty.data(), ncols, &P, nullptr);
  Plan plan;
  plan_program(P, ty.data(), &plan);
  std::string js = "{\"path\": " + std::to_string(plan.path) +
                   ", \"const\": " + (plan.const_value ? "true" : "false") +
                   ", \"max_depth\": " + std::to_string(plan.max_depth) + ", \"ops\": [";
  for (size_t i = 0; i < plan.op.size(); ++i)
    js += (i ? ", [" : "[") + std::to_string(plan.op[i]) + ", " + std::to_string(plan.arg[i]) + "]";
  js += "], \"leaves\": [";
  for (size_t l = 0; l < plan.leaves.size(); ++l) {
    const PlanLeaf& L = plan.leaves[l];
    const int type = ty[L.col];
    const uint64_t bias = key_sign_bias(type);
    std::string lo, sp;
    for (size_t i = 0; i < L.iv.size(); ++i) {
      lo += (i ? ", " : "") + std::to_string(L.iv[i].lo ^ bias);
      sp += (i ? ", " : "") + std::to_string(L.iv[i].hi - L.iv[i].lo);
    }
    if (L.bitmap >= 0) {
      js += (l ? ", " : "") + std::string("{\"col\": ") + std::to_string(L.col) +
            ", \"wclass\": " + std::to_string(wclass_of(type)) + ", \"bitmap\": " +
            std::to_string(L.bitmap) + ", \"negate\": " + (L.negate ? "true" : "false") + "}";
      continue;
    }
    js += (l ? ", " : "") + std::string("{\"col\": ") + std::to_string(L.col) +
          ", \"wclass\": " + std::to_string(wclass_of(type)) +
          ", \"fkey\": " + (type == SEL_FLOAT32 ? "1" : "0") + ", \"lo\": [" + lo +
          "], \"span\": [" + sp + "]}";
  }
  js += "], \"fast\": [";
  uint8_t kind[kMaxFastLeaves], npts[kMaxFastLeaves];
  uint32_t pts[kMaxFastLeaves][4];
  const int nf = fast_kinds(plan, ty.data(), kind, pts, npts);
  for (int l = 0; l < nf; ++l) js += (l ? ", " : "") + std::to_string(kind[l]);
  js += "]}";
  if (buf && cap > 0) {
    const size_t n = std::min(cap - 1, js.size());
    std::memcpy(buf, js.data(), n);
    buf[n] = '\0';
  }
  return (long)js.size();
}

sel_status sel_bitmap_register(sel_ctx c, const uint64_t* words, uint64_t nbits, uint32_t* out_id) {
  clear_error();
  if (!c || !words || !out_id) return set_error(SEL_E_ARG, "null argument");
  if (c->destroyed) return set_error(SEL_E_STATE, "context destroyed");
  if (nbits == 0 || nbits >= (1ull << 31)) return set_error(SEL_E_ARG, "nbits must be 1..2^31-1");
  if (reinterpret_cast<uintptr_t>(words) % 16 != 0)
    return set_error(SEL_E_ALIGN, "bitmap words must be 16-byte aligned");
  size_t id = 0;
  while (id < c->bm_words.size() && c->bm_words[id] != nullptr) ++id;
  if (id >= kMaxBitmaps) return set_error(SEL_E_TOO_LARGE, "too many registered bitmaps");
  if (id == c->bm_words.size()) {
    c->bm_words.push_back(nullptr);
    c->bm_nbits.push_back(0);
  }
  c->bm_words[id] = words;
  c->bm_nbits[id] = nbits;
  c->kept_table = nullptr;  // a kept selection may have used a previous set under this id
  ++c->bm_gen;
  *out_id = (uint32_t)id;
  return SEL_OK;
}

sel_status sel_bitmap_release(sel_ctx c, uint32_t id) {
  clear_error();
  if (!c) return set_error(SEL_E_ARG, "null ctx");
  if (id >= c->bm_words.size() || c->bm_words[id] == nullptr)
    return set_error(SEL_E_ARG, "bitmap id not registered");
  c->bm_words[id] = nullptr;
  c->bm_nbits[id] = 0;
  c->kept_table = nullptr;
  ++c->bm_gen;
  return SEL_OK;
}

uint64_t sel_count(sel_table t, const void* prog, size_t prog_bytes, void* cuda_stream) {
  return sel_count_ex(t, prog, prog_bytes, 0u, nullptr, 0u, cuda_stream);
}


sel_status sel_ctx_last_times(sel_ctx ctx, float* count_ms, float* pushdown_ms) {
  clear_error();
  if (!ctx) return set_error(SEL_E_ARG, "null ctx");
  if (count_ms) *count_ms = ctx->timing ? ctx->last_count_ms : 0.f;
  if (pushdown_ms) *pushdown_ms = ctx->timing ? ctx->last_push_ms : 0.f;
  return SEL_OK;
}

int sel_ctx_last_pushdown_path(sel_ctx ctx) { return ctx ? ctx->last_pd_path : -1; }

double sel_sample_estimate(uint64_t sample_count, uint64_t sample_rows, uint64_t table_rows) {
  if (sample_rows == 0) return 0.0;
  return (double)sample_count * (double)table_rows / (double)sample_rows;
}

double sel_equi_depth_estimate(const int64_t* lo, const int64_t* hi, const uint64_t* distinct,
                               uint32_t nbuckets, uint64_t table_rows, int64_t value) {
  if (!lo || !hi || !distinct || nbuckets == 0) return std::nan("");
  const double d = (double)table_rows / (double)nbuckets;                   // D = T(R) / B
  double est = 0.0;
  for (uint32_t b = 0; b < nbuckets; ++b)                                   // D / V(b_x)
    if (distinct[b] && lo[b] <= value && value <= hi[b]) est += d / (double)distinct[b];
  return est;
}
int sel_ctx_last_pushdown_flags(sel_ctx ctx) {
  return ctx ? (ctx->last_pd_path == 1 || ctx->last_pd_path == 2 ? ctx->last_pd_flags : 0) : -1;
}

}  // extern "C"

namespace {

// Timing event on `s`; inside a stream capture it must be an external event-record node (a plain
// record would only express a dependency within the capture).
void record(sel_ctx c, cudaEvent_t ev, cudaStream_t s) {
  if (c->capturing) cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal);
  else cudaEventRecord(ev, s);
}

// Columns whose value is the same in every selected row: in a conjunction of leaves, a leaf whose
// key-space set is one point {k} pins its column to the single raw bit pattern that maps to k
// (exact: the key maps are bijections, and -0/+0 are two keys so x = 0.0 is never a point).
// Returns (column, raw bits) pairs; the push-down fills them instead of keeping or gathering.
std::vector<std::pair<int, uint64_t>> const_columns(sel_table t, const Plan& plan) {
  std::vector<std::pair<int, uint64_t>> out;
  if (plan.path != PATH_CONJ) return out;
  for (const PlanLeaf& L : plan.leaves) {
    if (L.bitmap >= 0 || L.iv.size() != 1 || L.iv[0].lo != L.iv[0].hi) continue;
    const int type = t->types[L.col];
    const uint64_t k = L.iv[0].lo;
    uint64_t raw;
    if (type == SEL_FLOAT32) {
      const uint32_t x = (uint32_t)k;
      raw = (x & 0x80000000u) ? (x ^ 0x80000000u) : (~x & 0xFFFFFFFFu);
    } else {
      const int w = width_of(type);
      raw = (k ^ key_sign_bias(type)) & (w == 8 ? ~0ull : ((1ull << (8 * w)) - 1));
    }
    out.emplace_back(L.col, raw);
  }
  return out;
}

bool is_const_col(const std::vector<std::pair<int, uint64_t>>& cc, int col, uint64_t* raw) {
  for (auto& x : cc)
    if (x.first == col) {
      if (raw) *raw = x.second;
      return true;
    }
  return false;
}

// The projected predicate columns whose selected values a keeping count stores (<= kMaxKeep,
// within the warp's capture budget) with their shared-memory capture offsets; *off advances.
std::vector<std::pair<int, uint32_t>> choose_kept(sel_table t, const Plan& plan,
                                                  const uint32_t* keep_cols, uint32_t nkeep,
                                                  uint32_t* off) {
  std::vector<std::pair<int, uint32_t>> chosen;
  const auto consts = const_columns(t, plan);   // filled by the push-down, never kept
  for (uint32_t j = 0; j < nkeep && (int)chosen.size() < kMaxKeep; ++j) {
    const int col = (int)keep_cols[j];
    if (is_const_col(consts, col, nullptr)) continue;
    bool pred_col = false, dup = false;
    for (auto& L : plan.leaves) pred_col = pred_col || L.col == col;
    for (auto& ck : chosen) dup = dup || ck.first == col;
    const uint32_t w = (uint32_t)width_of(t->types[col]);
    if (!pred_col || dup || *off + w * kChunkRows > kIdxBytes + kCaptureBudget) continue;
    chosen.emplace_back(col, *off);
    *off += w * kChunkRows;
  }
  return chosen;
}

// Device memory a keeping count of t needs (selection + kept-value slots); allocates only when
// the context's buffers are too small (bumping alloc_gen, which invalidates captured graphs).
sel_status reserve_selection(sel_table t, uint64_t nchunks,
                             const std::vector<std::pair<int, uint32_t>>& chosen) {
  sel_ctx c = t->ctx;
  if (ensure_selection(c, nchunks) != SEL_OK) return g_status;
  for (size_t k = 0; k < chosen.size(); ++k) {
    const uint64_t w = (uint64_t)width_of(t->types[chosen[k].first]);
    if (ensure_slot(c, (int)k, nchunks * (uint64_t)kChunkRows * w) != SEL_OK) return g_status;
  }
  return SEL_OK;
}

// Enqueue the count of `plan` over t's shard on `stream`: the count kernel
// (keeping the selection with SEL_KEEP_SELECTION) writes the local count to *d_out, then the
// 8-byte all-reduce makes it global in place. Nothing waits for the host.
// code_cols (a keeping count without kept values): projected columns the materialisation will
// write; one pinned by a two-point 1-byte leaf of the fast path gets its per-row code bit kept
// (SelectionBufs::which) so that the push-down never reads it (kCodedProj).
sel_status enqueue_count(sel_table t, const Plan& plan, uint32_t flags, const uint32_t* keep_cols,
                         uint32_t nkeep, cudaStream_t stream, uint64_t* d_out,
                         bool allreduce = true, const uint32_t* code_cols = nullptr,
                         uint32_t ncode = 0, const ExecFinish* fin = nullptr) {
  sel_ctx c = t->ctx;
  const uint64_t n = t->local_rows;
  const bool scan = n > 0 && plan.path != PATH_CONST;
  cudaError_t e;
  if (scan) {
    const uint64_t nchunks = (n + kChunkRows - 1) / kChunkRows;
    const uint64_t units = (nchunks + kWarpsPerCta - 1) / kWarpsPerCta;
    const size_t nslots = count_slots(plan);
    const SelectionBufs* keep = nullptr;
    std::vector<int> cap_off(t->cols.size(), -1);
    if (flags & SEL_KEEP_SELECTION) {
      if (ensure_selection(c, nchunks) != SEL_OK) return g_status;
      c->kept_table = nullptr;  // valid again only once this probe has completed
      c->kept_cols.clear();
      // projected predicate columns: capture while evaluating, keep the selected values
      uint32_t off = kIdxBytes;
      auto chosen = choose_kept(t, plan, keep_cols, nkeep, &off);
      // Key sets staged in shared memory save far more than kept values do: when both do not
      // fit, keep no values (the push-down then gathers those columns).
      const uint64_t bmb = plan_bitmap_bytes(c, plan);
      if (!chosen.empty() && bmb > 0 && bmb <= kMaxCountSmem &&
          (uint64_t)((off + 15u) & ~15u) * kWarpsPerCta + bmb > kMaxCountSmem) {
        chosen.clear();
        off = kIdxBytes;
      }
      if (reserve_selection(t, nchunks, chosen) != SEL_OK) return g_status;
      for (const auto& ck : chosen) {
        const int col = ck.first, k = (int)c->kept_cols.size();
        cap_off[col] = (int)ck.second;
        c->sel.keep_col[k] = (uint8_t)col;
        c->sel.keep_wclass[k] = wclass_of(t->types[col]);
        c->sel.keep_cap_off[k] = (uint16_t)ck.second;
        c->sel.keep_slot[k] = c->slot_buf[k];
        c->kept_cols.push_back(col);
      }
      c->sel.n_keep = (uint32_t)c->kept_cols.size();
      c->sel.warp_smem = c->sel.n_keep ? ((off + 15u) & ~15u) : 0u;
      keep = &c->sel;
    }
    auto mark_captures = [&](auto* p) {
      std::vector<bool> marked(t->cols.size(), false);
      for (size_t i = 0; i < plan.op.size(); ++i) {
        if (plan.op[i] != DOP_LEAF) continue;
        const int l = plan.arg[i];
        const int col = plan.leaves[l].col;
        if (cap_off[col] >= 0 && !marked[col]) {
          p->leaf[l].cap = 1;
          p->leaf[l].cap_off = (uint16_t)cap_off[col];
          marked[col] = true;
        }
      }
    };
    const size_t dyn = keep ? (size_t)keep->warp_smem * kWarpsPerCta : 0;
    Scratch s = c->s;
    s.result = d_out;
    // the exchange fused into the count (for an Execute inside its finish, `fin`)
    s.xg = (c->peers && (allreduce || fin)) ? c->xg : PeerXchg{};
    if (c->timing) record(c, c->ev0, stream);
    int le;
    if (fits_block<DevProgramSmall>(plan, nslots, 0)) {
      DevProgramSmall p;
      pack(plan, t, &p);
      mark_captures(&p);
      choose_bitmap_staging(&p, dyn);
      if (keep) {
        c->sel.code_col = -1;
        if (keep->n_keep == 0 && p.fast_n > 0 && c->code_enabled) {
          for (uint32_t s2 = 0; s2 < p.fast_n && c->sel.code_col < 0; ++s2) {
            const DevLeaf& L = p.leaf[s2];
            const bool s1 = p.fast_kind[s2] == FK_S1 && p.fast_npts[s2] == 2;
            const bool s4 = p.fast_kind[s2] == FK_S4 && L.iv_count == 2 &&
                            p.span[L.iv_begin] == 0 && p.span[L.iv_begin + 1] == 0;
            if (!s1 && !s4) continue;
            const int col = plan.leaves[s2].col;
            for (uint32_t j = 0; j < ncode; ++j) {
              if ((int)code_cols[j] != col) continue;
              p.fast_code = (int32_t)s2;
              c->sel.code_col = col;
              c->sel.code_pts =
                  s1 ? (uint64_t)((p.fast_pts[s2][0] & 0xFFu) | ((p.fast_pts[s2][1] & 0xFFu) << 8))
                     : ((uint64_t)(uint32_t)p.lo[L.iv_begin] |
                        ((uint64_t)(uint32_t)p.lo[L.iv_begin + 1] << 32));
              break;
            }
          }
        }
      }
      if (c->prefetch_mode < 0) p.prefetch = ((keep && keep->n_keep) || p.bm_smem) ? 1u : 0u;
      int occ = keep ? occupancy_count_keep_small(dyn + p.bm_smem)
                     : (p.bm_smem ? occupancy_count_dyn_small(p.bm_smem) : c->occ_count_small);
      if (p.fast_n && !p.bm_smem) occ = occupancy_count_fast((int)p.fast_n, keep != nullptr, dyn);
      const int nw = pick_count_warps(c, p, dyn, occ);
      le = launch_count_small(p, n, grid_for(c, nw == kWarpsPerCta ? units : (nchunks + nw - 1) / nw,
                                             nw == kWarpsPerCta ? occ : 1), s, keep, stream, nw, fin);
    } else {
      static thread_local DevProgramLarge p;
      pack(plan, t, &p);
      mark_captures(&p);
      choose_bitmap_staging(&p, dyn);
      if (keep) c->sel.code_col = -1;
      if (c->prefetch_mode < 0) p.prefetch = ((keep && keep->n_keep) || p.bm_smem) ? 1u : 0u;
      const int occ = keep ? occupancy_count_keep_large(dyn + p.bm_smem)
                           : (p.bm_smem ? occupancy_count_dyn_large(p.bm_smem) : c->occ_count_large);
      const int nw = pick_count_warps(c, p, dyn, occ);
      le = launch_count_large(p, n, grid_for(c, nw == kWarpsPerCta ? units : (nchunks + nw - 1) / nw,
                                             nw == kWarpsPerCta ? occ : 1), s, keep, stream, nw, fin);
    }
    if (le != cudaSuccess) return set_error(SEL_E_CUDA, cuda_msg("count kernel launch", (cudaError_t)le));
    if (c->timing) record(c, c->ev1, stream);
  } else {
    uint64_t* h = c->h_result + (d_out - c->s.result);
    *h = plan.path == PATH_CONST && plan.const_value ? n : 0;
    e = cudaMemcpyAsync(d_out, h, sizeof(uint64_t), cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) return set_error(SEL_E_CUDA, cuda_msg("cudaMemcpyAsync", e));
  }
  if (c->peers && allreduce && !scan) {  // SURVEY §8a a4 over peer memory (a scan fuses it, above)
    const int le = launch_peer_exchange(c->xg, d_out, 1, nullptr, d_out, stream);
    if (le != cudaSuccess) return set_error(SEL_E_CUDA, cuda_msg("peer exchange", (cudaError_t)le));
  } else if (c->comm && allreduce && !c->peers) {  // one 8-byte all-reduce on the probe stream
    ncclResult_t r = nccl().AllReduce(d_out, d_out, 1, ncclUint64, ncclSum, c->comm, stream);
    if (r != ncclSuccess) return set_error(SEL_E_NCCL, nccl_msg("ncclAllReduce", r));
  }
  return SEL_OK;
}

// Enqueue the materialisation from the kept selection (pushdown_sel): every
// projection gathered from global memory or copied from its kept-value slot. gate: write nothing
// when the global count in Scratch::result[kGateSlot] exceeds gate_max (sel_execute).
sel_status enqueue_pushdown_sel(sel_table t, const Plan& plan, const uint32_t* proj_cols,
                                uint32_t nproj, uint32_t* out_rowids, void* const* out_cols,
                                uint64_t capacity_rows, bool gate, uint64_t gate_max,
                                cudaStream_t stream, int gate_ranks = 0,
                                const PeerXchg* xg = nullptr, bool global_out = false,
                                bool finished = false, uint64_t* host = nullptr) {
  sel_ctx c = t->ctx;
  const auto consts = const_columns(t, plan);
  const uint64_t n = t->local_rows;
  const uint64_t ntiles = (n + kChunkRows - 1) / kChunkRows;
  auto fill_sel = [&](auto* p) {
    std::memset(p, 0, sizeof(*p));
    p->row_offset = t->row_offset;
    p->capacity = capacity_rows;
    p->gate = gate ? 1u : 0u;
    p->gate_max = gate_max;
    p->global_out = global_out ? 1u : 0u;
    p->dense_split = (c->dense_split && n >= kDenseSplitMinRows) ? 1u : 0u;
    p->n_proj = capacity_rows > 0 ? nproj : 0;
    for (uint32_t j = 0; j < p->n_proj; ++j) {
      p->proj_src[j] = t->cols[proj_cols[j]].data;
      p->proj_dst[j] = out_cols[j];
      p->proj_wclass[j] = wclass_of(t->types[proj_cols[j]]);
      p->proj_cap_off[j] = kNoCapture;
      uint64_t raw = 0;
      if (is_const_col(consts, (int)proj_cols[j], &raw)) {
        p->proj_cap_off[j] = kConstProj;
        p->proj_src[j] = reinterpret_cast<const void*>((uintptr_t)raw);
      } else if (c->sel.code_col >= 0 && c->sel.code_col == (int)proj_cols[j]) {
        p->proj_cap_off[j] = kCodedProj;   // from the kept code bits (enqueue_count)
        p->proj_src[j] = reinterpret_cast<const void*>((uintptr_t)c->sel.code_pts);
        p->coded = 1;
        continue;
      } else {
        for (size_t k = 0; k < c->kept_cols.size(); ++k)
          if (c->kept_cols[k] == (int)proj_cols[j]) p->proj_cap_off[j] = (uint16_t)(kKeptBase + k);
      }
      if (p->proj_cap_off[j] != kNoCapture) ++p->n_direct;
    }
  };
  const uint64_t nblocks = (ntiles + kSelBlockChunks - 1) / kSelBlockChunks;
  const uint64_t units = (nblocks + kWarpsPerCta - 1) / kWarpsPerCta;
  auto flags_of = [](const auto& p) {
    int f = (p.coded ? SEL_PD_CODED : 0) | (p.dense_split ? SEL_PD_WHOLE_CHUNKS : 0);
    for (uint32_t j = 0; j < p.n_proj; ++j) {
      if (p.proj_cap_off[j] == kConstProj) f |= SEL_PD_CONSTANT;
      else if (p.proj_cap_off[j] >= kKeptBase && p.proj_cap_off[j] < kCodedProj) f |= SEL_PD_KEPT_VALUES;
    }
    return f;
  };
  int le;
  if (nproj <= (uint32_t)DevProgramSmall::kMaxProj) {
    DevProgramSmall p;
    fill_sel(&p);
    c->last_pd_flags = flags_of(p);
    le = launch_pushdown_sel_small(p, n, out_rowids, grid_for(c, units, occupancy_pushdown_sel_small()),
                                   c->s, c->sel, stream, gate_ranks, xg, c->rank, finished, host);
  } else {
    static thread_local DevProgramLarge p;
    fill_sel(&p);
    c->last_pd_flags = flags_of(p);
    le = launch_pushdown_sel_large(p, n, out_rowids, grid_for(c, units, occupancy_pushdown_sel_large()),
                                   c->s, c->sel, stream, gate_ranks, xg, c->rank, finished, host);
  }
  if (le != cudaSuccess) return set_error(SEL_E_CUDA, cuda_msg("push-down kernel launch", (cudaError_t)le));
  c->last_pd_path = 1;
  return SEL_OK;
}

// All-gather a per-rank count into result[1..nranks] and its pinned mirror,
// blocking (used where a rank has nothing of its own to enqueue but must match the collectives of
// the others).
sel_status gather_counts(sel_ctx c, uint64_t local, void* cuda_stream) {
  cudaStream_t stream = (cudaStream_t)cuda_stream;
  DeviceGuard g(c->device);
  if (!g.ok) return set_error(SEL_E_CUDA, "cudaSetDevice failed");
  c->h_result[0] = local;
  cudaError_t e = cudaMemcpyAsync(c->s.result, c->h_result, sizeof(uint64_t), cudaMemcpyHostToDevice, stream);
  if (e != cudaSuccess) return set_error(SEL_E_CUDA, cuda_msg("cudaMemcpyAsync", e));
  if (c->peers) {
    const int le = launch_peer_exchange(c->xg, c->s.result, 1, c->s.result + 1, nullptr, stream);
    if (le != cudaSuccess) return set_error(SEL_E_CUDA, cuda_msg("peer exchange", (cudaError_t)le));
  } else {
    ncclResult_t r = nccl().AllGather(c->s.result, c->s.result + 1, 1, ncclUint64, c->comm, stream);
    if (r != ncclSuccess) return set_error(SEL_E_NCCL, nccl_msg("ncclAllGather", r));
  }
  e = cudaMemcpyAsync(c->h_result + 1, c->s.result + 1, c->nranks * sizeof(uint64_t),
                      cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = sync_stream(c, stream);
  if (e != cudaSuccess) return set_error(sync_code(e), cuda_msg("all-gather result", e));
  return peer_status(c);
}

// The device work of a device-gated Execute on `stream` (sel_execute, prepared executes): the
// count keeping the selection (local count -> result[kGateSlot]) whose last CTA also leaves the
// superblock prefix and — without NCCL — finishes the result words (ExecFinish: the peer exchange,
// the gate count, the mirror and the offset, stored into the pinned host mirror too); with NCCL
// the all-gather of the per-rank counts into result[1..nranks] and a 1-CTA kernel finishing the
// same words; then the gated materialisation. No copy: the host reads its pinned mirror after its
// one synchronisation (more than kMirrorMax ranks: two D2H copies instead).
sel_status enqueue_execute(sel_table t, const Plan& plan, const uint32_t* proj, uint32_t nproj,
                           uint32_t nkeep, uint64_t max_size, uint32_t* out_rowids,
                           void* const* outs, uint64_t capacity, cudaStream_t s,
                           bool global_out = false) {
  sel_ctx c = t->ctx;
  const bool nccl_gate = c->comm && !c->peers;
  const int nr = multi(c) ? c->nranks : 0;
  uint64_t* host = nr <= kMirrorMax ? c->h_result_dev : nullptr;
  const ExecFinish fin{c->s.result, host, 0, c->rank};
  sel_status st = enqueue_count(t, plan, SEL_KEEP_SELECTION, proj, nkeep, s, c->s.result + kGateSlot,
                                false, proj, nproj, nccl_gate ? nullptr : &fin);
  if (st != SEL_OK) return st;
  if (nccl_gate) {  // SURVEY §8a a4 + a7 in one collective
    ncclResult_t r = nccl().AllGather(c->s.result + kGateSlot, c->s.result + 1, 1, ncclUint64,
                                      c->comm, s);
    if (r != ncclSuccess) return set_error(SEL_E_NCCL, nccl_msg("ncclAllGather", r));
  }
  if (c->timing) record(c, c->ev2, s);
  st = enqueue_pushdown_sel(t, plan, proj, nproj, out_rowids, outs, capacity, true, max_size, s,
                            nccl_gate ? c->nranks : 0, nullptr, global_out, !nccl_gate, host);
  if (st != SEL_OK) return st;
  if (c->timing) record(c, c->ev3, s);
  if (host) return SEL_OK;
  cudaError_t e = cudaMemcpyAsync(c->h_result + kGateSlot, c->s.result + kGateSlot, sizeof(uint64_t),
                                  cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(c->h_result + 1, c->s.result + 1, nr * sizeof(uint64_t),
                        cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return set_error(SEL_E_CUDA, cuda_msg("cudaMemcpyAsync (execute)", e));
  return SEL_OK;
}

// Outputs of a completed device-gated Execute from the pinned result mirror.
uint64_t execute_outputs(sel_ctx c, uint64_t max_size, uint64_t* out_local_count,
                         uint64_t* out_global_offset, int* out_materialized) {
  const uint64_t count = c->h_result[kGateSlot];
  if (count > max_size) return count;  // "throw exception": nothing written
  const int nr = multi(c) ? c->nranks : 0;
  uint64_t local = c->h_result[kGateSlot - 1], offset = 0;   // the mirrors (enqueue_execute)
  if (nr > 0) {
    const uint64_t* v = c->h_result + (nr <= kMirrorMax ? kGateSlot - nr : 1);
    for (int r2 = 0; r2 < c->rank; ++r2) offset += v[r2];
    local = v[c->rank];
  }
  if (out_local_count) *out_local_count = local;
  if (out_global_offset) *out_global_offset = offset;
  if (out_materialized) *out_materialized = 1;
  return count;
}

sel_status check_projection(sel_table t, const uint32_t* proj_cols, uint32_t nproj,
                            uint32_t* out_rowids, void* const* out_cols, uint64_t capacity_rows) {
  if (nproj > 0 && !proj_cols) return set_error(SEL_E_ARG, "null proj_cols");
  if (nproj > 255) return set_error(SEL_E_ARG, "nproj must be <= 255");
  for (uint32_t j = 0; j < nproj; ++j)
    if (proj_cols[j] >= t->cols.size()) return set_error(SEL_E_ARG, "projection index out of range");
  if (capacity_rows > 0) {
    if (!out_rowids) return set_error(SEL_E_ARG, "null out_rowids with capacity > 0");
    if (nproj > 0 && !out_cols) return set_error(SEL_E_ARG, "null out_cols with capacity > 0");
    for (uint32_t j = 0; j < nproj; ++j)
      if (!out_cols[j]) return set_error(SEL_E_ARG, "null out_cols entry with capacity > 0");
  }
  return SEL_OK;
}

}  // namespace

extern "C" {

uint64_t sel_count_ex(sel_table t, const void* prog, size_t prog_bytes, uint32_t flags,
                      const uint32_t* keep_cols, uint32_t nkeep, void* cuda_stream) {
  clear_error();
  if (flags & ~SEL_KEEP_SELECTION) return fail64(SEL_E_ARG, "unknown flags");
  if (nkeep > 0 && !keep_cols) return fail64(SEL_E_ARG, "null keep_cols");
  if (t)
    for (uint32_t j = 0; j < nkeep; ++j)
      if (keep_cols[j] >= t->cols.size()) return fail64(SEL_E_ARG, "keep column index out of range");
  if (!t) return fail64(SEL_E_ARG, "null table");
  sel_ctx c = t->ctx;
  if (c->destroyed) return fail64(SEL_E_STATE, "context destroyed");
  Plan plan;
  if (plan_for(t, prog, prog_bytes, &plan) != SEL_OK) return SEL_ERR;
  cudaStream_t stream = (cudaStream_t)cuda_stream;
  DeviceGuard g(c->device);
  if (!g.ok) return fail64(SEL_E_CUDA, "cudaSetDevice failed");
  c->last_ms = 0.f;
  const uint64_t n = t->local_rows;
  const bool scan = n > 0 && plan.path != PATH_CONST;
  if ((flags & SEL_KEEP_SELECTION) && !scan) c->kept_table = nullptr;
  if (!scan && !multi(c)) return plan.path == PATH_CONST && plan.const_value ? n : 0;
  // without an NCCL all-reduce after it the count kernel stores the count into the pinned host
  // word itself (ExecFinish::host); otherwise one 8-byte copy follows the collective
  const bool direct = scan && !(c->comm && !c->peers);
  const ExecFinish fin{nullptr, c->h_result_dev, 0, c->rank};
  if (enqueue_count(t, plan, flags, keep_cols, nkeep, stream, c->s.result, true, nullptr, 0,
                    direct ? &fin : nullptr) != SEL_OK)
    return SEL_ERR;
  cudaError_t e = direct ? cudaSuccess
                         : cudaMemcpyAsync(c->h_result, c->s.result, sizeof(uint64_t),
                                           cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = sync_stream(c, stream);
  if (e != cudaSuccess) return fail64(sync_code(e), cuda_msg("count result", e));
  if (peer_status(c) != SEL_OK) return SEL_ERR;
  if (scan && c->timing) {
    cudaEventElapsedTime(&c->last_ms, c->ev0, c->ev1);
    c->last_count_ms = c->last_ms;
  }
  if (scan && (flags & SEL_KEEP_SELECTION)) {
    c->kept_table = t;
    c->kept_prog.assign(static_cast<const char*>(prog), prog_bytes);
  }
  return c->h_result[0];
}

sel_status sel_count_async(sel_table t, const void* prog, size_t prog_bytes, uint64_t* d_out,
                           void* cuda_stream) {
  clear_error();
  if (!t || !d_out) return set_error(SEL_E_ARG, "null argument");
  sel_ctx c = t->ctx;
  if (c->destroyed) return set_error(SEL_E_STATE, "context destroyed");
  Plan plan;
  if (plan_for(t, prog, prog_bytes, &plan) != SEL_OK) return g_status;
  cudaStream_t stream = (cudaStream_t)cuda_stream;
  DeviceGuard g(c->device);
  if (!g.ok) return set_error(SEL_E_CUDA, "cudaSetDevice failed");
  const uint64_t n = t->local_rows;
  if (n == 0 || plan.path == PATH_CONST) {  // no scan: the local value by a device-side store
    const int le = launch_set_u64(d_out, plan.path == PATH_CONST && plan.const_value ? n : 0, stream);
    if (le != cudaSuccess) return set_error(SEL_E_CUDA, cuda_msg("launch", (cudaError_t)le));
    if (c->peers) {
      const int le2 = launch_peer_exchange(c->xg, d_out, 1, nullptr, d_out, stream);
      if (le2 != cudaSuccess) return set_error(SEL_E_CUDA, cuda_msg("peer exchange", (cudaError_t)le2));
    } else if (c->comm) {
      ncclResult_t r = nccl().AllReduce(d_out, d_out, 1, ncclUint64, ncclSum, c->comm, stream);
      if (r != ncclSuccess) return set_error(SEL_E_NCCL, nccl_msg("ncclAllReduce", r));
    }
    return SEL_OK;
  }
  return enqueue_count(t, plan, 0u, nullptr, 0u, stream, d_out);
}

}  // extern "C"

namespace {

// sel_pushdown's body. collective = false: no all-gather — the local count is returned (and
// *out_global_offset left 0); sel_execute's host-gated path has gathered the counts already.
uint64_t pushdown_impl(sel_table t, const void* prog, size_t prog_bytes, const uint32_t* proj_cols,
                       uint32_t nproj, uint32_t* out_rowids, void* const* out_cols,
                       uint64_t capacity_rows, uint64_t* out_local_count,
                       uint64_t* out_global_offset, void* cuda_stream, bool collective) {
  if (!t) return fail64(SEL_E_ARG, "null table");
  sel_ctx c = t->ctx;
  if (c->destroyed) return fail64(SEL_E_STATE, "context destroyed");
  if (check_projection(t, proj_cols, nproj, out_rowids, out_cols, capacity_rows) != SEL_OK)
    return SEL_ERR;
  Plan plan;
  if (plan_for(t, prog, prog_bytes, &plan) != SEL_OK) return SEL_ERR;
  cudaStream_t stream = (cudaStream_t)cuda_stream;
  DeviceGuard g(c->device);
  if (!g.ok) return fail64(SEL_E_CUDA, "cudaSetDevice failed");
  c->last_ms = 0.f;
  const uint64_t n = t->local_rows;
  const bool scan = n > 0 && !(plan.path == PATH_CONST && !plan.const_value);
  c->last_pd_path = -1;
  cudaError_t e;
  bool two_pass = false;
  if (scan) {
    const uint64_t ntiles = (n + kChunkRows - 1) / kChunkRows;
    if (ensure_status(c, ntiles, stream) != SEL_OK) return SEL_ERR;
    if (++c->epoch >= (1u << 30)) {
      e = cudaMemsetAsync(c->s.status, 0, c->s.status_cap * sizeof(uint64_t), stream);
      if (e != cudaSuccess) return fail64(SEL_E_CUDA, cuda_msg("cudaMemsetAsync(status)", e));
      c->epoch = 1;
    }
    const size_t nslots = count_slots(plan);
    auto fill = [&](auto* p) {
      pack(plan, t, p);
      p->row_offset = t->row_offset;
      p->capacity = capacity_rows;
      p->n_proj = capacity_rows > 0 ? nproj : 0;
      // Projected predicate columns are captured in shared memory while the predicate loads them
      // (no second read from HBM); the rest are gathered from global memory at write-out.
      std::vector<int> cap_off(t->cols.size(), -1);
      uint32_t off = kIdxBytes;
      const auto consts = const_columns(t, plan);
      for (uint32_t j = 0; j < p->n_proj; ++j) {
        const int c = (int)proj_cols[j];
        const uint32_t w = (uint32_t)width_of(t->types[c]);
        uint64_t raw = 0;
        if (is_const_col(consts, c, &raw)) {   // a fill: no capture, no gather
          p->proj_src[j] = reinterpret_cast<const void*>((uintptr_t)raw);
          p->proj_dst[j] = out_cols[j];
          p->proj_wclass[j] = wclass_of(t->types[c]);
          p->proj_cap_off[j] = kConstProj;
          continue;
        }
        bool pred_col = false;
        for (auto& L : plan.leaves) pred_col = pred_col || L.col == c;
        if (pred_col && cap_off[c] < 0 && off + w * kChunkRows <= kIdxBytes + kCaptureBudget) {
          cap_off[c] = (int)off;
          off += w * kChunkRows;
        }
        p->proj_src[j] = t->cols[c].data;
        p->proj_dst[j] = out_cols[j];
        p->proj_wclass[j] = wclass_of(t->types[c]);
        p->proj_cap_off[j] = cap_off[c] >= 0 ? (uint16_t)cap_off[c] : kNoCapture;
      }
      std::vector<bool> marked(t->cols.size(), false);
      for (size_t i = 0; i < plan.op.size(); ++i) {
        if (plan.op[i] != DOP_LEAF) continue;
        const int l = plan.arg[i];
        const int c = plan.leaves[l].col;
        if (cap_off[c] >= 0 && !marked[c]) {
          p->leaf[l].cap = 1;
          p->leaf[l].cap_off = (uint16_t)cap_off[c];
          marked[c] = true;
        }
      }
      p->warp_smem = (off + 15u) & ~15u;
    };
    const bool from_sel = !c->force_single && c->kept_table == t &&
                          c->kept_prog.size() == prog_bytes &&
                          std::memcmp(c->kept_prog.data(), prog, prog_bytes) == 0;
    // No kept selection: large shards take two passes — the count keeping the selection and the
    // projected predicate columns' values, then the materialisation from it (Algorithm 1's
    // count-then-execute order, without the gate) — instead of the single
    // pass, whose decoupled look-back waits dominate at this size.
    two_pass = !from_sel && !c->force_single && n >= c->two_pass_min_rows &&
               plan.path != PATH_CONST;  // TRUE runs no count kernel: nothing would be kept
    if (c->timing) cudaEventRecord(c->ev0, stream);
    int le, grid;
    if (two_pass) {
      if (enqueue_count(t, plan, SEL_KEEP_SELECTION, proj_cols, c->keep_values ? nproj : 0u, stream,
                        c->s.result + kGateSlot, false, proj_cols, nproj) != SEL_OK)
        return SEL_ERR;
      if (c->timing) cudaEventRecord(c->ev2, stream);
      if (enqueue_pushdown_sel(t, plan, proj_cols, nproj, out_rowids, out_cols, capacity_rows, false,
                               0, stream) != SEL_OK)
        return SEL_ERR;
      c->last_pd_path = 2;
      le = cudaSuccess;
    } else if (from_sel) {
      if (enqueue_pushdown_sel(t, plan, proj_cols, nproj, out_rowids, out_cols, capacity_rows, false,
                               0, stream) != SEL_OK)
        return SEL_ERR;
      le = cudaSuccess;
    } else if (fits_block<DevProgramSmall>(plan, nslots, nproj)) {
      DevProgramSmall p;
      fill(&p);
      grid = grid_for(c, (ntiles + kWarpsPerCta - 1) / kWarpsPerCta,
                      occupancy_pushdown_small((size_t)p.warp_smem * kWarpsPerCta));
      le = launch_pushdown_small(p, n, out_rowids, grid, c->s, c->ticket_base, c->epoch, stream);
    } else {
      static thread_local DevProgramLarge p;
      fill(&p);
      grid = grid_for(c, (ntiles + kWarpsPerCta - 1) / kWarpsPerCta,
                      occupancy_pushdown_large((size_t)p.warp_smem * kWarpsPerCta));
      le = launch_pushdown_large(p, n, out_rowids, grid, c->s, c->ticket_base, c->epoch, stream);
    }
    if (!from_sel && !two_pass) {
      if (le != cudaSuccess) {
        cudaMemsetAsync(c->s.ticket, 0, sizeof(unsigned long long), stream);
        c->ticket_base = 0;
        return fail64(SEL_E_CUDA, cuda_msg("push-down kernel launch", (cudaError_t)le));
      }
      c->ticket_base += ntiles + (uint64_t)grid * kWarpsPerCta;  // every warp draws one ticket past the last tile
      c->last_pd_path = 0;
    }
    if (c->timing) cudaEventRecord(c->ev1, stream);
  } else {
    c->h_result[0] = 0;
    if (multi(c) && collective) {
      e = cudaMemcpyAsync(c->s.result, c->h_result, sizeof(uint64_t), cudaMemcpyHostToDevice, stream);
      if (e != cudaSuccess) return fail64(SEL_E_CUDA, cuda_msg("cudaMemcpyAsync", e));
    }
  }
  uint64_t local = 0, offset = 0, total = 0;
  if (multi(c) && collective) {  // all-gather the per-rank counts, exclusive scan on the host
    if (c->peers) {
      const int le2 = launch_peer_exchange(c->xg, c->s.result, 1, c->s.result + 1, nullptr, stream);
      if (le2 != cudaSuccess) return fail64(SEL_E_CUDA, cuda_msg("peer exchange", (cudaError_t)le2));
    } else {
      ncclResult_t r = nccl().AllGather(c->s.result, c->s.result + 1, 1, ncclUint64, c->comm, stream);
      if (r != ncclSuccess) return fail64(SEL_E_NCCL, nccl_msg("ncclAllGather", r));
    }
    e = cudaMemcpyAsync(c->h_result + 1, c->s.result + 1, c->nranks * sizeof(uint64_t),
                        cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = sync_stream(c, stream);
    if (e != cudaSuccess) return fail64(sync_code(e), cuda_msg("push-down result", e));
    if (peer_status(c) != SEL_OK) return SEL_ERR;
    for (int r2 = 0; r2 < c->nranks; ++r2) {
      if (r2 < c->rank) offset += c->h_result[1 + r2];
      total += c->h_result[1 + r2];
    }
    local = c->h_result[1 + c->rank];
  } else {
    if (scan) {
      e = cudaMemcpyAsync(c->h_result, c->s.result, sizeof(uint64_t), cudaMemcpyDeviceToHost, stream);
      if (e == cudaSuccess) e = sync_stream(c, stream);
      if (e != cudaSuccess) return fail64(sync_code(e), cuda_msg("push-down result", e));
    }
    local = total = c->h_result[0];
  }
  if (scan && c->timing) {
    cudaEventElapsedTime(&c->last_ms, c->ev0, c->ev1);
    c->last_push_ms = c->last_ms;
    if (two_pass) {  // last_times: (keeping count, materialisation); last_ms: the whole call
      cudaEventElapsedTime(&c->last_count_ms, c->ev0, c->ev2);
      cudaEventElapsedTime(&c->last_push_ms, c->ev2, c->ev1);
    }
  }
  if (two_pass) {  // the selection this call kept serves a following push-down of the program
    c->kept_table = t;
    c->kept_prog.assign(static_cast<const char*>(prog), prog_bytes);
  }
  if (out_local_count) *out_local_count = local;
  if (out_global_offset) *out_global_offset = offset;
  return total;
}

}  // namespace

extern "C" {

uint64_t sel_pushdown(sel_table t, const void* prog, size_t prog_bytes, const uint32_t* proj_cols,
                      uint32_t nproj, uint32_t* out_rowids, void* const* out_cols,
                      uint64_t capacity_rows, uint64_t* out_local_count,
                      uint64_t* out_global_offset, void* cuda_stream) {
  clear_error();
  return pushdown_impl(t, prog, prog_bytes, proj_cols, nproj, out_rowids, out_cols, capacity_rows,
                       out_local_count, out_global_offset, cuda_stream, true);
}

sel_status sel_histogram(sel_table t, uint32_t col, uint32_t stride, uint32_t phase,
                         uint32_t nbuckets, int64_t* out_lo, int64_t* out_hi, uint64_t* out_rows,
                         uint64_t* out_distinct, uint64_t* out_sample_rows, void* cuda_stream) {
  clear_error();
  if (!t || !out_lo || !out_hi || !out_rows || !out_distinct) return set_error(SEL_E_ARG, "null argument");
  if (stride == 0 || phase >= stride) return set_error(SEL_E_ARG, "need stride >= 1 and phase < stride");
  if (nbuckets < 1 || nbuckets > 65536) return set_error(SEL_E_ARG, "nbuckets must be 1..65536");
  sel_ctx c = t->ctx;
  if (c->destroyed) return set_error(SEL_E_STATE, "context destroyed");
  if (col >= t->cols.size()) return set_error(SEL_E_ARG, "column index out of range");
  const int type = t->types[col];
  uint32_t flip;
  if (type == SEL_INT32 || type == SEL_DATE32) flip = 0x80000000u;
  else if (type == SEL_DICT8 || type == SEL_DICT16 || type == SEL_DICT32) flip = 0u;
  else return set_error(SEL_E_TYPE, "histograms take INT32, DATE32 and DICT columns");
  const uint64_t n = t->local_rows;
  const uint64_t nchunks = (n + kChunkRows - 1) / kChunkRows;
  const uint64_t nsamp = nchunks > phase ? (nchunks - phase + stride - 1) / stride : 0;
  uint64_t m = nsamp * kChunkRows;
  if (nsamp > 0) {   // the last sampled chunk may be the table's partial tail
    const uint64_t last = phase + (nsamp - 1) * (uint64_t)stride;
    m -= kChunkRows - std::min<uint64_t>(kChunkRows, n - last * kChunkRows);
  }
  if (m >= (1ull << 31)) return set_error(SEL_E_TOO_LARGE, "sample of 2^31 rows or more");
  if (out_sample_rows) *out_sample_rows = m;
  cudaStream_t stream = (cudaStream_t)cuda_stream;
  DeviceGuard g(c->device);
  if (!g.ok) return set_error(SEL_E_CUDA, "cudaSetDevice failed");
  const size_t tb = histogram_temp_bytes(std::max<uint64_t>(m, 1));
  const size_t kb = std::max<uint64_t>(m, 1) * sizeof(uint32_t);
  const size_t ob = (size_t)nbuckets * (2 * sizeof(uint32_t) + 2 * sizeof(uint64_t));
  const size_t need = 2 * kb + tb + ob + 64;
  cudaError_t e = cudaSuccess;
  if (c->hist_cap < need) {   // grows only (kept by the context for the next histogram)
    e = sync_stream(c, stream);
    if (e == cudaSuccess && c->hist_buf) e = cudaFree(c->hist_buf);
    c->hist_buf = nullptr;
    c->hist_cap = 0;
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&c->hist_buf), need);
    if (e != cudaSuccess) return set_error(SEL_E_CUDA, cuda_msg("cudaMalloc(histogram)", e));
    c->hist_cap = need;
  }
  char* buf = c->hist_buf;
  uint32_t* keys = reinterpret_cast<uint32_t*>(buf);
  uint32_t* sorted = keys + kb / sizeof(uint32_t);
  uint64_t* rows = reinterpret_cast<uint64_t*>(buf + ((2 * kb + 7) & ~size_t(7)));
  uint64_t* distinct = rows + nbuckets;
  uint32_t* lo = reinterpret_cast<uint32_t*>(distinct + nbuckets);
  uint32_t* hi = lo + nbuckets;
  void* temp = hi + nbuckets + 16;
  int le = launch_histogram(t->cols[col].data, wclass_of(type), flip, n, stride, phase, nsamp, m,
                            nbuckets, keys, sorted, temp, tb, lo, hi, rows, distinct, stream);
  std::vector<uint32_t> hlo(nbuckets), hhi(nbuckets);
  e = (cudaError_t)le;
  if (e == cudaSuccess) e = cudaMemcpyAsync(out_rows, rows, nbuckets * sizeof(uint64_t), cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(out_distinct, distinct, nbuckets * sizeof(uint64_t), cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(hlo.data(), lo, nbuckets * sizeof(uint32_t), cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(hhi.data(), hi, nbuckets * sizeof(uint32_t), cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = sync_stream(c, stream);
  if (e != cudaSuccess) return set_error(sync_code(e), cuda_msg("histogram", e));
  for (uint32_t b = 0; b < nbuckets; ++b) {   // keys back to values; an empty bucket reports 0, 0
    const uint32_t l = hlo[b] ^ flip, h = hhi[b] ^ flip;
    out_lo[b] = out_rows[b] == 0 ? 0 : (flip ? (int64_t)(int32_t)l : (int64_t)l);
    out_hi[b] = out_rows[b] == 0 ? 0 : (flip ? (int64_t)(int32_t)h : (int64_t)h);
  }
  return SEL_OK;
}

uint64_t sel_count_sampled(sel_table t, const void* prog, size_t prog_bytes, uint32_t stride,
                           uint32_t phase, uint64_t* out_sample_rows, void* cuda_stream) {
  clear_error();
  if (!t) return fail64(SEL_E_ARG, "null table");
  if (stride == 0 || phase >= stride) return fail64(SEL_E_ARG, "need stride >= 1 and phase < stride");
  sel_ctx c = t->ctx;
  if (c->destroyed) return fail64(SEL_E_STATE, "context destroyed");
  Plan plan;
  if (plan_for(t, prog, prog_bytes, &plan) != SEL_OK) return SEL_ERR;
  cudaStream_t stream = (cudaStream_t)cuda_stream;
  DeviceGuard g(c->device);
  if (!g.ok) return fail64(SEL_E_CUDA, "cudaSetDevice failed");
  const uint64_t n = t->local_rows;
  const uint64_t nfull = n / kChunkRows, rem = n % kChunkRows;
  const uint64_t ns_full = nfull > phase ? (nfull - phase + stride - 1) / stride : 0;
  const bool tail = rem != 0 && nfull >= phase && (nfull - phase) % stride == 0;
  const uint64_t sample_rows = ns_full * kChunkRows + (tail ? rem : 0);
  const bool scan = sample_rows > 0 && plan.path != PATH_CONST;
  uint64_t local = scan ? 0 : (plan.path == PATH_CONST && plan.const_value ? sample_rows : 0);
  cudaError_t e;
  if (scan) {
    const uint64_t units = (ns_full + 1 + kWarpsPerCta - 1) / kWarpsPerCta;
    const size_t nslots = count_slots(plan);
    int le;
    if (fits_block<DevProgramSmall>(plan, nslots, 0)) {
      DevProgramSmall p;
      pack(plan, t, &p);
      p.chunk_stride = stride;
      p.chunk_phase = phase;
      choose_bitmap_staging(&p, 0);
      int occ = p.bm_smem ? occupancy_count_dyn_small(p.bm_smem) : c->occ_count_small;
      if (p.fast_n && !p.bm_smem) occ = occupancy_count_fast((int)p.fast_n, false, 0);
      const int nw = pick_count_warps(c, p, 0, occ);
      le = launch_count_small(p, n, grid_for(c, nw == kWarpsPerCta ? units : (ns_full + nw) / nw,
                                             nw == kWarpsPerCta ? occ : 1), c->s, nullptr, stream, nw);
    } else {
      static thread_local DevProgramLarge p;
      pack(plan, t, &p);
      p.chunk_stride = stride;
      p.chunk_phase = phase;
      choose_bitmap_staging(&p, 0);
      const int occ = p.bm_smem ? occupancy_count_dyn_large(p.bm_smem) : c->occ_count_large;
      const int nw = pick_count_warps(c, p, 0, occ);
      le = launch_count_large(p, n, grid_for(c, nw == kWarpsPerCta ? units : (ns_full + nw) / nw,
                                             nw == kWarpsPerCta ? occ : 1), c->s, nullptr, stream, nw);
    }
    if (le != cudaSuccess) return fail64(SEL_E_CUDA, cuda_msg("sampled count launch", (cudaError_t)le));
  } else {
    c->h_result[0] = local;
    e = cudaMemcpyAsync(c->s.result, c->h_result, sizeof(uint64_t), cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) return fail64(SEL_E_CUDA, cuda_msg("cudaMemcpyAsync", e));
  }
  c->h_result[1] = sample_rows;
  e = cudaMemcpyAsync(c->s.result + 1, c->h_result + 1, sizeof(uint64_t), cudaMemcpyHostToDevice, stream);
  if (e != cudaSuccess) return fail64(SEL_E_CUDA, cuda_msg("cudaMemcpyAsync", e));
  if (c->peers) {
    const int le2 = launch_peer_exchange(c->xg, c->s.result, 2, nullptr, c->s.result, stream);
    if (le2 != cudaSuccess) return fail64(SEL_E_CUDA, cuda_msg("peer exchange", (cudaError_t)le2));
  } else if (c->comm) {
    ncclResult_t r = nccl().AllReduce(c->s.result, c->s.result, 2, ncclUint64, ncclSum, c->comm, stream);
    if (r != ncclSuccess) return fail64(SEL_E_NCCL, nccl_msg("ncclAllReduce(sampled)", r));
  }
  e = cudaMemcpyAsync(c->h_result, c->s.result, 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = sync_stream(c, stream);
  if (e != cudaSuccess) return fail64(sync_code(e), cuda_msg("sampled count result", e));
  if (peer_status(c) != SEL_OK) return SEL_ERR;
  if (out_sample_rows) *out_sample_rows = c->h_result[1];
  return c->h_result[0];
}

sel_status sel_count_batch(sel_table t, const void* const* progs, const size_t* prog_bytes,
                           uint32_t nprog, uint64_t* out_counts, void* cuda_stream) {
  clear_error();
  if (!t || !progs || !prog_bytes || !out_counts) return set_error(SEL_E_ARG, "null argument");
  if (nprog == 0 || nprog > (uint32_t)kBatchMaxProgs) return set_error(SEL_E_ARG, "nprog must be 1..32");
  sel_ctx c = t->ctx;
  if (c->destroyed) return set_error(SEL_E_STATE, "context destroyed");
  std::vector<Plan> plans(nprog);
  for (uint32_t k = 0; k < nprog; ++k) {
    if (plan_for(t, progs[k], prog_bytes[k], &plans[k]) != SEL_OK) return g_status;
    for (auto& L : plans[k].leaves)
      if (L.bitmap >= 0) return set_error(SEL_E_ARG, "IN_BITMAP leaves are not batched");
  }
  // distinct leaves, grouped by column (first-appearance order)
  std::vector<int> col_order;
  std::map<int, std::vector<std::vector<Interval>>> by_col;
  auto leaf_key = [&](const PlanLeaf& L) -> std::pair<int, int> {
    auto& lst = by_col[L.col];
    if (lst.empty()) col_order.push_back(L.col);
    for (size_t i = 0; i < lst.size(); ++i) {
      if (lst[i].size() == L.iv.size() &&
          std::equal(lst[i].begin(), lst[i].end(), L.iv.begin(),
                     [](const Interval& x, const Interval& y) { return x.lo == y.lo && x.hi == y.hi; }))
        return {L.col, (int)i};
    }
    lst.push_back(L.iv);
    return {L.col, (int)lst.size() - 1};
  };
  std::vector<std::vector<std::pair<int, int>>> prog_leaf(nprog);
  for (uint32_t k = 0; k < nprog; ++k)
    for (auto& L : plans[k].leaves) prog_leaf[k].push_back(leaf_key(L));
  static thread_local BatchProgram bp;
  std::memset(&bp, 0, sizeof(bp));
  std::map<std::pair<int, int>, int> leaf_id;
  uint32_t nl = 0, niv = 0;
  for (int col : col_order) {
    if (bp.n_cols >= (uint32_t)kBatchMaxCols) return set_error(SEL_E_ARG, "batch exceeds 32 columns");
    BatchColumn& C = bp.col[bp.n_cols++];
    const int type = t->types[col];
    C.data = t->cols[col].data;
    C.wclass = wclass_of(type);
    C.fkey = type == SEL_FLOAT32 ? 1 : 0;
    C.leaf_begin = (uint16_t)nl;
    const uint64_t bias = key_sign_bias(type);
    auto& lst = by_col[col];
    for (size_t i = 0; i < lst.size(); ++i) {
      if (nl >= (uint32_t)kBatchMaxLeaves) return set_error(SEL_E_ARG, "batch exceeds 32 distinct leaves");
      if (niv + lst[i].size() > 1024) return set_error(SEL_E_ARG, "batch exceeds 1024 intervals");
      leaf_id[{col, (int)i}] = (int)nl;
      bp.leaf_iv_begin[nl] = (uint16_t)niv;
      bp.leaf_iv_count[nl] = (uint16_t)lst[i].size();
      for (const Interval& x : lst[i]) {
        bp.lo[niv] = x.lo ^ bias;
        bp.span[niv] = x.hi - x.lo;
        ++niv;
      }
      ++nl;
    }
    C.leaf_count = (uint16_t)(nl - C.leaf_begin);
  }
  bp.n_leaves = nl;
  uint32_t nop = 0;
  std::vector<bool> host_zero(nprog, false);
  for (uint32_t k = 0; k < nprog; ++k) {
    const Plan& P = plans[k];
    if (P.path == PATH_CONST && !P.const_value) { host_zero[k] = true; continue; }  // FALSE: 0
    if (nop + P.op.size() + 1 > sizeof(bp.op)) return set_error(SEL_E_ARG, "batch exceeds 512 ops");
    for (size_t i = 0; i < P.op.size(); ++i) {
      bp.op[nop] = P.op[i];
      bp.arg[nop] = P.op[i] == DOP_LEAF ? (uint8_t)leaf_id[prog_leaf[k][P.arg[i]]] : 0;
      ++nop;
    }
    bp.op[nop] = DOP_EMIT;   // TRUE (no ops) emits the all-ones mask
    bp.arg[nop] = (uint8_t)k;
    ++nop;
  }
  bp.n_ops = nop;
  bp.n_progs = nprog;
  bp.all_conj = 1;
  bp.prog_live = 0;
  for (uint32_t k = 0; k < nprog; ++k) {
    const Plan& P = plans[k];
    bp.conj_set[k] = 0;
    if (host_zero[k]) continue;
    bp.prog_live |= 1u << k;
    if (P.path == PATH_CONST) continue;               // TRUE: every row
    if (P.path != PATH_CONJ) { bp.all_conj = 0; continue; }
    for (size_t i = 0; i < P.op.size(); ++i)
      if (P.op[i] == DOP_LEAF) bp.conj_set[k] |= 1u << leaf_id[prog_leaf[k][P.arg[i]]];
  }
  cudaStream_t stream = (cudaStream_t)cuda_stream;
  DeviceGuard g(c->device);
  if (!g.ok) return set_error(SEL_E_CUDA, "cudaSetDevice failed");
  const uint64_t n = t->local_rows;
  uint64_t* d_out = c->s.result + 1;
  cudaError_t e = cudaMemsetAsync(d_out, 0, nprog * sizeof(uint64_t), stream);
  if (e != cudaSuccess) return set_error(SEL_E_CUDA, cuda_msg("cudaMemsetAsync(batch)", e));
  if (n > 0 && nop > 0) {
    const uint64_t nchunks = (n + kChunkRows - 1) / kChunkRows;
    const uint64_t units = (nchunks + kWarpsPerCta - 1) / kWarpsPerCta;
    if (c->timing) cudaEventRecord(c->ev0, stream);
    const int le = launch_count_batch(bp, n, grid_for(c, units, occupancy_count_batch()), d_out, stream);
    if (le != cudaSuccess) return set_error(SEL_E_CUDA, cuda_msg("batch kernel launch", (cudaError_t)le));
    if (c->timing) cudaEventRecord(c->ev1, stream);
  }
  if (c->peers) {
    const int le2 = launch_peer_exchange(c->xg, d_out, (int)nprog, nullptr, d_out, stream);
    if (le2 != cudaSuccess) return set_error(SEL_E_CUDA, cuda_msg("peer exchange", (cudaError_t)le2));
  } else if (c->comm) {
    ncclResult_t r = nccl().AllReduce(d_out, d_out, nprog, ncclUint64, ncclSum, c->comm, stream);
    if (r != ncclSuccess) return set_error(SEL_E_NCCL, nccl_msg("ncclAllReduce(batch)", r));
  }
  e = cudaMemcpyAsync(c->h_result + 1, d_out, nprog * sizeof(uint64_t), cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = sync_stream(c, stream);
  if (e != cudaSuccess) return set_error(sync_code(e), cuda_msg("batch result", e));
  if (peer_status(c) != SEL_OK) return g_status;
  if (n > 0 && nop > 0 && c->timing) {
    cudaEventElapsedTime(&c->last_ms, c->ev0, c->ev1);
    c->last_count_ms = c->last_ms;
  }
  for (uint32_t k = 0; k < nprog; ++k) out_counts[k] = c->h_result[1 + k];  // FALSE programs stay 0
  return SEL_OK;
}

// sel_execute and sel_execute_to (global_out: the outputs are the global result; each rank
// writes at its offset in it).
static uint64_t execute_impl(sel_table t, const void* prog, size_t prog_bytes,
                             const uint32_t* proj_cols, uint32_t nproj, uint64_t max_size,
                             uint32_t* out_rowids, void* const* out_cols, uint64_t capacity_rows,
                             uint64_t* out_local_count, uint64_t* out_global_offset,
                             int* out_materialized, void* cuda_stream, bool global_out) {
  clear_error();
  if (out_materialized) *out_materialized = 0;
  if (out_local_count) *out_local_count = 0;
  if (out_global_offset) *out_global_offset = 0;
  if (!t) return fail64(SEL_E_ARG, "null table");
  sel_ctx c = t->ctx;
  if (c->destroyed) return fail64(SEL_E_STATE, "context destroyed");
  if (check_projection(t, proj_cols, nproj, out_rowids, out_cols, capacity_rows) != SEL_OK)
    return SEL_ERR;
  Plan plan;
  if (plan_for(t, prog, prog_bytes, &plan) != SEL_OK) return SEL_ERR;
  // Execute(isSPD): gamma_COUNT over the compound, keeping what the materialisation reuses: the
  // selection (SEL_KEEP_VALUES=1: also the projected predicate columns' values — measured equal
  // or slower on every config).
  // With a communicator every Execute issues exactly one collective, an all-gather of the
  // per-rank counts (their sum is the global count the gate compares; their exclusive prefix
  // the rank's offset), on both paths below, so ranks on different paths stay matched.
  const uint32_t nkeep = c->keep_values ? nproj : 0u;
  const bool scan = t->local_rows > 0 && plan.path != PATH_CONST;
  if (!scan || c->force_single) {  // host-side gate: count, then (maybe) the push-down
    uint64_t local;
    if (multi(c)) {
      local = scan ? 0 : (plan.path == PATH_CONST && plan.const_value ? t->local_rows : 0);
      if (scan) {
        cudaStream_t stream = (cudaStream_t)cuda_stream;
        DeviceGuard g(c->device);
        if (!g.ok) return fail64(SEL_E_CUDA, "cudaSetDevice failed");
        if (enqueue_count(t, plan, SEL_KEEP_SELECTION, proj_cols, nkeep, stream, c->s.result,
                          false, proj_cols, nproj) != SEL_OK)
          return SEL_ERR;
        cudaError_t e = cudaMemcpyAsync(c->h_result, c->s.result, sizeof(uint64_t),
                                        cudaMemcpyDeviceToHost, stream);
        if (e == cudaSuccess) e = sync_stream(c, stream);
        if (e != cudaSuccess) return fail64(sync_code(e), cuda_msg("count result", e));
        local = c->h_result[0];
        c->kept_table = t;
        c->kept_prog.assign(static_cast<const char*>(prog), prog_bytes);
      }
      if (gather_counts(c, local, cuda_stream) != SEL_OK) return SEL_ERR;
    } else {
      local = sel_count_ex(t, prog, prog_bytes, SEL_KEEP_SELECTION, proj_cols, nkeep, cuda_stream);
      if (local == SEL_ERR) return SEL_ERR;
    }
    uint64_t count = local, offset = 0;
    if (multi(c)) {
      count = 0;
      for (int r2 = 0; r2 < c->nranks; ++r2) {
        if (r2 < c->rank) offset += c->h_result[1 + r2];
        count += c->h_result[1 + r2];
      }
    }
    if (count > max_size) return count;  // "throw exception": nothing written
    uint32_t* ids = out_rowids;
    std::vector<void*> cols(out_cols, out_cols + (out_cols ? nproj : 0));
    uint64_t cap = capacity_rows;
    if (global_out && offset > 0) {   // this rank's slice of the global result
      cap = capacity_rows > offset ? capacity_rows - offset : 0;
      if (cap > 0) {
        ids = out_rowids + offset;
        for (uint32_t j = 0; j < nproj; ++j)
          cols[j] = static_cast<char*>(cols[j]) + offset * (uint64_t)width_of(t->types[proj_cols[j]]);
      }
    }
    const uint64_t r = pushdown_impl(t, prog, prog_bytes, proj_cols, nproj, ids,
                                     cols.empty() ? nullptr : cols.data(), cap, out_local_count,
                                     nullptr, cuda_stream, false);
    if (r == SEL_ERR) return SEL_ERR;
    if (out_global_offset) *out_global_offset = offset;
    if (out_materialized) *out_materialized = 1;
    return count;
  }
  // Device-side gate (PAPER.md:393-400 in one stream, one host synchronisation): count keeping
  // the selection -> global count into result[kGateSlot] (without a communicator the count
  // itself; with one, the sum of the all-gathered per-rank counts) -> the push-down kernels
  // read it and write nothing if count > maxSize -> one D2H.
  cudaStream_t stream = (cudaStream_t)cuda_stream;
  DeviceGuard g(c->device);
  if (!g.ok) return fail64(SEL_E_CUDA, "cudaSetDevice failed");
  c->last_ms = 0.f;
  c->last_pd_path = -1;
  sel_status st = enqueue_execute(t, plan, proj_cols, nproj, nkeep, max_size, out_rowids, out_cols,
                                  capacity_rows, stream, global_out);
  if (st != SEL_OK) return SEL_ERR;
  cudaError_t e = sync_stream(c, stream);
  if (e != cudaSuccess) return fail64(sync_code(e), cuda_msg("execute result", e));
  if (peer_status(c) != SEL_OK) return SEL_ERR;
  c->kept_table = t;
  c->kept_prog.assign(static_cast<const char*>(prog), prog_bytes);
  if (c->timing) {
    cudaEventElapsedTime(&c->last_count_ms, c->ev0, c->ev1);
    cudaEventElapsedTime(&c->last_push_ms, c->ev2, c->ev3);
    c->last_ms = c->last_push_ms;
  }
  return execute_outputs(c, max_size, out_local_count, out_global_offset, out_materialized);
}

uint64_t sel_execute(sel_table t, const void* prog, size_t prog_bytes, const uint32_t* proj_cols,
                     uint32_t nproj, uint64_t max_size, uint32_t* out_rowids,
                     void* const* out_cols, uint64_t capacity_rows, uint64_t* out_local_count,
                     uint64_t* out_global_offset, int* out_materialized, void* cuda_stream) {
  return execute_impl(t, prog, prog_bytes, proj_cols, nproj, max_size, out_rowids, out_cols,
                      capacity_rows, out_local_count, out_global_offset, out_materialized,
                      cuda_stream, false);
}

uint64_t sel_execute_to(sel_table t, const void* prog, size_t prog_bytes, const uint32_t* proj_cols,
                        uint32_t nproj, uint64_t max_size, uint32_t* out_rowids,
                        void* const* out_cols, uint64_t capacity_rows, uint64_t* out_local_count,
                        uint64_t* out_global_offset, int* out_materialized, void* cuda_stream) {
  return execute_impl(t, prog, prog_bytes, proj_cols, nproj, max_size, out_rowids, out_cols,
                      capacity_rows, out_local_count, out_global_offset, out_materialized,
                      cuda_stream, true);
}

}  // extern "C"

namespace {

// (Re)build a prepared execute: plan (validating bitmap ids), reserve device memory outside the
// capture, then capture the one-synchronisation Execute sequence of sel_execute into a graph.
sel_status capture_prepared(sel_prepared q) {
  sel_table t = q->t;
  sel_ctx c = t->ctx;
  if (q->exec) cudaGraphExecDestroy(q->exec);
  q->exec = nullptr;
  q->graph = false;
  Plan plan;
  if (plan_for(t, q->prog.data(), q->prog.size(), &plan) != SEL_OK) return g_status;
  q->alloc_gen = c->alloc_gen;
  q->bm_gen = c->bm_gen;
  q->timing = c->timing;
  q->comm = c->comm;
  // With a communicator the two collectives are captured too (NCCL operations are capturable);
  // SEL_GRAPH_COMM=0 keeps those executes uncaptured.
  if (t->local_rows == 0 || plan.path == PATH_CONST || c->force_single ||
      (c->comm && !c->graph_comm))
    return SEL_OK;
  DeviceGuard g(c->device);
  if (!g.ok) return set_error(SEL_E_CUDA, "cudaSetDevice failed");
  const uint32_t nproj = (uint32_t)q->proj.size();
  const uint32_t nkeep = c->keep_values ? nproj : 0u;
  const uint32_t* proj = nproj ? q->proj.data() : nullptr;
  void* const* outs = nproj ? q->out_cols.data() : nullptr;
  const uint64_t nchunks = (t->local_rows + kChunkRows - 1) / kChunkRows;
  uint32_t off = kIdxBytes;
  if (reserve_selection(t, nchunks, choose_kept(t, plan, proj, nkeep, &off)) != SEL_OK) return g_status;
  q->alloc_gen = c->alloc_gen;
  cudaStream_t s = c->cap_stream;
  cudaError_t e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) return set_error(SEL_E_CUDA, cuda_msg("cudaStreamBeginCapture", e));
  c->capturing = true;
  sel_status st = enqueue_execute(t, plan, proj, nproj, nkeep, q->max_size, q->out_rowids, outs,
                                  q->capacity, s);
  c->capturing = false;
  cudaGraph_t graph = nullptr;
  e = cudaStreamEndCapture(s, &graph);
  if (st == SEL_OK && e != cudaSuccess) st = set_error(SEL_E_CUDA, cuda_msg("cudaStreamEndCapture", e));
  if (st == SEL_OK) {
    e = cudaGraphInstantiate(&q->exec, graph, 0);
    if (e != cudaSuccess) {
      q->exec = nullptr;
      st = set_error(SEL_E_CUDA, cuda_msg("cudaGraphInstantiate", e));
    }
  }
  if (graph) cudaGraphDestroy(graph);
  c->kept_table = nullptr;  // the capture only configured the kept-selection bookkeeping
  q->kept_cols = c->kept_cols;
  q->sel = c->sel;
  q->graph = st == SEL_OK;
  return st;
}

}  // namespace

extern "C" {

sel_status sel_prepare_execute(sel_table t, const void* prog, size_t prog_bytes,
                               const uint32_t* proj_cols, uint32_t nproj, uint64_t max_size,
                               uint32_t* out_rowids, void* const* out_cols,
                               uint64_t capacity_rows, sel_prepared* out) {
  clear_error();
  if (!out) return set_error(SEL_E_ARG, "null out");
  *out = nullptr;
  if (!t) return set_error(SEL_E_ARG, "null table");
  if (!prog) return set_error(SEL_E_PROGRAM, "program shorter than its header");
  if (t->ctx->destroyed) return set_error(SEL_E_STATE, "context destroyed");
  if (check_projection(t, proj_cols, nproj, out_rowids, out_cols, capacity_rows) != SEL_OK)
    return g_status;
  sel_prepared q = new sel_prepared_s();
  q->t = t;
  q->prog.assign(static_cast<const char*>(prog), prog_bytes);
  q->proj.assign(proj_cols, proj_cols + nproj);
  if (out_cols) q->out_cols.assign(out_cols, out_cols + nproj);
  else q->out_cols.assign(nproj, nullptr);
  q->out_rowids = out_rowids;
  q->max_size = max_size;
  q->capacity = capacity_rows;
  if (capture_prepared(q) != SEL_OK) {
    const sel_status st = g_status;
    if (q->exec) cudaGraphExecDestroy(q->exec);
    delete q;
    return st;
  }
  t->prepared.push_back(q);
  *out = q;
  return SEL_OK;
}

uint64_t sel_prepared_execute(sel_prepared q, uint64_t* out_local_count,
                              uint64_t* out_global_offset, int* out_materialized,
                              void* cuda_stream) {
  clear_error();
  if (out_materialized) *out_materialized = 0;
  if (out_local_count) *out_local_count = 0;
  if (out_global_offset) *out_global_offset = 0;
  if (!q) return fail64(SEL_E_ARG, "null prepared execute");
  if (!q->t) return fail64(SEL_E_STATE, "table released");
  sel_table t = q->t;
  sel_ctx c = t->ctx;
  if (c->destroyed) return fail64(SEL_E_STATE, "context destroyed");
  if (q->alloc_gen != c->alloc_gen || q->bm_gen != c->bm_gen || q->timing != c->timing ||
      q->comm != c->comm) {
    if (capture_prepared(q) != SEL_OK) return SEL_ERR;
  }
  if (!q->graph)
    return sel_execute(t, q->prog.data(), q->prog.size(), q->proj.empty() ? nullptr : q->proj.data(),
                       (uint32_t)q->proj.size(), q->max_size, q->out_rowids,
                       q->out_cols.empty() ? nullptr : q->out_cols.data(), q->capacity,
                       out_local_count, out_global_offset, out_materialized, cuda_stream);
  DeviceGuard g(c->device);
  if (!g.ok) return fail64(SEL_E_CUDA, "cudaSetDevice failed");
  cudaStream_t stream = (cudaStream_t)cuda_stream;
  c->kept_table = nullptr;
  cudaError_t e = cudaGraphLaunch(q->exec, stream);
  if (e == cudaSuccess) e = sync_stream(c, stream);
  if (e != cudaSuccess) return fail64(sync_code(e), cuda_msg("prepared execute", e));
  if (peer_status(c) != SEL_OK) return SEL_ERR;
  c->kept_table = t;
  c->kept_prog = q->prog;
  c->kept_cols = q->kept_cols;
  c->sel = q->sel;
  c->last_pd_path = 1;
  if (c->timing) {
    cudaEventElapsedTime(&c->last_count_ms, c->ev0, c->ev1);
    cudaEventElapsedTime(&c->last_push_ms, c->ev2, c->ev3);
    c->last_ms = c->last_push_ms;
  }
  return execute_outputs(c, q->max_size, out_local_count, out_global_offset, out_materialized);
}

void sel_prepared_release(sel_prepared q) {
  if (!q) return;
  if (q->t) {
    auto& v = q->t->prepared;
    v.erase(std::remove(v.begin(), v.end(), q), v.end());
  }
  if (q->exec) cudaGraphExecDestroy(q->exec);
  delete q;
}

}  // extern "C"

