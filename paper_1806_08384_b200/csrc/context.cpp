// context.cpp — libsel contexts (include/sel.h): device scratch, communicators (NCCL and the
// library's own peer exchange), exported/imported buffers, table registry, IN_BITMAP key sets,
// timing and error accessors.
#include "host.h"

#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <atomic>
#include <thread>

using namespace sel;

namespace sel {

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
std::string cuda_msg(const char* what, cudaError_t e) {
  if (e == kNcclAsyncFailed)
    return std::string(what) + ": NCCL asynchronous error (a rank failed; communicator aborted)";
  if (e == kSeqMissing)
    return std::string(what) + ": the stream drained without the Execute's result words";
  return std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
}

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

// Wait until the device-gated Execute enqueued after the host read `seq0` from the mirror's
// sequence word has stored its result words (finish_execute), not for the rest of the stream:
// the materialisation that follows keeps running. Errors as sync_stream; a stream that drains
// without the word changing (no Execute was enqueued) is kSeqMissing.
cudaError_t wait_result_seq(sel_ctx c, cudaStream_t s, uint64_t seq0) {
  volatile const uint64_t* w = c->h_result + kSeqSlot;
  for (unsigned spin = 0;; ++spin) {
    if (*w != seq0) {
      std::atomic_thread_fence(std::memory_order_acquire);
      return cudaSuccess;
    }
    if ((spin & 255u) != 255u) continue;
    const cudaError_t q = cudaStreamQuery(s);
    if (q == cudaSuccess) {
      if (*w != seq0) continue;
      return kSeqMissing;
    }
    if (q != cudaErrorNotReady) return q;
    if (c->comm && nccl().CommGetAsyncError) {
      ncclResult_t st = ncclSuccess;
      if (nccl().CommGetAsyncError(c->comm, &st) == ncclSuccess && st != ncclSuccess &&
          st != ncclInProgress) {
        if (nccl().CommAbort) nccl().CommAbort(c->comm);
        c->comm = nullptr;
        c->comm_failed = true;
        return kNcclAsyncFailed;
      }
    }
    if (spin > 4096) std::this_thread::yield();
  }
}

cudaStream_t ordered_stream(sel_ctx c, void* cuda_stream) {
  cudaStream_t s = (cudaStream_t)cuda_stream;
  if (c->async_pending && s != c->async_stream) {
    // not inside the caller's stream capture (an event recorded outside it cannot be waited on
    // there); a captured probe is ordered by the caller
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess) {
      (void)cudaGetLastError();   // e.g. the legacy stream while another thread captures: no wait
    } else if (cs == cudaStreamCaptureStatusNone) {
      cudaStreamWaitEvent(s, c->async_ev, 0);
    }
  }
  return s;
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

}  // namespace sel

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
  c->occ_small_max = c->occ_count_small;
  c->occ_large_max = c->occ_count_large;
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
              cudaMalloc(&c->s.result, kResultAlloc * sizeof(uint64_t)) == cudaSuccess &&
              cudaMalloc(&c->s.ticket, sizeof(unsigned long long)) == cudaSuccess &&
              cudaHostAlloc(&c->h_result, kResultAlloc * sizeof(uint64_t), cudaHostAllocMapped) == cudaSuccess &&
              cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->h_result_dev), c->h_result, 0) == cudaSuccess &&
              cudaMemset(c->s.done, 0, sizeof(unsigned int)) == cudaSuccess &&
              cudaMemset(c->s.ticket, 0, sizeof(unsigned long long)) == cudaSuccess &&
              cudaMemset(c->s.result, 0, kResultAlloc * sizeof(uint64_t)) == cudaSuccess &&
              (std::memset(c->h_result, 0, kResultAlloc * sizeof(uint64_t)), true) &&
              cudaEventCreateWithFlags(&c->async_ev, cudaEventDisableTiming) == cudaSuccess &&
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

}  // extern "C"

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
  if (c->async_ev) cudaEventDestroy(c->async_ev);
  c->async_ev = nullptr;
  c->async_pending = false;
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

extern "C" {

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

sel_status sel_ctx_set_option(sel_ctx ctx, const char* name, int64_t value) {
  clear_error();
  if (!ctx || !name) return set_error(SEL_E_ARG, "null argument");
  if (ctx->destroyed) return set_error(SEL_E_STATE, "context destroyed");
  const std::string k(name);
  const bool flag = value == 0 || value == 1;
  if (k == "fast" && flag) ctx->fast_enabled = value;
  else if (k == "coded" && flag) ctx->code_enabled = value;
  else if (k == "dense_split" && flag) ctx->dense_split = value;
  else if (k == "keep_values" && flag) ctx->keep_values = value;
  else if (k == "graph_comm" && flag) ctx->graph_comm = value;
  else if (k == "prefetch" && value >= -1 && value <= 1) ctx->prefetch_mode = (int)value;
  else if (k == "count_warps" && (value == 0 || value == kWarpsPerCta)) ctx->count_nw = (int)value;
  else if (k == "two_pass_min_rows" && value >= 0) {
    if (!ctx->force_single) ctx->two_pass_min_rows = (uint64_t)value;   // else: ignored (sel.h)
  }
  else if (k == "ctas_per_sm" && value >= 0) {
    ctx->occ_count_small = value ? std::min(ctx->occ_small_max, (int)value) : ctx->occ_small_max;
    ctx->occ_count_large = value ? std::min(ctx->occ_large_max, (int)value) : ctx->occ_large_max;
  } else {
    return set_error(SEL_E_ARG, "unknown option or value out of range: " + k);
  }
  // a kept selection was made under the old settings, and prepared executes baked them
  ctx->kept_table = nullptr;
  ++ctx->alloc_gen;
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

sel_status sel_ctx_last_times(sel_ctx ctx, float* count_ms, float* pushdown_ms) {
  clear_error();
  if (!ctx) return set_error(SEL_E_ARG, "null ctx");
  if (count_ms) *count_ms = ctx->timing ? ctx->last_count_ms : 0.f;
  if (pushdown_ms) *pushdown_ms = ctx->timing ? ctx->last_push_ms : 0.f;
  return SEL_OK;
}

int sel_ctx_last_pushdown_path(sel_ctx ctx) { return ctx ? ctx->last_pd_path : -1; }
int sel_ctx_last_pushdown_flags(sel_ctx ctx) {
  return ctx ? (ctx->last_pd_path == 1 || ctx->last_pd_path == 2 ? ctx->last_pd_flags : 0) : -1;
}

}  // extern "C"
