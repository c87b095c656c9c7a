// graph.cpp — prepared executes (sel_prepare_execute): a fixed Algorithm 1 Execute validated
// once and captured, with its collective, into a CUDA graph; each run is one graph launch and
// one synchronisation.
#include "host.h"

using namespace sel;

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

static uint64_t run_prepared(sel_prepared q, uint64_t* out_local_count,
                             uint64_t* out_global_offset, int* out_materialized,
                             void* cuda_stream, bool async) {
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
  cudaStream_t stream = ordered_stream(c, cuda_stream);
  c->kept_table = nullptr;
  // Returning at the count needs its words in the pinned mirror (finish_execute) and no timing
  // events to read; otherwise the run blocks.
  async = async && !c->timing && (multi(c) ? c->nranks : 0) <= kMirrorMax;
  const uint64_t seq0 = *(volatile const uint64_t*)(c->h_result + kSeqSlot);
  cudaError_t e = cudaGraphLaunch(q->exec, stream);
  if (e == cudaSuccess && async) {   // later calls on other streams order after this one
    e = cudaEventRecord(c->async_ev, stream);
    c->async_pending = e == cudaSuccess;
    c->async_stream = stream;
  }
  if (e == cudaSuccess) e = async ? wait_result_seq(c, stream, seq0) : sync_stream(c, stream);
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

uint64_t sel_prepared_execute(sel_prepared q, uint64_t* out_local_count,
                              uint64_t* out_global_offset, int* out_materialized,
                              void* cuda_stream) {
  return run_prepared(q, out_local_count, out_global_offset, out_materialized, cuda_stream, false);
}

uint64_t sel_prepared_execute_async(sel_prepared q, uint64_t* out_local_count,
                                    uint64_t* out_global_offset, int* out_materialized,
                                    void* cuda_stream) {
  return run_prepared(q, out_local_count, out_global_offset, out_materialized, cuda_stream, true);
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
