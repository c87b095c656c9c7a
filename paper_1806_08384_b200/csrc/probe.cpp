// probe.cpp — the probe path: count, push-down and Algorithm 1's Execute
// enqueued on the caller's stream, and their ABI entry points (sel_count*, sel_pushdown,
// sel_execute*).
#include "host.h"

using namespace sel;

namespace sel {

// Timing event on `s`; inside a stream capture it must be an external event-record node (a plain
// record would only express a dependency within the capture).
void record(sel_ctx c, cudaEvent_t ev, cudaStream_t s) {
  if (c->capturing) cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal);
  else cudaEventRecord(ev, s);
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
                         bool allreduce, const uint32_t* code_cols,
                         uint32_t ncode, const ExecFinish* fin) {
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
                                cudaStream_t stream, int gate_ranks,
                                const PeerXchg* xg, bool global_out,
                                bool finished, uint64_t* host) {
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
  const int bc = pushdown_block_chunks(n);
  const uint64_t nblocks = (ntiles + bc - 1) / bc;
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
                                   c->s, c->sel, stream, gate_ranks, xg, c->rank, finished, host, bc);
  } else {
    static thread_local DevProgramLarge p;
    fill_sel(&p);
    c->last_pd_flags = flags_of(p);
    le = launch_pushdown_sel_large(p, n, out_rowids, grid_for(c, units, occupancy_pushdown_sel_large()),
                                   c->s, c->sel, stream, gate_ranks, xg, c->rank, finished, host, bc);
  }
  if (le != cudaSuccess) return set_error(SEL_E_CUDA, cuda_msg("push-down kernel launch", (cudaError_t)le));
  c->last_pd_path = 1;
  return SEL_OK;
}

// All-gather a per-rank count into result[1..nranks] and its pinned mirror,
// blocking (used where a rank has nothing of its own to enqueue but must match the collectives of
// the others).
sel_status gather_counts(sel_ctx c, uint64_t local, void* cuda_stream) {
  cudaStream_t stream = ordered_stream(c, cuda_stream);
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
                           bool global_out) {
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

}  // namespace sel

extern "C" {

uint64_t sel_count(sel_table t, const void* prog, size_t prog_bytes, void* cuda_stream) {
  return sel_count_ex(t, prog, prog_bytes, 0u, nullptr, 0u, cuda_stream);
}

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
  cudaStream_t stream = ordered_stream(c, cuda_stream);
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
  cudaStream_t stream = ordered_stream(c, cuda_stream);
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
  cudaStream_t stream = ordered_stream(c, cuda_stream);
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
        cudaStream_t stream = ordered_stream(c, cuda_stream);
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
  cudaStream_t stream = ordered_stream(c, cuda_stream);
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
