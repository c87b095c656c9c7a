// synopsis.cpp — many predicates in one scan (sel_count_batch, NEXT(2)) and the synopsis
// baselines beside the exact probe (NEXT(4)): block-sampled counts, equi-depth histograms and
// their estimators.
#include "host.h"

#include <cmath>

using namespace sel;

extern "C" {

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
  cudaStream_t stream = ordered_stream(c, cuda_stream);
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
  cudaStream_t stream = ordered_stream(c, cuda_stream);
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
      bool points = C.wclass == W1 && !lst[i].empty() && lst[i].size() <= 4;
      for (const Interval& x : lst[i]) points = points && x.lo == x.hi;
      bp.leaf_pts[nl] = points ? (uint8_t)lst[i].size() : 0;
      for (const Interval& x : lst[i]) {
        bp.lo[niv] = x.lo ^ bias;
        bp.span[niv] = x.hi - x.lo;
        ++niv;
      }
      ++nl;
    }
    C.leaf_count = (uint16_t)(nl - C.leaf_begin);
    C.swar = C.wclass == W1 ? 1 : 0;
    for (uint32_t l = C.leaf_begin; l < nl; ++l) C.swar = C.swar && bp.leaf_pts[l] ? 1 : 0;
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
  cudaStream_t stream = ordered_stream(c, cuda_stream);
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

}  // extern "C"
