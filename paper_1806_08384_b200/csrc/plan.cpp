// plan.cpp — program -> canonical plan (canon.cpp) -> kernel parameter block: the fast-path
// classification, the planner helpers, and the host-only ABI (sel_program_check/path/plan_json).
#include "host.h"

using namespace sel;

namespace sel {

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

}  // namespace sel

extern "C" {

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

}  // extern "C"
