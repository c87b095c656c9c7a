// canon.cpp — decode + validate (include/sel.h "Program validation", in that exact order) and
// canonicalise predicate programs for the device.
//
// Canonical form. Every column type has an order-preserving bijection onto unsigned keys:
//   INT32/DATE32  key = bits ^ 0x80000000           (32-bit key space)
//   INT64         key = bits ^ 0x8000000000000000   (64-bit)
//   DICT8/16/32   key = code                         (8/16/32-bit)
//   FLOAT32       key = bits ^ (sign ? 0xFFFFFFFF : 0x80000000)  — IEEE total order with -0
//                 and +0 adjacent; NaNs map outside [key(-inf), key(+inf)].
// A comparison leaf `v op c` (=, <, > and OR-of-= as IN) is then exactly a union
// of key intervals: for FLOAT32 every comparison excludes the NaN keys and treats -0 == +0
// ([key(-0), key(+0)] for c = ±0); a NaN constant gives the empty set. NOT is the complement
// within the full key space, which *includes* the NaN keys, so NOT(x < c) stays true for NaN
// (never rewritten as x >= c; SURVEY §7 "Bit-exactness hazards"). AND/OR of leaves on one column
// are intersections/unions. All rewrites are exact set identities, so the planned predicate
// selects exactly the rows of the original program.
#include "canon.h"

#include <algorithm>
#include <cstring>
#include <memory>

#include "sel_internal.h"

namespace sel {

namespace {

enum : int { S_OK = 0, S_E_TYPE = 3, S_E_PROGRAM = 4 };
enum : int { T_INT32 = 1, T_INT64 = 2, T_FLOAT32 = 3, T_DATE32 = 4, T_DICT8 = 5, T_DICT16 = 6,
             T_DICT32 = 7 };
enum : uint8_t { OP_TRUE = 0x01, OP_FALSE = 0x02, OP_EQ = 0x10, OP_LT = 0x11, OP_GT = 0x12,
                 OP_LE = 0x13, OP_GE = 0x14, OP_BETWEEN = 0x20, OP_IN = 0x30,
                 OP_IN_BITMAP = 0x31, OP_AND = 0x40, OP_OR = 0x41, OP_NOT = 0x42 };

constexpr size_t kHeader = 12, kSlot = 8;
constexpr unsigned kMaxInstr = 128, kMaxConsts = 512, kMaxDepth = 16, kMaxIn = 256;

inline uint16_t le16(const uint8_t* p) { return (uint16_t)(p[0] | (p[1] << 8)); }
inline uint64_t le64(const uint8_t* p) {
  uint64_t v;
  std::memcpy(&v, p, 8);  // little-endian host (x86-64 / aarch64)
  return v;
}

bool is_leaf_op(uint8_t op) {
  return op == OP_EQ || op == OP_LT || op == OP_GT || op == OP_LE || op == OP_GE ||
         op == OP_BETWEEN || op == OP_IN || op == OP_IN_BITMAP;
}

bool fits(int type, uint64_t k) {
  switch (type) {
    case T_INT32:
    case T_DATE32: return (int64_t)k == (int64_t)(int32_t)(uint32_t)k;
    case T_INT64: return true;
    case T_FLOAT32: return k <= 0xFFFFFFFFull;
    case T_DICT8: return k < (1ull << 8);
    case T_DICT16: return k < (1ull << 16);
    case T_DICT32: return k < (1ull << 32);
    default: return false;
  }
}

}  // namespace

int decode_program(const void* bytes, size_t len, const int* types, uint32_t ncols, Program* out,
                   std::string* msg) {
  auto fail = [&](int st, const std::string& m) {
    if (msg) *msg = m;
    return st;
  };
  const uint8_t* b = static_cast<const uint8_t*>(bytes);
  // 1. header
  if (b == nullptr || len < kHeader) return fail(S_E_PROGRAM, "program shorter than its header");
  if (std::memcmp(b, "SELP", 4) != 0) return fail(S_E_PROGRAM, "bad magic");
  const unsigned version = le16(b + 4), n_instr = le16(b + 6), n_consts = le16(b + 8),
                 reserved = le16(b + 10);
  if (version != 1) return fail(S_E_PROGRAM, "unsupported program version");
  if (n_instr == 0 || n_instr > kMaxInstr) return fail(S_E_PROGRAM, "n_instr out of range");
  if (n_consts > kMaxConsts) return fail(S_E_PROGRAM, "n_consts out of range");
  if (reserved != 0) return fail(S_E_PROGRAM, "header reserved field nonzero");
  if (len != kHeader + kSlot * (size_t)(n_instr + n_consts))
    return fail(S_E_PROGRAM, "program length does not match its header");
  out->ins.resize(n_instr);
  out->consts.resize(n_consts);
  const uint8_t* kbase = b + kHeader + kSlot * n_instr;
  for (unsigned i = 0; i < n_consts; ++i) out->consts[i] = le64(kbase + kSlot * i);
  // 2. instructions in order
  unsigned depth = 0;
  for (unsigned i = 0; i < n_instr; ++i) {
    const uint8_t* q = b + kHeader + kSlot * i;
    Instr in{q[0], q[1], le16(q + 2), le16(q + 4)};
    // the position suffix of an error message (built only on failure: no allocation per probe)
    const auto at = [i] { return " at instruction " + std::to_string(i); };
    if (le16(q + 6) != 0) return fail(S_E_PROGRAM, "instruction reserved field nonzero" + at());
    const bool leaf = is_leaf_op(in.op);
    const bool logic = in.op == OP_TRUE || in.op == OP_FALSE || in.op == OP_AND ||
                       in.op == OP_OR || in.op == OP_NOT;
    if (!leaf && !logic) return fail(S_E_PROGRAM, "unknown opcode" + at());
    if (logic && (in.col | in.a | in.b) != 0)
      return fail(S_E_PROGRAM, "logic opcode with nonzero operands" + at());
    if (leaf) {
      if (in.col >= ncols) return fail(S_E_PROGRAM, "column index out of range" + at());
      if (in.op == OP_BETWEEN) {
        if (in.a >= n_consts || in.b >= n_consts)
          return fail(S_E_PROGRAM, "BETWEEN constant out of range" + at());
      } else if (in.op == OP_IN) {
        if (in.b == 0 || in.b > kMaxIn || (unsigned)in.a + in.b > n_consts)
          return fail(S_E_PROGRAM, "IN list out of range" + at());
      } else if (in.op == OP_IN_BITMAP) {
        if (in.b != 0) return fail(S_E_PROGRAM, "IN_BITMAP with nonzero b" + at());
      } else if (in.b != 0 || in.a >= n_consts) {
        return fail(S_E_PROGRAM, "comparison constant out of range" + at());
      }
    }
    const unsigned need = in.op == OP_AND || in.op == OP_OR ? 2u : in.op == OP_NOT ? 1u : 0u;
    if (depth < need) return fail(S_E_PROGRAM, "stack underflow" + at());
    depth = depth - need + 1;
    if (depth > kMaxDepth) return fail(S_E_PROGRAM, "stack deeper than 16" + at());
    if (leaf) {
      const int t = types[in.col];
      unsigned first = in.a, last = in.a;
      if (in.op == OP_IN) last = in.a + in.b - 1u;
      if (in.op == OP_IN_BITMAP) {
        if (t == T_FLOAT32) return fail(S_E_TYPE, "IN_BITMAP on a FLOAT32 column" + at());
      } else if (in.op == OP_BETWEEN) {
        if (!fits(t, out->consts[in.a]) || !fits(t, out->consts[in.b]))
          return fail(S_E_TYPE, "BETWEEN constant not representable in its column" + at());
      } else {
        for (unsigned k = first; k <= last; ++k)
          if (!fits(t, out->consts[k]))
            return fail(S_E_TYPE, "constant not representable in its column" + at());
      }
    }
    out->ins[i] = in;
  }
  // 3. result
  if (depth != 1) return fail(S_E_PROGRAM, "program does not leave exactly one value");
  return S_OK;
}

// ------------------------------------------------------------------------------------------
// Key spaces

int key_bits(int type) {
  switch (type) {
    case T_INT64: return 64;
    case T_DICT8: return 8;
    case T_DICT16: return 16;
    default: return 32;
  }
}

uint64_t key_sign_bias(int type) {
  switch (type) {
    case T_INT32:
    case T_DATE32: return 0x80000000ull;
    case T_INT64: return 0x8000000000000000ull;
    default: return 0;
  }
}

namespace {

using IvSet = std::vector<Interval>;

uint64_t key_max(int type) {
  const int b = key_bits(type);
  return b == 64 ? ~0ull : ((1ull << b) - 1);
}

uint32_t fkey(uint32_t bits) { return bits ^ ((bits & 0x80000000u) ? 0xFFFFFFFFu : 0x80000000u); }

IvSet normalize(IvSet v) {
  std::sort(v.begin(), v.end(), [](const Interval& x, const Interval& y) { return x.lo < y.lo; });
  IvSet out;
  for (const Interval& x : v) {
    if (!out.empty() && (x.lo <= out.back().hi || x.lo - 1 == out.back().hi)) {
      out.back().hi = std::max(out.back().hi, x.hi);
    } else {
      out.push_back(x);
    }
  }
  return out;
}

IvSet unite(const IvSet& a, const IvSet& b) {
  IvSet v(a);
  v.insert(v.end(), b.begin(), b.end());
  return normalize(v);
}

IvSet intersect(const IvSet& a, const IvSet& b) {
  IvSet out;
  size_t i = 0, j = 0;
  while (i < a.size() && j < b.size()) {
    const uint64_t lo = std::max(a[i].lo, b[j].lo), hi = std::min(a[i].hi, b[j].hi);
    if (lo <= hi) out.push_back({lo, hi});
    if (a[i].hi < b[j].hi) ++i; else ++j;
  }
  return out;
}

IvSet complement(const IvSet& a, uint64_t kmax) {
  IvSet out;
  uint64_t next = 0;
  bool more = true;  // `next` still inside the key space
  for (const Interval& x : a) {
    if (x.lo > next) out.push_back({next, x.lo - 1});
    if (x.hi == kmax) { more = false; break; }
    next = x.hi + 1;
  }
  if (more) out.push_back({next, kmax});
  return out;
}

bool is_full(const IvSet& s, uint64_t kmax) {
  return s.size() == 1 && s[0].lo == 0 && s[0].hi == kmax;
}

// The key set of `v op c` for one constant slot (include/sel.h "Opcodes").
IvSet cmp_set(int type, uint8_t op, uint64_t c) {
  if (type == T_FLOAT32) {
    const uint32_t bits = (uint32_t)c;
    if ((bits & 0x7FFFFFFFu) > 0x7F800000u) return {};           // NaN: every compare false
    const bool zero = (bits & 0x7FFFFFFFu) == 0;
    const uint64_t klo = zero ? fkey(0x80000000u) : fkey(bits);   // -0 and +0 compare equal
    const uint64_t khi = zero ? fkey(0x00000000u) : fkey(bits);
    const uint64_t fmin = fkey(0xFF800000u), fmax = fkey(0x7F800000u);  // -inf, +inf
    switch (op) {
      case OP_EQ: return {{klo, khi}};
      case OP_LT: return klo > fmin ? IvSet{{fmin, klo - 1}} : IvSet{};
      case OP_LE: return {{fmin, khi}};
      case OP_GT: return khi < fmax ? IvSet{{khi + 1, fmax}} : IvSet{};
      case OP_GE: return {{klo, fmax}};
    }
    return {};
  }
  const uint64_t kmax = key_max(type);
  uint64_t k;
  if (type == T_INT32 || type == T_DATE32) k = (uint64_t)((uint32_t)c ^ 0x80000000u);
  else if (type == T_INT64) k = c ^ 0x8000000000000000ull;
  else k = c;
  switch (op) {
    case OP_EQ: return {{k, k}};
    case OP_LT: return k > 0 ? IvSet{{0, k - 1}} : IvSet{};
    case OP_LE: return {{0, k}};
    case OP_GT: return k < kmax ? IvSet{{k + 1, kmax}} : IvSet{};
    case OP_GE: return {{k, kmax}};
  }
  return {};
}

struct Node {
  enum Kind { LEAF, AND, OR, NOT, CONST, BMLEAF } kind;
  bool value = false;  // CONST; BMLEAF: negated
  int col = -1;        // LEAF, BMLEAF
  int bitmap = -1;     // BMLEAF
  IvSet set;           // LEAF
  std::vector<std::unique_ptr<Node>> kids;
};
using NodeP = std::unique_ptr<Node>;

NodeP make_const(bool v) {
  NodeP n(new Node{Node::CONST});
  n->value = v;
  return n;
}

// Leaf set -> node, folding empty/full sets into constants.
NodeP make_leaf(int col, IvSet set, const int* types) {
  if (set.empty()) return make_const(false);
  if (is_full(set, key_max(types[col]))) return make_const(true);
  NodeP n(new Node{Node::LEAF});
  n->col = col;
  n->set = std::move(set);
  return n;
}

// Push NOT down (negate), flatten, fold constants, merge same-column leaves. Exact.
NodeP simplify(NodeP n, bool negate, const int* types) {
  switch (n->kind) {
    case Node::CONST: return make_const(n->value != negate);
    case Node::LEAF:
      return make_leaf(n->col, negate ? complement(n->set, key_max(types[n->col])) : n->set, types);
    case Node::BMLEAF: {  // NOT folds into the key-set test
      NodeP b(new Node{Node::BMLEAF});
      b->col = n->col;
      b->bitmap = n->bitmap;
      b->value = n->value != negate;
      return b;
    }
    case Node::NOT: return simplify(std::move(n->kids[0]), !negate, types);
    default: break;
  }
  const bool is_and = (n->kind == Node::AND) != negate;  // De Morgan
  std::vector<NodeP> flat;
  for (auto& k : n->kids) {
    NodeP s = simplify(std::move(k), negate, types);
    if (s->kind == (is_and ? Node::AND : Node::OR)) {
      for (auto& g : s->kids) flat.push_back(std::move(g));
    } else {
      flat.push_back(std::move(s));
    }
  }
  // merge leaves on the same column, fold constants; repeat until stable
  for (bool changed = true; changed;) {
    changed = false;
    std::vector<NodeP> next;
    for (auto& k : flat) {
      if (k->kind == Node::CONST) {
        if (k->value == !is_and) return make_const(!is_and);  // absorbing element
        changed = true;                                        // identity element: drop
        continue;
      }
      if (k->kind == Node::LEAF) {
        bool merged = false;
        for (auto& m : next) {
          if (m->kind == Node::LEAF && m->col == k->col) {
            IvSet s = is_and ? intersect(m->set, k->set) : unite(m->set, k->set);
            m = make_leaf(k->col, std::move(s), types);
            merged = changed = true;
            break;
          }
        }
        if (merged) continue;
      }
      next.push_back(std::move(k));
    }
    flat = std::move(next);
  }
  if (flat.empty()) return make_const(is_and);
  if (flat.size() == 1) return std::move(flat[0]);
  NodeP out(new Node{is_and ? Node::AND : Node::OR});
  out->kids = std::move(flat);
  return out;
}

// Stack slots needed to evaluate a subtree in postfix, children ordered deepest first.
int need(const Node* n) {
  if (n->kind == Node::LEAF || n->kind == Node::CONST || n->kind == Node::BMLEAF) return 1;
  std::vector<int> d;
  for (auto& k : n->kids) d.push_back(need(k.get()));
  std::sort(d.rbegin(), d.rend());
  int m = 0;
  for (size_t i = 0; i < d.size(); ++i) m = std::max(m, d[i] + (i ? 1 : 0));
  return m;
}

void emit(const Node* n, Plan* out) {
  if (n->kind == Node::LEAF) {
    out->op.push_back(DOP_LEAF);
    out->arg.push_back((uint8_t)out->leaves.size());
    out->leaves.push_back(PlanLeaf{n->col, n->set});
    out->n_intervals += n->set.size();
    return;
  }
  if (n->kind == Node::BMLEAF) {
    out->op.push_back(DOP_LEAF);
    out->arg.push_back((uint8_t)out->leaves.size());
    PlanLeaf L{n->col, {}};
    L.bitmap = n->bitmap;
    L.negate = n->value;
    out->leaves.push_back(L);
    out->n_intervals += 1;  // its (words, nbits) table entry
    return;
  }
  std::vector<const Node*> kids;
  for (auto& k : n->kids) kids.push_back(k.get());
  std::stable_sort(kids.begin(), kids.end(),
                   [](const Node* x, const Node* y) { return need(x) > need(y); });
  for (size_t i = 0; i < kids.size(); ++i) {
    emit(kids[i], out);
    if (i) out->op.push_back(n->kind == Node::AND ? DOP_AND : DOP_OR), out->arg.push_back(0);
  }
}

}  // namespace

void plan_program(const Program& prog, const int* types, Plan* out) {
  // postfix -> tree
  std::vector<NodeP> st;
  for (const Instr& in : prog.ins) {
    switch (in.op) {
      case OP_TRUE: st.push_back(make_const(true)); break;
      case OP_FALSE: st.push_back(make_const(false)); break;
      case OP_AND:
      case OP_OR: {
        NodeP n(new Node{in.op == OP_AND ? Node::AND : Node::OR});
        NodeP y = std::move(st.back()); st.pop_back();
        NodeP x = std::move(st.back()); st.pop_back();
        n->kids.push_back(std::move(x));
        n->kids.push_back(std::move(y));
        st.push_back(std::move(n));
        break;
      }
      case OP_NOT: {
        NodeP n(new Node{Node::NOT});
        n->kids.push_back(std::move(st.back()));
        st.back() = std::move(n);
        break;
      }
      case OP_IN_BITMAP: {
        NodeP b(new Node{Node::BMLEAF});
        b->col = in.col;
        b->bitmap = in.a;
        st.push_back(std::move(b));
        break;
      }
      default: {
        const int t = types[in.col];
        IvSet s;
        if (in.op == OP_BETWEEN) {
          s = intersect(cmp_set(t, OP_GE, prog.consts[in.a]), cmp_set(t, OP_LE, prog.consts[in.b]));
        } else if (in.op == OP_IN) {
          for (unsigned k = in.a; k < (unsigned)in.a + in.b; ++k)
            s = unite(s, cmp_set(t, OP_EQ, prog.consts[k]));
        } else {
          s = cmp_set(t, in.op, prog.consts[in.a]);
        }
        st.push_back(make_leaf(in.col, normalize(std::move(s)), types));
      }
    }
  }
  NodeP root = simplify(std::move(st.back()), false, types);
  *out = Plan();
  if (root->kind == Node::CONST) {
    out->path = PATH_CONST;
    out->const_value = root->value;
    return;
  }
  emit(root.get(), out);
  out->max_depth = need(root.get());
  out->conj = root->kind == Node::LEAF || root->kind == Node::BMLEAF || root->kind == Node::AND;
  if (out->conj) {
    for (auto& k : root->kids)
      if (k->kind != Node::LEAF && k->kind != Node::BMLEAF) out->conj = false;
  }
  out->path = out->conj ? PATH_CONJ : PATH_INTERP;
}

}  // namespace sel
