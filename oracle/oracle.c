/*
 * oracle.c — TEST INFRASTRUCTURE ONLY. The plain, slow, obviously-correct CPU oracle of the
 * exact-selectivity probe. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it. It shares no code, header or table with the CUDA path
 * (paper_1806_08384_b200/csrc); it has its own decoder and validator written from the format
 * text in include/sel.h (the format is the interface; this file does not include that header).
 *
 * What it computes (plain definitions, no blocking, no reordering):
 *   count(T, P)   = |{ i in [0, N) : P(T[i]) }|
 *       — PAPER.md:226-233 (Listing 3.1, "the exact cardinality of the given selection") and
 *         "it iterates through all the tuples and simply increase a counter
 *         whenever it finds a tuple which satisfies the given condition".
 *   pushdown(T, P, proj) = the selected row ids in ascending order, and for each projected
 *         column j, out_j[k] = T[proj_j][ids[k]] (selection + projection push-down,
 *         PAPER.md:141, 235, 329; Compound = Project(Filter)), with Algorithm 1's
 *         gate "if count > maxSize throw": only the first `capacity` ids are
 *         written, the full count is returned.
 * P is evaluated row at a time as a postfix program over a bool stack; every comparison is done
 * in the column's own C type (int32_t, int64_t, float, unsigned codes), so IEEE semantics (NaN
 * false, -0 == +0) come from the C compiler. Build with -O2 and WITHOUT -ffast-math.
 *
 * Parity pins for this file live in tests/test_oracle_pins.py (SQLite and NumPy leaf semantics,
 * brute force against a recursive AST evaluator, closed-form tuple-multiset and affine-threshold
 * counts and row ids, the worked example of PAPER.md:64/88, invariants).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

enum { O_OK = 0, O_E_ARG = 1, O_E_TYPE = 3, O_E_PROGRAM = 4 };
enum { T_INT32 = 1, T_INT64 = 2, T_FLOAT32 = 3, T_DATE32 = 4, T_DICT8 = 5, T_DICT16 = 6,
       T_DICT32 = 7 };
enum { OP_TRUE = 0x01, OP_FALSE = 0x02, OP_EQ = 0x10, OP_LT = 0x11, OP_GT = 0x12, OP_LE = 0x13,
       OP_GE = 0x14, OP_BETWEEN = 0x20, OP_IN = 0x30, OP_IN_BITMAP = 0x31, OP_AND = 0x40,
       OP_OR = 0x41, OP_NOT = 0x42 };

/* Key sets of IN_BITMAP leaves: set `id` holds key i iff bit i%64 of words[id][i/64] is set. */
typedef struct {
  const uint64_t* const* words;
  const uint64_t* nbits;
  uint32_t count;
} bitmaps_t;

#define MAX_INSTR 128
#define MAX_CONSTS 512
#define MAX_DEPTH 16
#define MAX_IN 256

typedef struct {
  int op, col, a, b;
} instr_t;

typedef struct {
  int n_instr, n_consts;
  instr_t ins[MAX_INSTR];
  uint64_t k[MAX_CONSTS];
} program_t;

static unsigned get16(const uint8_t* p) { return (unsigned)p[0] | ((unsigned)p[1] << 8); }

static uint64_t get64(const uint8_t* p) {
  uint64_t v = 0;
  for (int i = 7; i >= 0; i--) v = (v << 8) | p[i];
  return v;
}

static int known_type(int t) { return t >= T_INT32 && t <= T_DICT32; }

/* Is constant slot value k representable in column type t? (include/sel.h, "Constant slots") */
static int representable(uint64_t k, int t) {
  switch (t) {
    case T_INT32:
    case T_DATE32: {
      int64_t s = (int64_t)k;
      return s >= INT32_MIN && s <= INT32_MAX;
    }
    case T_INT64: return 1;
    case T_FLOAT32: return (k >> 32) == 0;
    case T_DICT8: return k <= 0xFFu;
    case T_DICT16: return k <= 0xFFFFu;
    case T_DICT32: return k <= 0xFFFFFFFFu;
  }
  return 0;
}

/* Decode and validate, in exactly the order include/sel.h's "Program validation" lists. */
int oracle_check_into(const uint8_t* b, size_t len, const int32_t* types, uint32_t ncols,
                      program_t* P) {
  if (len < 12) return O_E_PROGRAM;
  if (b[0] != 'S' || b[1] != 'E' || b[2] != 'L' || b[3] != 'P') return O_E_PROGRAM;
  unsigned version = get16(b + 4), n_instr = get16(b + 6), n_consts = get16(b + 8),
           reserved = get16(b + 10);
  if (version != 1) return O_E_PROGRAM;
  if (n_instr == 0 || n_instr > MAX_INSTR) return O_E_PROGRAM;
  if (n_consts > MAX_CONSTS) return O_E_PROGRAM;
  if (reserved != 0) return O_E_PROGRAM;
  if (len != 12 + 8 * (size_t)(n_instr + n_consts)) return O_E_PROGRAM;
  P->n_instr = (int)n_instr;
  P->n_consts = (int)n_consts;
  for (unsigned i = 0; i < n_consts; i++) P->k[i] = get64(b + 12 + 8 * (size_t)(n_instr + i));
  int depth = 0;
  for (unsigned i = 0; i < n_instr; i++) {
    const uint8_t* q = b + 12 + 8 * (size_t)i;
    int op = q[0], col = q[1];
    unsigned a = get16(q + 2), bb = get16(q + 4), res = get16(q + 6);
    if (res != 0) return O_E_PROGRAM;
    int pops, is_leaf;
    switch (op) {
      case OP_TRUE: case OP_FALSE: pops = 0; is_leaf = 0; break;
      case OP_EQ: case OP_LT: case OP_GT: case OP_LE: case OP_GE:
      case OP_BETWEEN: case OP_IN: case OP_IN_BITMAP: pops = 0; is_leaf = 1; break;
      case OP_AND: case OP_OR: pops = 2; is_leaf = 0; break;
      case OP_NOT: pops = 1; is_leaf = 0; break;
      default: return O_E_PROGRAM;
    }
    if (!is_leaf && (col != 0 || a != 0 || bb != 0)) return O_E_PROGRAM;
    if (is_leaf) {
      if ((uint32_t)col >= ncols) return O_E_PROGRAM;
      if (op == OP_BETWEEN) {
        if (a >= n_consts || bb >= n_consts) return O_E_PROGRAM;
      } else if (op == OP_IN) {
        if (bb == 0 || bb > MAX_IN || a + bb > n_consts) return O_E_PROGRAM;
      } else if (op == OP_IN_BITMAP) {
        if (bb != 0) return O_E_PROGRAM;
      } else {
        if (bb != 0 || a >= n_consts) return O_E_PROGRAM;
      }
    }
    if (depth < pops) return O_E_PROGRAM;
    depth = depth - pops + 1;
    if (depth > MAX_DEPTH) return O_E_PROGRAM;
    if (is_leaf) {
      int t = types[col];
      if (op == OP_BETWEEN) {
        if (!representable(P->k[a], t) || !representable(P->k[bb], t)) return O_E_TYPE;
      } else if (op == OP_IN) {
        for (unsigned j = a; j < a + bb; j++)
          if (!representable(P->k[j], t)) return O_E_TYPE;
      } else if (op == OP_IN_BITMAP) {
        if (t == T_FLOAT32) return O_E_TYPE;
      } else {
        if (!representable(P->k[a], t)) return O_E_TYPE;
      }
    }
    P->ins[i].op = op;
    P->ins[i].col = col;
    P->ins[i].a = (int)a;
    P->ins[i].b = (int)bb;
  }
  if (depth != 1) return O_E_PROGRAM;
  return O_OK;
}

int oracle_check(const uint8_t* b, size_t len, const int32_t* types, uint32_t ncols) {
  for (uint32_t c = 0; c < ncols; c++)
    if (!known_type(types[c])) return O_E_TYPE;
  program_t* P = (program_t*)malloc(sizeof(program_t));
  int s = oracle_check_into(b, len, types, ncols, P);
  free(P);
  return s;
}

/* One comparison "v op k" of row i of a column, in the column's own type. */
static int compare(int op, const void* col, int t, uint64_t i, uint64_t k) {
  switch (t) {
    case T_INT32:
    case T_DATE32: {
      int32_t v = ((const int32_t*)col)[i];
      int32_t c = (int32_t)(int64_t)k;
      switch (op) {
        case OP_EQ: return v == c;
        case OP_LT: return v < c;
        case OP_GT: return v > c;
        case OP_LE: return v <= c;
        case OP_GE: return v >= c;
      }
      break;
    }
    case T_INT64: {
      int64_t v = ((const int64_t*)col)[i];
      int64_t c = (int64_t)k;
      switch (op) {
        case OP_EQ: return v == c;
        case OP_LT: return v < c;
        case OP_GT: return v > c;
        case OP_LE: return v <= c;
        case OP_GE: return v >= c;
      }
      break;
    }
    case T_FLOAT32: {
      float v = ((const float*)col)[i];
      uint32_t bits = (uint32_t)k;
      float c;
      memcpy(&c, &bits, sizeof c);
      switch (op) {
        case OP_EQ: return v == c;
        case OP_LT: return v < c;
        case OP_GT: return v > c;
        case OP_LE: return v <= c;
        case OP_GE: return v >= c;
      }
      break;
    }
    case T_DICT8:
    case T_DICT16:
    case T_DICT32: {
      uint64_t v = t == T_DICT8 ? ((const uint8_t*)col)[i]
                 : t == T_DICT16 ? ((const uint16_t*)col)[i]
                                 : ((const uint32_t*)col)[i];
      switch (op) {
        case OP_EQ: return v == k;
        case OP_LT: return v < k;
        case OP_GT: return v > k;
        case OP_LE: return v <= k;
        case OP_GE: return v >= k;
      }
      break;
    }
  }
  return 0;
}

/* v in key set `id`: 0 <= v < nbits and its bit set; v read in the column's own type. */
static int in_bitmap(const void* col, int t, uint64_t i, const bitmaps_t* bm, int id) {
  uint64_t u;
  switch (t) {
    case T_INT32:
    case T_DATE32: {
      int32_t v = ((const int32_t*)col)[i];
      if (v < 0) return 0;
      u = (uint64_t)v;
      break;
    }
    case T_INT64: {
      int64_t v = ((const int64_t*)col)[i];
      if (v < 0) return 0;
      u = (uint64_t)v;
      break;
    }
    case T_DICT8: u = ((const uint8_t*)col)[i]; break;
    case T_DICT16: u = ((const uint16_t*)col)[i]; break;
    case T_DICT32: u = ((const uint32_t*)col)[i]; break;
    default: return 0;
  }
  if (u >= bm->nbits[id]) return 0;
  return (int)((bm->words[id][u / 64] >> (u % 64)) & 1u);
}

/* P(row i): postfix evaluation on a bool stack (include/sel.h "Opcodes"). */
static int eval_row(const program_t* P, const void* const* cols, const int32_t* types,
                    uint64_t i, const bitmaps_t* bm) {
  unsigned char st[MAX_DEPTH];
  int sp = 0;
  for (int n = 0; n < P->n_instr; n++) {
    const instr_t* in = &P->ins[n];
    int r;
    switch (in->op) {
      case OP_TRUE: st[sp++] = 1; break;
      case OP_FALSE: st[sp++] = 0; break;
      case OP_EQ: case OP_LT: case OP_GT: case OP_LE: case OP_GE:
        st[sp++] = (unsigned char)compare(in->op, cols[in->col], types[in->col], i,
                                          P->k[in->a]);
        break;
      case OP_BETWEEN:
        r = compare(OP_GE, cols[in->col], types[in->col], i, P->k[in->a]) &&
            compare(OP_LE, cols[in->col], types[in->col], i, P->k[in->b]);
        st[sp++] = (unsigned char)r;
        break;
      case OP_IN:
        r = 0;
        for (int j = in->a; j < in->a + in->b; j++)
          if (compare(OP_EQ, cols[in->col], types[in->col], i, P->k[j])) r = 1;
        st[sp++] = (unsigned char)r;
        break;
      case OP_IN_BITMAP:
        st[sp++] = (unsigned char)in_bitmap(cols[in->col], types[in->col], i, bm, in->a);
        break;
      case OP_AND: sp--; st[sp - 1] = (unsigned char)(st[sp - 1] && st[sp]); break;
      case OP_OR: sp--; st[sp - 1] = (unsigned char)(st[sp - 1] || st[sp]); break;
      case OP_NOT: st[sp - 1] = (unsigned char)!st[sp - 1]; break;
    }
  }
  return st[0];
}

static int prepare(const void* const* cols, const int32_t* types, uint32_t ncols, uint64_t n,
                   const uint8_t* prog, size_t len, program_t* P, const bitmaps_t* bm) {
  if (ncols == 0 || (n > 0 && cols == NULL)) return O_E_ARG;
  for (uint32_t c = 0; c < ncols; c++) {
    if (!known_type(types[c])) return O_E_TYPE;
    if (n > 0 && cols[c] == NULL) return O_E_ARG;
  }
  int s = oracle_check_into(prog, len, types, ncols, P);
  if (s != O_OK) return s;
  for (int i = 0; i < P->n_instr; i++)   /* an IN_BITMAP id must name a given bitmap */
    if (P->ins[i].op == OP_IN_BITMAP && (uint32_t)P->ins[i].a >= bm->count) return O_E_ARG;
  return O_OK;
}


/* count(T, P) over rows [0, n). *status receives the validation status; returns UINT64_MAX
 * on error. bm_*: the IN_BITMAP key sets (may be NULL/0). */
uint64_t oracle_count_bm(const void* const* cols, const int32_t* types, uint32_t ncols,
                         uint64_t n, const uint8_t* prog, size_t len,
                         const uint64_t* const* bm_words, const uint64_t* bm_nbits,
                         uint32_t nbm, int* status) {
  const bitmaps_t bm = {bm_words, bm_nbits, nbm};
  program_t* P = (program_t*)malloc(sizeof(program_t));
  int s = prepare(cols, types, ncols, n, prog, len, P, &bm);
  if (status) *status = s;
  if (s != O_OK) { free(P); return UINT64_MAX; }
  uint64_t count = 0;
  for (uint64_t i = 0; i < n; i++)
    if (eval_row(P, cols, types, i, &bm)) count++;
  free(P);
  return count;
}

uint64_t oracle_count(const void* const* cols, const int32_t* types, uint32_t ncols, uint64_t n,
                      const uint8_t* prog, size_t len, int* status) {
  return oracle_count_bm(cols, types, ncols, n, prog, len, NULL, NULL, 0, status);
}

static size_t width_of(int t) {
  switch (t) {
    case T_INT64: return 8;
    case T_DICT8: return 1;
    case T_DICT16: return 2;
    default: return 4;
  }
}

/* pushdown(T, P, proj): ascending ids (+ row_offset), gathered projected columns, gate. */
uint64_t oracle_pushdown_bm(const void* const* cols, const int32_t* types, uint32_t ncols,
                            uint64_t n, const uint8_t* prog, size_t len, const uint32_t* proj,
                            uint32_t nproj, uint64_t row_offset, uint32_t* out_ids,
                            void* const* out_cols, uint64_t capacity,
                            const uint64_t* const* bm_words, const uint64_t* bm_nbits,
                            uint32_t nbm, int* status) {
  const bitmaps_t bm = {bm_words, bm_nbits, nbm};
  program_t* P = (program_t*)malloc(sizeof(program_t));
  int s = prepare(cols, types, ncols, n, prog, len, P, &bm);
  for (uint32_t j = 0; s == O_OK && j < nproj; j++)
    if (proj[j] >= ncols) s = O_E_ARG;
  if (status) *status = s;
  if (s != O_OK) { free(P); return UINT64_MAX; }
  uint64_t count = 0;
  for (uint64_t i = 0; i < n; i++) {
    if (!eval_row(P, cols, types, i, &bm)) continue;
    if (count < capacity) {
      out_ids[count] = (uint32_t)(row_offset + i);
      for (uint32_t j = 0; j < nproj; j++) {
        size_t w = width_of(types[proj[j]]);
        memcpy((char*)out_cols[j] + count * w, (const char*)cols[proj[j]] + i * w, w);
      }
    }
    count++;
  }
  free(P);
  return count;
}

uint64_t oracle_pushdown(const void* const* cols, const int32_t* types, uint32_t ncols,
                         uint64_t n, const uint8_t* prog, size_t len, const uint32_t* proj,
                         uint32_t nproj, uint64_t row_offset, uint32_t* out_ids,
                         void* const* out_cols, uint64_t capacity, int* status) {
  return oracle_pushdown_bm(cols, types, ncols, n, prog, len, proj, nproj, row_offset, out_ids,
                            out_cols, capacity, NULL, NULL, 0, status);
}

/* Row-sharded count over `nthreads` POSIX threads (contiguous shards, summed) — used only to
 * time the oracle on all host cores (bench.py cpu_baseline); each shard runs oracle_count. */
typedef struct {
  const void* const* cols;
  const int32_t* types;
  uint32_t ncols;
  uint64_t begin, end;
  const uint8_t* prog;
  size_t len;
  const uint64_t* const* bm_words;
  const uint64_t* bm_nbits;
  uint32_t nbm;
  uint64_t result;
  int status;
  const void* shifted[256];
} shard_t;

static void* shard_main(void* arg) {
  shard_t* s = (shard_t*)arg;
  for (uint32_t c = 0; c < s->ncols; c++)
    s->shifted[c] = (const char*)s->cols[c] + s->begin * width_of(s->types[c]);
  int st;
  s->result = oracle_count_bm(s->shifted, s->types, s->ncols, s->end - s->begin, s->prog, s->len,
                              s->bm_words, s->bm_nbits, s->nbm, &st);
  s->status = st;
  return NULL;
}

uint64_t oracle_count_mt_bm(const void* const* cols, const int32_t* types, uint32_t ncols,
                            uint64_t n, const uint8_t* prog, size_t len, int nthreads,
                            const uint64_t* const* bm_words, const uint64_t* bm_nbits,
                            uint32_t nbm, int* status) {
  int s = oracle_check(prog, len, types, ncols);
  if (status) *status = s;
  if (s != O_OK) return UINT64_MAX;
  if (ncols > 256) { if (status) *status = O_E_ARG; return UINT64_MAX; }
  if (nthreads < 1) nthreads = 1;
  shard_t* sh = (shard_t*)calloc((size_t)nthreads, sizeof(shard_t));
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  for (int t = 0; t < nthreads; t++) {
    sh[t].cols = cols; sh[t].types = types; sh[t].ncols = ncols;
    sh[t].begin = n * (uint64_t)t / (uint64_t)nthreads;
    sh[t].end = n * (uint64_t)(t + 1) / (uint64_t)nthreads;
    sh[t].prog = prog; sh[t].len = len;
    sh[t].bm_words = bm_words; sh[t].bm_nbits = bm_nbits; sh[t].nbm = nbm;
    pthread_create(&th[t], NULL, shard_main, &sh[t]);
  }
  uint64_t total = 0;
  int failed = O_OK;
  for (int t = 0; t < nthreads; t++) {
    pthread_join(th[t], NULL);
    if (sh[t].status != O_OK) failed = sh[t].status;   /* e.g. an unknown IN_BITMAP id */
    total += sh[t].result;
  }
  if (failed != O_OK) {
    if (status) *status = failed;
    free(sh);
    free(th);
    return UINT64_MAX;
  }
  free(sh);
  free(th);
  return total;
}

uint64_t oracle_count_mt(const void* const* cols, const int32_t* types, uint32_t ncols,
                         uint64_t n, const uint8_t* prog, size_t len, int nthreads,
                         int* status) {
  return oracle_count_mt_bm(cols, types, ncols, n, prog, len, nthreads, NULL, NULL, 0, status);
}

/* Row-sharded push-down over `nthreads` POSIX threads, so that whole full-size tables can be
 * checked in a test (tests/test_gpu_fullsize.py). It is the plain definition applied to
 * contiguous shards and concatenated — nothing else:
 *   1. shard t = rows [n*t/T, n*(t+1)/T); its count c_t = oracle_count_bm over the shard;
 *   2. o_t = c_0 + ... + c_{t-1} (the shard's position in the ascending result);
 *   3. shard t runs oracle_pushdown_bm over its rows with row ids offset by its first row, writing
 *      output positions [o_t, o_t + c_t) truncated at `capacity` (Algorithm 1's gate).
 * Because shards are contiguous and each shard's ids ascend, the concatenation is exactly the
 * single-threaded oracle_pushdown's result (pinned equal in tests/test_oracle_pins.py). */
typedef struct {
  const void* const* cols;
  const int32_t* types;
  uint32_t ncols;
  uint64_t begin, end;
  const uint8_t* prog;
  size_t len;
  const uint32_t* proj;
  uint32_t nproj;
  uint64_t row_offset;
  uint32_t* out_ids;       /* already shifted to the shard's output position */
  void** out_cols;         /* already shifted */
  uint64_t capacity;       /* rows this shard may write */
  const uint64_t* const* bm_words;
  const uint64_t* bm_nbits;
  uint32_t nbm;
  uint64_t result;
  int status;
  const void* shifted[256];
} pd_shard_t;

static void* pd_shard_main(void* arg) {
  pd_shard_t* s = (pd_shard_t*)arg;
  for (uint32_t c = 0; c < s->ncols; c++)
    s->shifted[c] = (const char*)s->cols[c] + s->begin * width_of(s->types[c]);
  int st;
  s->result = oracle_pushdown_bm(s->shifted, s->types, s->ncols, s->end - s->begin, s->prog,
                                 s->len, s->proj, s->nproj, s->row_offset + s->begin, s->out_ids,
                                 (void* const*)s->out_cols, s->capacity, s->bm_words, s->bm_nbits,
                                 s->nbm, &st);
  s->status = st;
  return NULL;
}

uint64_t oracle_pushdown_mt_bm(const void* const* cols, const int32_t* types, uint32_t ncols,
                               uint64_t n, const uint8_t* prog, size_t len, const uint32_t* proj,
                               uint32_t nproj, uint64_t row_offset, uint32_t* out_ids,
                               void* const* out_cols, uint64_t capacity, int nthreads,
                               const uint64_t* const* bm_words, const uint64_t* bm_nbits,
                               uint32_t nbm, int* status) {
  int s = oracle_check(prog, len, types, ncols);
  for (uint32_t j = 0; s == O_OK && j < nproj; j++)
    if (proj[j] >= ncols) s = O_E_ARG;
  if (s == O_OK && ncols > 256) s = O_E_ARG;
  if (status) *status = s;
  if (s != O_OK) return UINT64_MAX;
  if (nthreads < 1) nthreads = 1;
  /* 1. per-shard counts (the multi-threaded count's shards) */
  shard_t* cs = (shard_t*)calloc((size_t)nthreads, sizeof(shard_t));
  pd_shard_t* ps = (pd_shard_t*)calloc((size_t)nthreads, sizeof(pd_shard_t));
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  void** shifted_outs = (void**)calloc((size_t)nthreads * (nproj ? nproj : 1), sizeof(void*));
  for (int t = 0; t < nthreads; t++) {
    cs[t].cols = cols; cs[t].types = types; cs[t].ncols = ncols;
    cs[t].begin = n * (uint64_t)t / (uint64_t)nthreads;
    cs[t].end = n * (uint64_t)(t + 1) / (uint64_t)nthreads;
    cs[t].prog = prog; cs[t].len = len;
    cs[t].bm_words = bm_words; cs[t].bm_nbits = bm_nbits; cs[t].nbm = nbm;
    pthread_create(&th[t], NULL, shard_main, &cs[t]);
  }
  int failed = O_OK;
  for (int t = 0; t < nthreads; t++) {
    pthread_join(th[t], NULL);
    if (cs[t].status != O_OK) failed = cs[t].status;
  }
  /* 2. + 3. exclusive offsets, then each shard writes its slice */
  uint64_t total = 0;
  if (failed == O_OK) {
    for (int t = 0; t < nthreads; t++) {
      const uint64_t off = total;
      total += cs[t].result;
      pd_shard_t* p = &ps[t];
      p->cols = cols; p->types = types; p->ncols = ncols;
      p->begin = cs[t].begin; p->end = cs[t].end;
      p->prog = prog; p->len = len; p->proj = proj; p->nproj = nproj;
      p->row_offset = row_offset;
      p->capacity = off < capacity ? capacity - off : 0;
      if (p->capacity > cs[t].result) p->capacity = cs[t].result;
      p->out_ids = out_ids + (p->capacity ? off : 0);
      p->out_cols = shifted_outs + (size_t)t * (nproj ? nproj : 1);
      for (uint32_t j = 0; j < nproj; j++)
        p->out_cols[j] = (char*)out_cols[j] + (p->capacity ? off : 0) * width_of(types[proj[j]]);
      p->bm_words = bm_words; p->bm_nbits = bm_nbits; p->nbm = nbm;
      pthread_create(&th[t], NULL, pd_shard_main, p);
    }
    for (int t = 0; t < nthreads; t++) {
      pthread_join(th[t], NULL);
      if (ps[t].status != O_OK) failed = ps[t].status;
    }
  }
  free(cs);
  free(ps);
  free(th);
  free(shifted_outs);
  if (failed != O_OK) {
    if (status) *status = failed;
    return UINT64_MAX;
  }
  return total;
}
