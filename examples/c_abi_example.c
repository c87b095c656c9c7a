/*
 * c_abi_example.c — the exact-selectivity probe through the plain C ABI (include/sel.h), no
 * Python, no torch: the worked example's predicate (Listing 3.1)
 *     A = 2 AND B < 2001 AND B > 1000 AND (C = 1 OR C = 4)
 * over a small table whose exact answer is known by construction, then Algorithm 1's
 * Execute(isSPD, maxSize) gate and error reporting.
 *
 *   gcc -std=c11 -I include -I /usr/local/cuda/include examples/c_abi_example.c \
 *       -L paper_1806_08384_b200 -lsel -L /usr/local/cuda/lib64 -lcudart -o c_abi_example
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "sel.h"

static void put16(uint8_t* p, unsigned v) { p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); }
static void put64(uint8_t* p, uint64_t v) { for (int i = 0; i < 8; ++i) p[i] = (uint8_t)(v >> (8 * i)); }

/* program bytes (include/sel.h format): postfix instructions + constant slots */
static size_t build_program(uint8_t* out) {
  const uint8_t ins[][4] = {
      {0x10, 0, 0, 0},  /* EQ  A, k0 (2)     */
      {0x11, 1, 1, 0},  /* LT  B, k1 (2001)  */
      {0x40, 0, 0, 0},  /* AND               */
      {0x12, 1, 2, 0},  /* GT  B, k2 (1000)  */
      {0x40, 0, 0, 0},  /* AND               */
      {0x30, 2, 3, 2},  /* IN  C, k3..k4     */
      {0x40, 0, 0, 0},  /* AND               */
  };
  const uint64_t k[] = {2, 2001, 1000, 1, 4};
  const unsigned n_ins = sizeof ins / sizeof ins[0], n_k = sizeof k / sizeof k[0];
  memcpy(out, "SELP", 4);
  put16(out + 4, 1);
  put16(out + 6, n_ins);
  put16(out + 8, n_k);
  put16(out + 10, 0);
  uint8_t* p = out + 12;
  for (unsigned i = 0; i < n_ins; ++i, p += 8) {
    p[0] = ins[i][0];
    p[1] = ins[i][1];
    put16(p + 2, ins[i][2]);
    put16(p + 4, ins[i][3]);
    put16(p + 6, 0);
  }
  for (unsigned i = 0; i < n_k; ++i, p += 8) put64(p, k[i]);
  return (size_t)(p - out);
}

#define CHECK(x)                                                                  \
  do {                                                                            \
    if ((x) != 0) {                                                               \
      fprintf(stderr, "%s failed: %s\n", #x, sel_last_error_message());         \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

/* Write `bytes` of `p` to dir/name (the test harness compares them with the CPU oracle). */
static int dump(const char* dir, const char* name, const void* p, size_t bytes) {
  char path[4096];
  snprintf(path, sizeof path, "%s/%s", dir, name);
  FILE* f = fopen(path, "wb");
  if (!f) return 1;
  const size_t w = fwrite(p, 1, bytes, f);
  fclose(f);
  return w != bytes;
}

/* usage: c_abi_example [dump_dir] — with dump_dir, the table, the program bytes and the
 * Execute's row ids and projected column are written there (tests/test_c_abi.py checks them
 * against the oracle). */
int main(int argc, char** argv) {
  const uint64_t n = 1000003;              /* ragged: not a multiple of 1024 */
  int32_t* a = malloc(n * 4);
  int32_t* b = malloc(n * 4);
  uint8_t* c = malloc(n);
  uint64_t want = 0;
  for (uint64_t i = 0; i < n; ++i) {
    a[i] = (int32_t)(i % 5);
    b[i] = (int32_t)((i * 7919) % 2500);
    c[i] = (uint8_t)((i * 31) % 7);
    if (a[i] == 2 && b[i] < 2001 && b[i] > 1000 && (c[i] == 1 || c[i] == 4)) ++want;
  }
  void *da, *db, *dc;
  cudaMalloc(&da, n * 4);
  cudaMalloc(&db, n * 4);
  cudaMalloc(&dc, n);
  cudaMemcpy(da, a, n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b, n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dc, c, n, cudaMemcpyHostToDevice);

  sel_ctx ctx;
  CHECK(sel_ctx_create(0, &ctx));
  sel_column cols[3] = {{SEL_INT32, da, 0}, {SEL_INT32, db, 0}, {SEL_DICT8, dc, 7}};
  sel_table t;
  CHECK(sel_table_register(ctx, cols, 3, n, 0, n, &t));

  uint8_t prog[256];
  const size_t len = build_program(prog);
  const uint64_t count = sel_count(t, prog, len, NULL);
  printf("count = %llu (expected %llu)\n", (unsigned long long)count, (unsigned long long)want);
  if (count != want) return 2;

  /* Execute(isSPD, maxSize): gate passes with maxSize = count, "throws" with count - 1 */
  uint32_t* ids;
  int32_t* proj;
  cudaMalloc((void**)&ids, count * 4);
  cudaMalloc((void**)&proj, count * 4);
  const uint32_t pcol[1] = {1};
  void* outs[1] = {proj};
  uint64_t local = 0, off = 0;
  int materialized = -1;
  uint64_t r = sel_execute(t, prog, len, pcol, 1, count, ids, outs, count, &local, &off,
                           &materialized, NULL);
  if (r != want || !materialized || local != want) return 3;
  uint32_t* hids = malloc(count * 4);
  int32_t* hb = malloc(count * 4);
  cudaMemcpy(hids, ids, count * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hb, proj, count * 4, cudaMemcpyDeviceToHost);
  uint64_t k = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (a[i] == 2 && b[i] < 2001 && b[i] > 1000 && (c[i] == 1 || c[i] == 4)) {
      if (hids[k] != i || hb[k] != b[i]) { printf("mismatch at %llu\n", (unsigned long long)k); return 4; }
      ++k;
    }
  }
  if (argc > 1 && (dump(argv[1], "A.bin", a, n * 4) || dump(argv[1], "B.bin", b, n * 4) ||
                   dump(argv[1], "C.bin", c, n) || dump(argv[1], "prog.bin", prog, len) ||
                   dump(argv[1], "ids.bin", hids, count * 4) || dump(argv[1], "projB.bin", hb, count * 4))) {
    fprintf(stderr, "cannot write to %s\n", argv[1]);
    return 7;
  }
  r = sel_execute(t, prog, len, pcol, 1, count - 1, ids, outs, count, &local, &off, &materialized, NULL);
  if (r != want || materialized) return 5;
  printf("execute: materialised %llu ascending ids; gate at maxSize = count - 1 -> reverted\n",
         (unsigned long long)want);

  /* the asynchronous count: lands in a device word, no host synchronisation in the call */
  uint64_t* dcount;
  uint64_t hcount = 0;
  cudaMalloc((void**)&dcount, sizeof(uint64_t));
  CHECK(sel_count_async(t, prog, len, dcount, NULL));
  cudaMemcpy(&hcount, dcount, sizeof(uint64_t), cudaMemcpyDeviceToHost);   /* synchronises */
  if (hcount != want) return 6;
  cudaFree(dcount);

  /* error path: a malformed program */
  const uint8_t bad[4] = {'S', 'E', 'L', 'P'};
  if (sel_count(t, bad, sizeof bad, NULL) != SEL_ERR || sel_last_error() != SEL_E_PROGRAM) return 6;
  printf("bad program -> SEL_E_PROGRAM: %s\n", sel_last_error_message());

  sel_table_release(t);
  sel_ctx_destroy(ctx);
  cudaFree(da); cudaFree(db); cudaFree(dc); cudaFree(ids); cudaFree(proj);
  free(a); free(b); free(c); free(hids); free(hb);
  printf("C ABI example ok\n");
  return 0;
}
