// Attempted minimal standalone repro of the nvcc 12.9 / sm_100a miscompile described in
// DESIGN.md §9 (two inlined copies of the dynamic interval loop). This reduced form compiles
// correctly; the hazard only reproduced inside the full kernel. Kept as the record of the attempt.
#include <stdint.h>
struct Leaf { uint8_t slot, wclass, fkey, pad; uint16_t iv_begin, iv_count; };
struct P { uint32_t n_leaves; Leaf leaf[4]; const void* col[4]; uint64_t lo[8]; uint64_t span[8]; };
__device__ __forceinline__ uint32_t leaf_eval(const P& p, const Leaf& L, uint64_t base, int lane) {
  const uint8_t* c = (const uint8_t*)p.col[L.slot] + base;
  uint32_t v[32];
  for (int k = 0; k < 8; ++k) { uint32_t w = *(const uint32_t*)(c + 4*(32*k+lane)); for (int e=0;e<4;++e) v[4*k+e] = __byte_perm(w, 0u, 0x4440|e); }
  uint32_t m = 0;
  for (int t = 0; t < L.iv_count; ++t) {
    const uint32_t lo = (uint32_t)p.lo[L.iv_begin + t], sp = (uint32_t)p.span[L.iv_begin + t];
#pragma unroll
    for (int i = 0; i < 32; ++i) m |= (v[i] - lo <= sp) ? (1u << i) : 0u;
  }
  return m;
}
__global__ void k(const __grid_constant__ P p, uint32_t* out) {
  int lane = threadIdx.x & 31;
  uint32_t m[2];
#pragma unroll
  for (int c = 0; c < 2; ++c) { m[c] = 0xFFFFFFFFu; for (uint32_t l = 0; l < p.n_leaves; ++l) m[c] &= leaf_eval(p, p.leaf[l], c * 1024, lane); }
  out[2*threadIdx.x] = m[0]; out[2*threadIdx.x+1] = m[1];
}
#include <cstdio>
#include <vector>
#include <cstring>
int main() {
  const int N = 2048;
  std::vector<uint8_t> h(N); for (int i = 0; i < N; ++i) h[i] = (uint8_t)((i * 7 + i / 5) % 7);
  uint8_t* d; cudaMalloc(&d, N); cudaMemcpy(d, h.data(), N, cudaMemcpyHostToDevice);
  uint32_t* o; cudaMalloc(&o, 64 * 4);
  P p; memset(&p, 0, sizeof p); p.n_leaves = 1; p.leaf[0].slot = 0; p.leaf[0].iv_begin = 0; p.leaf[0].iv_count = 2;
  p.col[0] = d; p.lo[0] = 1; p.span[0] = 0; p.lo[1] = 4; p.span[1] = 0;
  k<<<1, 32>>>(p, o); std::vector<uint32_t> ho(64); cudaMemcpy(ho.data(), o, 256, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int lane = 0; lane < 32; ++lane) for (int c = 0; c < 2; ++c) {
    uint32_t want = 0;
    for (int kk = 0; kk < 8; ++kk) for (int e = 0; e < 4; ++e) { int r = c * 1024 + 4 * (32 * kk + lane) + e; if (h[r] == 1 || h[r] == 4) want |= 1u << (4 * kk + e); }
    if (ho[2 * lane + c] != want) { if (bad < 4) printf("lane %d chunk %d got %08x want %08x\n", lane, c, ho[2*lane+c], want); bad++; }
  }
  printf("%s bad=%d\n", bad ? "MISMATCH" : "OK", bad);
}
