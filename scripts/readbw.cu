// readbw.cu — read-only HBM streaming microbenchmark (LDG.128 and TMA bulk rings) behind the
// 7,389 / 7,204 GB/s figures in DESIGN.md §6. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 readbw.cu
// Read-only streaming bandwidth microbenchmark (scratch, not product): how fast can a B200 stream
// a large buffer with LDG.128 (and with cp.async.bulk into shared memory)?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 ldg_na(const void* p) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

template <int U>
__global__ void __launch_bounds__(256) rd(const uint4* __restrict__ p, size_t n16, unsigned* out) {
  size_t i = (size_t)blockIdx.x * 256 * U + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * 256 * U;
  uint32_t acc = 0;
  for (; i + (U - 1) * 256 < n16; i += stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ldg_na(p + i + u * 256);
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// 1D bulk copies global -> shared with an mbarrier, 4-stage ring per CTA.
__global__ void __launch_bounds__(128) rd_bulk(const char* __restrict__ p, size_t bytes, unsigned* out) {
  constexpr int STAGES = 4, CHUNK = 32768;
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t bar[STAGES];
  const size_t nchunks = bytes / CHUNK;
  if (threadIdx.x == 0)
    for (int s = 0; s < STAGES; ++s)
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar[s])));
  __syncthreads();
  uint32_t acc = 0;
  size_t c = blockIdx.x;
  int issued = 0;
  auto issue = [&](size_t chunk, int s) {
    unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
    unsigned d = (unsigned)__cvta_generic_to_shared(smem + s * CHUNK);
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(CHUNK));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(d), "l"(p + chunk * CHUNK), "r"(CHUNK), "r"(b) : "memory");
  };
  if (threadIdx.x == 0)
    for (int s = 0; s < STAGES && c + (size_t)s * gridDim.x < nchunks; ++s) { issue(c + (size_t)s * gridDim.x, s); issued++; }
  int s = 0; unsigned phase = 0;
  for (size_t k = c; k < nchunks; k += gridDim.x) {
    unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
    unsigned done = 0;
    while (!done) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(b), "r"(phase));
    const uint4* q = reinterpret_cast<const uint4*>(smem + s * CHUNK);
    for (int i = threadIdx.x; i < CHUNK / 16; i += 128) { uint4 v = q[i]; acc ^= v.x ^ v.y ^ v.z ^ v.w; }
    __syncthreads();
    size_t nk = k + (size_t)STAGES * gridDim.x;
    if (threadIdx.x == 0 && nk < nchunks) issue(nk, s);
    if (++s == STAGES) { s = 0; phase ^= 1; }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  const size_t bytes = 8ull << 30;
  char* p; cudaMalloc(&p, bytes); cudaMemset(p, 1, bytes);
  unsigned* o; cudaMalloc(&o, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto timeit = [&](auto launch, const char* name) {
    for (int w = 0; w < 3; ++w) launch();
    cudaEventRecord(a);
    const int it = 10;
    for (int r = 0; r < it; ++r) launch();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-28s %8.1f GB/s  (%.3f ms)\n", name, bytes / (ms / it * 1e-3) / 1e9, ms / it);
  };
  for (int occ : {4, 8}) {
    char nm[64];
    snprintf(nm, 64, "ldg128 U=4 occ=%d", occ); timeit([&] { rd<4><<<sms * occ, 256>>>((const uint4*)p, bytes / 16, o); }, nm);
    snprintf(nm, 64, "ldg128 U=8 occ=%d", occ); timeit([&] { rd<8><<<sms * occ, 256>>>((const uint4*)p, bytes / 16, o); }, nm);
    snprintf(nm, 64, "ldg128 U=16 occ=%d", occ); timeit([&] { rd<16><<<sms * occ, 256>>>((const uint4*)p, bytes / 16, o); }, nm);
  }
  cudaFuncSetAttribute(rd_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768);
  for (int occ : {1}) {
    char nm[64];
    snprintf(nm, 64, "bulk 4x32KB occ=%d", occ);
    timeit([&] { rd_bulk<<<sms * occ, 128, 4 * 32768>>>(p, bytes, o); }, nm);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  // copy for reference
  char* q; cudaMalloc(&q, bytes / 2);
  cudaEventRecord(a);
  for (int r = 0; r < 10; ++r) cudaMemcpyAsync(q, p, bytes / 2, cudaMemcpyDeviceToDevice);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("%-28s %8.1f GB/s (read+write)\n", "cudaMemcpy D2D 4GiB", bytes / (ms / 10 * 1e-3) / 1e9);
}
