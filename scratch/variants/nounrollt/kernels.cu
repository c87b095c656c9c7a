// kernels.cu — sm_100a kernels of the exact-selectivity probe.
//
//   count_kernel    SURVEY §8a a3: |{ i : P(row i) }| (Listing 3.1; "iterates
//                   through all the tuples and simply increase a counter"), the whole
//                   predicate fused in registers, no per-predicate bitmap ever written.
//   pushdown_kernel SURVEY §8a a6: the same evaluation + single-pass stream compaction (ascending
//                   row ids and projected columns) with the capacity gate
//                   of Algorithm 1.
//
// Data layout per warp-chunk of 1024 consecutive rows: lane l owns the eight 4-row "quads"
// q = 32k + l (k = 0..7), i.e. rows 4q..4q+3. Bit 4k+e of the lane's 32-bit mask is row
// 4(32k+l)+e. For a 4-byte column one warp instruction (fixed k) loads 32 x 16 B = 512 contiguous
// bytes (LDG.128, fully coalesced); 1-, 2- and 8-byte columns load 4/8/32 B per lane per quad
// with the same row mapping, so every leaf of a program produces masks in the same bit layout and
// AND/OR/NOT-free combination (NOT was folded into the leaves by the host) is one LOP per 32 rows.
// Counting is popc per lane, a warp redux, a CTA reduction and one partial per CTA; the last CTA
// to finish sums the partials (self-resetting, so no memset is needed between probes).
#include <cuda_runtime.h>
#include <stdint.h>

#include "sel_internal.h"

namespace sel {
namespace {

// ---- streaming loads (read once: do not allocate in L1) ------------------------------------
__device__ __forceinline__ uint4 ld_stream_v4(const void* p) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ld_stream_v2(const void* p) {
  uint2 r;
  asm("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t ld_stream_u32(const void* p) {
  uint32_t r;
  asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}

__device__ __forceinline__ uint64_t ld_acquire_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// FLOAT32 sortable key (canon.cpp): sign ? ~bits : bits | 0x80000000.
__device__ __forceinline__ uint32_t fkey(uint32_t b) {
  return b ^ ((uint32_t)((int32_t)b >> 31) | 0x80000000u);
}

// Valid-row mask of a partial chunk: bit 4k+e <=> row 4(32k+lane)+e < nvalid.
__device__ __forceinline__ uint32_t valid_mask(int lane, uint32_t nvalid) {
  uint32_t m = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t r0 = 4u * (32u * k + lane);
#pragma unroll
    for (int e = 0; e < 4; ++e) m |= (uint32_t)(r0 + e < nvalid) << (4 * k + e);
  }
  return m;
}

// ---- per-width loaders: v[4k+e] = value of row 4(32k+lane)+e of the chunk at `base` ---------
template <bool TAIL>
__device__ __forceinline__ void load_w4(const void* col, uint64_t base, int lane, uint32_t nvalid,
                                        uint32_t (&v)[32]) {
  const uint32_t* c = static_cast<const uint32_t*>(col) + base;
  uint4 x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t r0 = 4u * (32u * k + lane);
    if (!TAIL || r0 + 3 < nvalid) {
      x[k] = ld_stream_v4(c + r0);
    } else {
      x[k].x = r0 + 0 < nvalid ? c[r0 + 0] : 0u;
      x[k].y = r0 + 1 < nvalid ? c[r0 + 1] : 0u;
      x[k].z = r0 + 2 < nvalid ? c[r0 + 2] : 0u;
      x[k].w = 0u;
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    v[4 * k + 0] = x[k].x;
    v[4 * k + 1] = x[k].y;
    v[4 * k + 2] = x[k].z;
    v[4 * k + 3] = x[k].w;
  }
}

template <bool TAIL>
__device__ __forceinline__ void load_w2(const void* col, uint64_t base, int lane, uint32_t nvalid,
                                        uint32_t (&v)[32]) {
  const uint16_t* c = static_cast<const uint16_t*>(col) + base;
  uint2 x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t r0 = 4u * (32u * k + lane);
    if (!TAIL || r0 + 3 < nvalid) {
      x[k] = ld_stream_v2(c + r0);
    } else {
      const uint32_t a = r0 + 0 < nvalid ? c[r0 + 0] : 0u, b = r0 + 1 < nvalid ? c[r0 + 1] : 0u,
                     d = r0 + 2 < nvalid ? c[r0 + 2] : 0u;
      x[k].x = a | (b << 16);
      x[k].y = d;
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    v[4 * k + 0] = x[k].x & 0xFFFFu;
    v[4 * k + 1] = x[k].x >> 16;
    v[4 * k + 2] = x[k].y & 0xFFFFu;
    v[4 * k + 3] = x[k].y >> 16;
  }
}

template <bool TAIL>
__device__ __forceinline__ void load_w1(const void* col, uint64_t base, int lane, uint32_t nvalid,
                                        uint32_t (&v)[32]) {
  const uint8_t* c = static_cast<const uint8_t*>(col) + base;
  uint32_t x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t r0 = 4u * (32u * k + lane);
    if (!TAIL || r0 + 3 < nvalid) {
      x[k] = ld_stream_u32(c + r0);
    } else {
      const uint32_t a = r0 + 0 < nvalid ? c[r0 + 0] : 0u, b = r0 + 1 < nvalid ? c[r0 + 1] : 0u,
                     d = r0 + 2 < nvalid ? c[r0 + 2] : 0u;
      x[k] = a | (b << 8) | (d << 16);
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
#pragma unroll
    for (int e = 0; e < 4; ++e) v[4 * k + e] = __byte_perm(x[k], 0u, 0x4440 | e);
  }
}

// 8-byte columns, half a chunk at a time (k = 4h .. 4h+3) to bound registers.
template <bool TAIL>
__device__ __forceinline__ void load_w8_half(const void* col, uint64_t base, int lane, int h,
                                             uint32_t nvalid, uint64_t (&v)[16]) {
  const uint64_t* c = static_cast<const uint64_t*>(col) + base;
  uint4 x[8];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const uint32_t r0 = 4u * (32u * (4 * h + kk) + lane);
    if (!TAIL || r0 + 3 < nvalid) {
      x[2 * kk] = ld_stream_v4(c + r0);
      x[2 * kk + 1] = ld_stream_v4(c + r0 + 2);
    } else {
      uint64_t a = r0 + 0 < nvalid ? c[r0 + 0] : 0ull, b = r0 + 1 < nvalid ? c[r0 + 1] : 0ull,
               d = r0 + 2 < nvalid ? c[r0 + 2] : 0ull;
      x[2 * kk] = make_uint4((uint32_t)a, (uint32_t)(a >> 32), (uint32_t)b, (uint32_t)(b >> 32));
      x[2 * kk + 1] = make_uint4((uint32_t)d, (uint32_t)(d >> 32), 0u, 0u);
    }
  }
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    v[4 * kk + 0] = ((uint64_t)x[2 * kk].y << 32) | x[2 * kk].x;
    v[4 * kk + 1] = ((uint64_t)x[2 * kk].w << 32) | x[2 * kk].z;
    v[4 * kk + 2] = ((uint64_t)x[2 * kk + 1].y << 32) | x[2 * kk + 1].x;
    v[4 * kk + 3] = ((uint64_t)x[2 * kk + 1].w << 32) | x[2 * kk + 1].z;
  }
}

// One leaf: bit i of the result <=> row i of the lane's 32 rows lies in the leaf's interval set.
template <bool TAIL, class P>
__device__ __forceinline__ uint32_t eval_leaf(const P& p, const DevLeaf& L, uint64_t base,
                                              int lane, uint32_t nvalid) {
  const void* col = p.col[L.slot];
  uint32_t m = 0;
  if (L.wclass == W8) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint64_t v[16];
      load_w8_half<TAIL>(col, base, lane, h, nvalid, v);
      uint32_t mh = 0;
#pragma unroll 1
      for (int t = 0; t < L.iv_count; ++t) {
        const uint64_t lo = p.lo[L.iv_begin + t], sp = p.span[L.iv_begin + t];
#pragma unroll
        for (int i = 0; i < 16; ++i) mh |= (v[i] - lo <= sp) ? (1u << i) : 0u;
      }
      m |= mh << (16 * h);
    }
    return m;
  }
  uint32_t v[32];
  if (L.wclass == W4) {
    load_w4<TAIL>(col, base, lane, nvalid, v);
    if (L.fkey) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = fkey(v[i]);
    }
  } else if (L.wclass == W1) {
    load_w1<TAIL>(col, base, lane, nvalid, v);
  } else {
    load_w2<TAIL>(col, base, lane, nvalid, v);
  }
#pragma unroll 1
  for (int t = 0; t < L.iv_count; ++t) {
    const uint32_t lo = (uint32_t)p.lo[L.iv_begin + t], sp = (uint32_t)p.span[L.iv_begin + t];
#pragma unroll
    for (int i = 0; i < 32; ++i) m |= (v[i] - lo <= sp) ? (1u << i) : 0u;
  }
  return m;
}

// The whole predicate over the lane's 32 rows of the chunk at `base` (nvalid rows valid).
template <bool TAIL, class P>
__device__ __forceinline__ uint32_t eval_program(const P& p, uint64_t base, int lane,
                                                 uint32_t nvalid) {
  uint32_t m;
  if (p.conj) {
    m = 0xFFFFFFFFu;
    for (uint32_t l = 0; l < p.n_leaves; ++l) m &= eval_leaf<TAIL>(p, p.leaf[l], base, lane, nvalid);
  } else {
    uint32_t st[kMaxDeviceStack];
    int sp = 0;
    for (uint32_t i = 0; i < p.n_ops; ++i) {
      const uint8_t op = p.op[i];
      if (op == DOP_LEAF) {
        st[sp++] = eval_leaf<TAIL>(p, p.leaf[p.arg[i]], base, lane, nvalid);
      } else {
        --sp;
        st[sp - 1] = op == DOP_AND ? (st[sp - 1] & st[sp]) : (st[sp - 1] | st[sp]);
      }
    }
    m = st[0];
  }
  if (TAIL) m &= valid_mask(lane, nvalid);
  return m;
}

// ---- count ----------------------------------------------------------------------------------
template <class P>
__global__ void __launch_bounds__(kThreads) count_kernel(const __grid_constant__ P p, uint64_t n,
                                                         uint64_t* __restrict__ partials,
                                                         unsigned int* __restrict__ done,
                                                         uint64_t* __restrict__ out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t nfull = n / kChunkRows;
  const uint32_t rem = (uint32_t)(n % kChunkRows);
  const uint64_t gw = (uint64_t)blockIdx.x * kWarpsPerCta + warp;
  const uint64_t nw = (uint64_t)gridDim.x * kWarpsPerCta;
  uint32_t cnt = 0;
  for (uint64_t c = gw; c < nfull; c += nw)
    cnt += __popc(eval_program<false>(p, c * kChunkRows, lane, kChunkRows));
  if (rem != 0 && gw == nfull % nw) cnt += __popc(eval_program<true>(p, nfull * kChunkRows, lane, rem));
  cnt = __reduce_add_sync(0xFFFFFFFFu, cnt);

  __shared__ uint32_t s_warp[kWarpsPerCta];
  __shared__ bool s_last;
  if (lane == 0) s_warp[warp] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t s = 0;
#pragma unroll
    for (int w = 0; w < kWarpsPerCta; ++w) s += s_warp[w];
    partials[blockIdx.x] = s;
    __threadfence();
    s_last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {  // the last CTA to finish sums every partial
    __threadfence();
    uint64_t s = 0;
    for (uint32_t b = threadIdx.x; b < gridDim.x; b += kThreads) s += ((volatile uint64_t*)partials)[b];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
    __shared__ uint64_t s_sum[kWarpsPerCta];
    if (lane == 0) s_sum[warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t t = 0;
#pragma unroll
      for (int w = 0; w < kWarpsPerCta; ++w) t += s_sum[w];
      *out = t;
      *done = 0u;
    }
  }
}

// ---- push-down ------------------------------------------------------------------------------
constexpr uint64_t kFlagAgg = 1, kFlagPrefix = 2;
__device__ __forceinline__ uint64_t pack_status(uint32_t epoch, uint64_t flag, uint32_t value) {
  return ((uint64_t)epoch << 34) | (flag << 32) | value;
}

// Coalesced write-out of one warp's compacted rows: positions [gbase, gbase + lim) receive the
// chunk-local rows s_idx[0..lim) (ascending). Stores are consecutive across lanes; gathers read
// ascending rows of the chunk the warp just evaluated.
template <class T>
__device__ __forceinline__ void gather_out(const void* src_v, void* dst_v, uint64_t cbase,
                                           uint64_t gbase, const uint16_t* s_idx, uint32_t lim,
                                           int lane) {
  const T* __restrict__ src = static_cast<const T*>(src_v) + cbase;
  T* __restrict__ dst = static_cast<T*>(dst_v) + gbase;
#pragma unroll 4
  for (uint32_t q = lane; q < lim; q += 32) dst[q] = src[s_idx[q]];
}

// Warp-granular single-pass compaction. Every warp runs independently (no CTA barriers): it draws
// a tile of kPdChunks x 1024 rows from a global ticket counter (tickets are handed out in order, so
// every tile a warp waits on belongs to a warp that is already running: forward progress), evaluates
// the predicate, scans its per-stripe counts, publishes its aggregate, resolves its exclusive
// prefix by decoupled look-back over up to 32 predecessors per step, publishes the inclusive
// prefix, stages the ascending tile-local indices of the selected rows in shared memory and writes
// row ids + projected columns with coalesced stores.
template <class P>
__global__ void __launch_bounds__(kThreads) pushdown_kernel(
    const __grid_constant__ P p, uint64_t n, uint32_t* __restrict__ out_ids,
    unsigned long long* __restrict__ ticket, uint64_t ticket_base, uint64_t* __restrict__ status,
    uint32_t epoch, uint64_t* __restrict__ out_count) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t ntiles = (n + kPdTileRows - 1) / kPdTileRows;
  __shared__ uint16_t s_idx[kWarpsPerCta][kPdTileRows];  // compacted tile-local rows
  uint16_t* my = s_idx[warp];

  for (;;) {
    unsigned long long tk = 0;
    if (lane == 0) tk = atomicAdd(ticket, 1ull);
    const uint64_t tile = __shfl_sync(0xFFFFFFFFu, tk, 0) - ticket_base;
    if (tile >= ntiles) break;
    const uint64_t tbase = tile * kPdTileRows;

    // 1. evaluate the tile's chunks
    uint32_t m[kPdChunks];
#pragma unroll
    for (int c = 0; c < kPdChunks; ++c) {
      const uint64_t cbase = tbase + (uint64_t)c * kChunkRows;
      const uint32_t nvalid = cbase >= n ? 0u : (n - cbase >= (uint64_t)kChunkRows ? (uint32_t)kChunkRows : (uint32_t)(n - cbase));
      m[c] = 0;
      if (nvalid == kChunkRows) m[c] = eval_program<false>(p, cbase, lane, kChunkRows);
      else if (nvalid > 0) m[c] = eval_program<true>(p, cbase, lane, nvalid);
    }

    // 2. warp scan of per-quad-stripe counts (4 stripes of 8 bits per word; fields <= 128)
    uint32_t cw[2 * kPdChunks], ex[2 * kPdChunks], tot[2 * kPdChunks];
#pragma unroll
    for (int c = 0; c < kPdChunks; ++c) {
      uint32_t lo = 0, hi = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        lo |= (uint32_t)__popc((m[c] >> (4 * k)) & 0xFu) << (8 * k);
        hi |= (uint32_t)__popc((m[c] >> (4 * (k + 4))) & 0xFu) << (8 * k);
      }
      cw[2 * c] = lo;
      cw[2 * c + 1] = hi;
    }
#pragma unroll
    for (int w = 0; w < 2 * kPdChunks; ++w) ex[w] = cw[w];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
      for (int w = 0; w < 2 * kPdChunks; ++w) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, ex[w], d);
        if (lane >= d) ex[w] += t;
      }
    }
#pragma unroll
    for (int w = 0; w < 2 * kPdChunks; ++w) {
      tot[w] = __shfl_sync(0xFFFFFFFFu, ex[w], 31);
      ex[w] -= cw[w];                          // exclusive, per field (no borrows: ex <= inclusive)
    }
    uint32_t stripe_base[8 * kPdChunks];
    uint32_t acc = 0;
#pragma unroll
    for (int sidx = 0; sidx < 8 * kPdChunks; ++sidx) {
      stripe_base[sidx] = acc;
      acc += (tot[sidx >> 2] >> (8 * (sidx & 3))) & 0xFFu;
    }

    // 3. publish the aggregate, look back for the exclusive prefix, publish the inclusive prefix
    uint64_t excl = 0;
    if (tile == 0) {
      if (lane == 0) st_release_u64(&status[0], pack_status(epoch, kFlagPrefix, acc));
    } else {
      if (lane == 0) st_release_u64(&status[tile], pack_status(epoch, kFlagAgg, acc));
      int64_t j = (int64_t)tile - 1;
      for (;;) {
        const int64_t idx = j - lane;
        const uint64_t sw = idx >= 0 ? ld_acquire_u64(&status[idx]) : pack_status(epoch, kFlagPrefix, 0);
        const uint64_t flag = (sw >> 32) & 3u;
        const bool ready = (uint32_t)(sw >> 34) == epoch && flag != 0;
        const uint32_t notready = __ballot_sync(0xFFFFFFFFu, !ready);
        const uint32_t pref = __ballot_sync(0xFFFFFFFFu, ready && flag == kFlagPrefix);
        const uint32_t lim = notready ? (uint32_t)(__ffs(notready) - 1) : 32u;
        const uint32_t okmask = lim == 32u ? 0xFFFFFFFFu : ((1u << lim) - 1u);
        const uint32_t pok = pref & okmask;
        if (pok) {
          const uint32_t pl = (uint32_t)(__ffs(pok) - 1);
          excl += __reduce_add_sync(0xFFFFFFFFu, (uint32_t)lane <= pl ? (uint32_t)sw : 0u);
          break;
        }
        excl += __reduce_add_sync(0xFFFFFFFFu, (uint32_t)lane < lim ? (uint32_t)sw : 0u);
        j -= lim;
        if (lim == 0) __nanosleep(20);
      }
      if (lane == 0) st_release_u64(&status[tile], pack_status(epoch, kFlagPrefix, (uint32_t)(excl + acc)));
    }
    if (tile == ntiles - 1 && lane == 0) *out_count = excl + acc;
    if (acc == 0) continue;

    // 4. stage the tile-local indices of the selected rows, ascending
#pragma unroll
    for (int c = 0; c < kPdChunks; ++c) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t nib = (m[c] >> (4 * k)) & 0xFu;
        if (nib == 0) continue;
        const int sidx = 8 * c + k;
        uint32_t pos = stripe_base[sidx] + ((ex[sidx >> 2] >> (8 * (sidx & 3))) & 0xFFu);
        const uint32_t r0 = (uint32_t)c * kChunkRows + 4u * (32u * k + lane);
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (nib & (1u << e)) my[pos++] = (uint16_t)(r0 + e);
      }
    }
    __syncwarp();

    // 5. coalesced write-out of the tile's slice, honouring the capacity gate
    const uint64_t gbase = excl;
    if (gbase < p.capacity) {
      const uint32_t lim = (uint32_t)min((uint64_t)acc, p.capacity - gbase);
      const uint32_t idbase = (uint32_t)(p.row_offset + tbase);
#pragma unroll 4
      for (uint32_t q = lane; q < lim; q += 32) out_ids[gbase + q] = idbase + my[q];
      for (uint32_t j = 0; j < p.n_proj; ++j) {
        switch (p.proj_wclass[j]) {
          case W1: gather_out<uint8_t>(p.proj_src[j], p.proj_dst[j], tbase, gbase, my, lim, lane); break;
          case W2: gather_out<uint16_t>(p.proj_src[j], p.proj_dst[j], tbase, gbase, my, lim, lane); break;
          case W4: gather_out<uint32_t>(p.proj_src[j], p.proj_dst[j], tbase, gbase, my, lim, lane); break;
          default: gather_out<uint64_t>(p.proj_src[j], p.proj_dst[j], tbase, gbase, my, lim, lane); break;
        }
      }
    }
    __syncwarp();  // `my` is rewritten by the next tile
  }
}

template <class Kern>
int occupancy_of(Kern k) {
  int blocks = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k, kThreads, 0) != cudaSuccess) return 1;
  return blocks > 0 ? blocks : 1;
}

}  // namespace

int launch_count_small(const DevProgramSmall& p, uint64_t n, int grid, const Scratch& s, void* st) {
  count_kernel<DevProgramSmall><<<grid, kThreads, 0, (cudaStream_t)st>>>(p, n, s.partials, s.done, s.result);
  return (int)cudaGetLastError();
}
int launch_count_large(const DevProgramLarge& p, uint64_t n, int grid, const Scratch& s, void* st) {
  count_kernel<DevProgramLarge><<<grid, kThreads, 0, (cudaStream_t)st>>>(p, n, s.partials, s.done, s.result);
  return (int)cudaGetLastError();
}
int launch_pushdown_small(const DevProgramSmall& p, uint64_t n, uint32_t* out_ids, int grid,
                          const Scratch& s, uint64_t ticket_base, uint32_t epoch, void* st) {
  pushdown_kernel<DevProgramSmall><<<grid, kThreads, 0, (cudaStream_t)st>>>(
      p, n, out_ids, s.ticket, ticket_base, s.status, epoch, s.result);
  return (int)cudaGetLastError();
}
int launch_pushdown_large(const DevProgramLarge& p, uint64_t n, uint32_t* out_ids, int grid,
                          const Scratch& s, uint64_t ticket_base, uint32_t epoch, void* st) {
  pushdown_kernel<DevProgramLarge><<<grid, kThreads, 0, (cudaStream_t)st>>>(
      p, n, out_ids, s.ticket, ticket_base, s.status, epoch, s.result);
  return (int)cudaGetLastError();
}
int occupancy_count_small() { return occupancy_of(count_kernel<DevProgramSmall>); }
int occupancy_count_large() { return occupancy_of(count_kernel<DevProgramLarge>); }
int occupancy_pushdown_small() { return occupancy_of(pushdown_kernel<DevProgramSmall>); }
int occupancy_pushdown_large() { return occupancy_of(pushdown_kernel<DevProgramLarge>); }

}  // namespace sel
