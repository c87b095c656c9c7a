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
// AND/OR combination (NOT was folded into the leaves by the host) is one LOP per 32 rows.
//
// Toolchain note (nvcc 12.9, sm_100a): when eval_leaf's dynamic interval loop was instantiated
// twice by unrolling an enclosing loop, the second instance produced wrong masks (intervals >= 2
// lost). Every loop enclosing eval_leaf is therefore kept rolled; tests/test_gpu_parity.py
// exercises multi-interval leaves of every width in both kernels.
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <tuple>
#include <stdint.h>

#include <type_traits>

#include <cub/device/device_radix_sort.cuh>

#include "sel_internal.h"

#ifndef SEL_BATCH_MINB
// batch count: 4 resident CTAs per SM (<= 64 registers; 62 used, no spills). A/B on the worked
// example's five programs: 0.845 -> 0.822-0.830 ms against the unbounded 79 registers (3 CTAs);
// 5 CTAs 0.828-0.839, a next-chunk L2 prefetch 0.833 alone, 0.840-0.851 with 4 CTAs
#define SEL_BATCH_MINB 4
#endif
#ifndef SEL_BATCH_PREFETCH
#define SEL_BATCH_PREFETCH 1   // batch count: bulk-prefetch a chunk's later columns into L2
#endif


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

// Tile status words carry their own payload (epoch | flag | value in one 64-bit word, single-copy
// atomic), so the look-back needs no acquire/release ordering: relaxed gpu-scope accesses only
// (an acquire load would emit CCTL.IVALL, an L1 invalidation, on every poll).
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// TMA bulk prefetch of [p, p + bytes) into L2 (bytes multiple of 16, p 16-byte aligned).
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// ---- peer exchange (sel_internal.h PeerXchg) -------------------------------------------------
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Run by all threads of ONE CTA (blockDim.x >= 32); see PeerXchg. A wait beyond x.timeout_ns (a
// rank did not take part) fails the whole exchange: every value written to out and sums is then
// kXchgFailed, never a partial sum.
__device__ void peer_gather_block(const PeerXchg& x, const uint64_t* src, int k, uint64_t* out,
                                  uint64_t* sums) {
  __shared__ uint32_t s_e;
  __shared__ int s_fail;
  __shared__ uint64_t s_v[kMaxXchgVals];
  __shared__ uint64_t s_got[kMaxPeers * kMaxXchgVals];
  const int t = threadIdx.x;
  if (t == 0) {
    s_e = *x.epoch + 1u;
    *x.epoch = s_e;
    s_fail = 0;
  }
  if (t < k) s_v[t] = src[t];
  __syncthreads();
  const uint64_t e = s_e;
  const uint32_t half = (s_e & 1u) * kMaxPeers * kMaxXchgVals;
  // write my k values into row `rank` of every rank's buffer
  for (int i = t; i < x.n * k; i += blockDim.x) {
    const int r = i / k, j = i - r * k;
    st_release_sys(x.peers[r] + half + x.rank * kMaxXchgVals + j, (e << 32) | (s_v[j] & 0xFFFFFFFFull));
  }
  // wait for every rank's row in my buffer
  for (int i = t; i < x.n * k; i += blockDim.x) {
    const int r = i / k, j = i - r * k;
    const uint64_t* slot = x.mine + half + r * kMaxXchgVals + j;
    uint64_t w = ld_acquire_sys(slot);
    if ((w >> 32) != e) {
      const uint64_t t0 = globaltimer_ns();
      while (((w = ld_acquire_sys(slot)) >> 32) != e) {
        if (globaltimer_ns() - t0 > x.timeout_ns) {  // a rank is missing
          atomicExch(x.err, 1u);
          s_fail = 1;
          w = 0;
          break;
        }
        __nanosleep(64);
      }
    }
    s_got[i] = w & 0xFFFFFFFFull;
  }
  __syncthreads();
  const bool fail = s_fail != 0;
  if (out)
    for (int i = t; i < x.n * k; i += blockDim.x) out[i] = fail ? kXchgFailed : s_got[i];
  if (sums && t < k) {
    uint64_t acc = 0;
    for (int r = 0; r < x.n; ++r) acc += s_got[r * k + t];
    sums[t] = fail ? kXchgFailed : acc;
  }
  __syncthreads();
}

// ExecFinish (sel_internal.h), run by all threads of ONE CTA; `local` = this rank's count, already
// in R[kGateSlot] when an exchange (xg.n > 0) or no rank combination (gate_ranks == 0) follows.
__device__ void finish_execute(const ExecFinish& f, const PeerXchg& xg, uint64_t local) {
  uint64_t* R = f.result;
  const uint32_t t = threadIdx.x;
  if (xg.n > 0) peer_gather_block(xg, R + kGateSlot, 1, R + 1, R + kGateSlot);  // ends in a barrier
  // a failed exchange left kXchgFailed in the gate slot: the push-down kernels write nothing
  const bool failed = xg.n > 0 && R[kGateSlot] == kXchgFailed;
  const int nr = xg.n > 0 ? xg.n : f.gate_ranks;
  if (t == 0) {
    if (f.gate_ranks > 0 && xg.n == 0) {   // NCCL: the all-gathered counts are summed here
      uint64_t g = 0;
      for (int r = 0; r < f.gate_ranks; ++r) g += R[1 + r];
      R[kGateSlot] = g;
    }
    uint64_t off = 0;   // this rank's position in the rank-ordered global result (sel_execute_to)
    for (int r = 0; r < f.rank && r < nr; ++r) off += R[1 + r];
    R[kOffsetSlot] = failed ? kXchgFailed : off;
    if (nr == 0) R[kGateSlot - 1] = local;
  }
  if (nr > 0 && nr <= kMirrorMax)
    for (int i = (int)t; i < nr; i += (int)blockDim.x) R[kGateSlot - nr + i] = R[1 + i];
  if (f.host) {   // the pinned mirror: the host reads it after its one synchronisation
    __syncthreads();
    const int lo = kGateSlot - (nr > 0 ? nr : 1);
    for (int i = lo + (int)t; i <= kOffsetSlot; i += (int)blockDim.x) f.host[i] = R[i];
    // then the sequence word, ordered after every thread's mirror stores (barrier, then thread
    // 0's system-scope fence, cumulative over what the barrier ordered before it — the pattern of
    // a grid barrier's arrival): sel_prepared_execute_async returns once it changes. (A fence in
    // every writer before the barrier as well: +3 us per Execute, profiles/r2/ab/)
    __syncthreads();
    if (t == 0) {
      const uint64_t q = R[kSeqSlot] + 1u;
      R[kSeqSlot] = q;
      __threadfence_system();
      f.host[kSeqSlot] = q;
    }
  }
}

// The kept selection's half of the superblock sums (sel_internal.h SelectionBufs), after its count.
__device__ __forceinline__ const uint32_t* kept_sb(const SelectionBufs& sb) {
  return sb.sb_sum + (size_t)((sb.state[0] - 1u) & 1u) * sb.sb_stride;
}

// Output position of chunk c0's first selected row in the local result: hyperblock prefix +
// superblock sums before c0 within its hyperblock + chunk counts before c0 within its superblock
// (every lane; loads issued together).
__device__ __forceinline__ uint64_t kept_base(const SelectionBufs& sb, const uint32_t* sbs,
                                              uint64_t c0, int lane) {
  const uint64_t s0 = c0 >> kSbShift, first = s0 << kSbShift;
  const uint64_t sfirst = (c0 >> kHbShift) << (kHbShift - kSbShift);
  uint32_t part = 0;
  if (first + lane < c0) part += sb.chunk_cnt[first + lane];
  if (first + 32 + lane < c0) part += sb.chunk_cnt[first + 32 + lane];
  if (sfirst + lane < s0) part += sbs[sfirst + lane];
  if (sfirst + 32 + lane < s0) part += sbs[sfirst + 32 + lane];
  const uint32_t hp = sb.hb_prefix[c0 >> kHbShift];
  return (uint64_t)hp + __reduce_add_sync(0xFFFFFFFFu, part);
}

// The last CTA of a keeping count (NW warps): the exclusive prefix of the hyperblock sums, each
// summed here from this count's superblock sums (thread t sums whole hyperblocks with 16-byte
// loads, all issued together; <= 4 per thread), the local count (their total, returned: no pass
// over the per-CTA partials) and the full-chunk flag beside it, and the epoch advanced (this
// count's half of the superblock sums becomes the selection's; the next count zeroes the other
// one, nsb words).
template <int NW>
__device__ uint32_t finish_selection(const SelectionBufs& sb, uint64_t n, uint32_t e,
                                     const uint32_t* my_sb) {
  constexpr uint32_t T = NW * 32;
  constexpr uint32_t kSbPerHb = 1u << (kHbShift - kSbShift);
  const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint64_t nchunks = (n + kChunkRows - 1) / kChunkRows;
  const uint32_t nsb = (uint32_t)((nchunks + kSbChunks - 1) / kSbChunks);
  const uint32_t nsb4 = (nsb + 3u) & ~3u;   // the half is zero-padded to a multiple of 4 words
  const uint32_t nhb = (uint32_t)((nchunks + kHbChunks - 1) / kHbChunks);
  const uint32_t per = (nhb + T - 1) / T;   // <= 4: nhb <= 1024 (tables < 2^32 rows)
  const uint32_t b = min(nhb, t * per), end = min(nhb, b + per);
  const uint4* q = reinterpret_cast<const uint4*>(my_sb);
  uint32_t v[4], sum = 0;
#pragma unroll
  for (uint32_t k = 0; k < 4; ++k) {
    v[k] = 0u;
    if (b + k < end) {
      const uint32_t w0 = (b + k) * kSbPerHb;
      uint4 x[kSbPerHb / 4];
#pragma unroll
      for (uint32_t i = 0; i < kSbPerHb / 4; ++i)
        x[i] = w0 + 4 * i < nsb4 ? __ldcg(q + w0 / 4 + i) : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (uint32_t i = 0; i < kSbPerHb / 4; ++i) v[k] += x[i].x + x[i].y + x[i].z + x[i].w;
    }
    sum += v[k];
  }
  uint32_t incl = sum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t x = __shfl_up_sync(0xFFFFFFFFu, incl, d);
    if (lane >= (uint32_t)d) incl += x;
  }
  __shared__ uint32_t s_w[NW];
  __shared__ uint32_t s_all;
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t w = lane < (uint32_t)NW ? s_w[lane] : 0u;
    uint32_t wi = w;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t x = __shfl_up_sync(0xFFFFFFFFu, wi, d);
      if (lane >= (uint32_t)d) wi += x;
    }
    if (lane < (uint32_t)NW) s_w[lane] = wi - w;
    if (lane == 31) s_all = wi;
  }
  __syncthreads();
  const uint32_t local = s_all;
  uint32_t run = s_w[warp] + incl - sum;
#pragma unroll
  for (uint32_t k = 0; k < 4; ++k) {
    if (b + k < end) sb.hb_prefix[b + k] = run;
    run += v[k];
  }
  if (t == 0) {
    sb.hb_prefix[nhb] = local;
    sb.hb_prefix[nhb + 1] = __ldcg(sb.state + 3);   // the full-chunk flag, reset for the next count
    sb.state[3] = 0u;
    sb.state[1 + (e & 1u)] = nsb;
    sb.state[0] = e + 1u;
  }
  return local;
}

// Prefetch every predicate column of chunk `c` into L2 (issued by one lane a chunk ahead).
template <class P>
__device__ __forceinline__ void prefetch_chunk(const P& p, uint64_t c) {
#pragma unroll 1
  for (uint32_t l = 0; l < p.n_leaves; ++l) {
    const DevLeaf& L = p.leaf[l];
    const uint32_t w = 1u << L.wclass;
    prefetch_l2(static_cast<const char*>(p.col[L.slot]) + c * kChunkRows * w, kChunkRows * w);
  }
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
// With cap != nullptr the raw quads are also stored to `cap` (shared memory, chunk row r at
// cap + r*w), so a projected predicate column is never read from global memory a second time.
// (A runtime pointer, not a template flag: one inlined copy of the interval loop per TAIL variant,
// see the toolchain note above.)
template <bool TAIL>
__device__ __forceinline__ void load_w4(const void* col, uint64_t base, int lane, uint32_t nvalid,
                                        uint32_t (&v)[32], char* cap) {
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
    if (cap) reinterpret_cast<uint4*>(cap)[32 * k + lane] = x[k];
    v[4 * k + 0] = x[k].x;
    v[4 * k + 1] = x[k].y;
    v[4 * k + 2] = x[k].z;
    v[4 * k + 3] = x[k].w;
  }
}

template <bool TAIL>
__device__ __forceinline__ void load_w2(const void* col, uint64_t base, int lane, uint32_t nvalid,
                                        uint32_t (&v)[32], char* cap) {
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
    if (cap) reinterpret_cast<uint2*>(cap)[32 * k + lane] = x[k];
    v[4 * k + 0] = x[k].x & 0xFFFFu;
    v[4 * k + 1] = x[k].x >> 16;
    v[4 * k + 2] = x[k].y & 0xFFFFu;
    v[4 * k + 3] = x[k].y >> 16;
  }
}

// A chunk of a 1-byte column as 8 words per lane (word k = rows 4(32k + lane) .. +3; bytes past
// nvalid are 0).
template <bool TAIL>
__device__ __forceinline__ void load_w1_words(const void* col, uint64_t base, int lane,
                                              uint32_t nvalid, uint32_t (&x)[8]) {
  const uint8_t* c = static_cast<const uint8_t*>(col) + base;
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
}

template <bool TAIL>
__device__ __forceinline__ void load_w1(const void* col, uint64_t base, int lane, uint32_t nvalid,
                                        uint32_t (&v)[32], char* cap) {
  uint32_t x[8];
  load_w1_words<TAIL>(col, base, lane, nvalid, x);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if (cap) reinterpret_cast<uint32_t*>(cap)[32 * k + lane] = x[k];
#pragma unroll
    for (int e = 0; e < 4; ++e) v[4 * k + e] = __byte_perm(x[k], 0u, 0x4440 | e);
  }
}

// 8-byte columns, half a chunk at a time (k = 4h .. 4h+3) to bound registers.
template <bool TAIL>
__device__ __forceinline__ void load_w8_half(const void* col, uint64_t base, int lane, int h,
                                             uint32_t nvalid, uint64_t (&v)[16], char* cap) {
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
    if (cap) {
      uint4* dst = reinterpret_cast<uint4*>(cap) + 2 * (32 * (4 * h + kk) + lane);
      dst[0] = x[2 * kk];
      dst[1] = x[2 * kk + 1];
    }
    v[4 * kk + 0] = ((uint64_t)x[2 * kk].y << 32) | x[2 * kk].x;
    v[4 * kk + 1] = ((uint64_t)x[2 * kk].w << 32) | x[2 * kk].z;
    v[4 * kk + 2] = ((uint64_t)x[2 * kk + 1].y << 32) | x[2 * kk + 1].x;
    v[4 * kk + 3] = ((uint64_t)x[2 * kk + 1].w << 32) | x[2 * kk + 1].z;
  }
}

// IN_BITMAP membership of N raw values: bit i <=> v[i] < nbits and bit v[i]
// of the key set is set. Raw unsigned compare: negative INT32/INT64 values are >= 2^31 > nbits.
// The set is small and hot (read-only path, L1/L2 resident); 32-bit words, little-endian layout.
template <int N, class T>
__device__ __forceinline__ uint32_t bitmap_test(const T (&v)[N], uint64_t words, uint64_t nbits) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(words);
  uint32_t m = 0;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const bool in = v[i] < (T)nbits;
    const uint32_t x = in ? __ldg(w + (uint32_t)(v[i] >> 5)) : 0u;
    m |= ((x >> ((uint32_t)v[i] & 31u)) & 1u) << i;
  }
  return m;
}

// The same test against a copy of the set staged in shared memory at shared address `sw`
// (count kernel, p.bm_smem): random 4-byte LDS cost ~conflict-degree cycles per warp instead of
// one L1 wavefront per distinct 128-byte line.
__device__ __forceinline__ uint32_t lds_u32(uint32_t saddr) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr));
  return v;
}
template <int N, class T>
__device__ __forceinline__ uint32_t bitmap_test_smem(const T (&v)[N], uint32_t sw, uint32_t nbits) {
  uint32_t m = 0;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const bool in = v[i] < (T)nbits;
    const uint32_t x = in ? lds_u32(sw + 4u * (uint32_t)(v[i] >> 5)) : 0u;
    m |= ((x >> ((uint32_t)v[i] & 31u)) & 1u) << i;
  }
  return m;
}

// One leaf: bit i of the result <=> row i of the lane's 32 rows lies in the leaf's interval set.
// bm_sbase: shared address of the staged key sets, or kNoStage (global lookups).
constexpr uint32_t kNoStage = 0xFFFFFFFFu;
template <bool TAIL>
__device__ __forceinline__ uint32_t leaf_mask(const void* col, const DevLeaf& L,
                                              const uint64_t* lo_tab, const uint64_t* span_tab,
                                              uint64_t base, int lane, uint32_t nvalid, char* cap,
                                              uint32_t bm_sbase) {
  uint32_t m = 0;
  if (L.wclass == W8) {
#pragma unroll 1  // one instance of the interval loop (see the toolchain note above)
    for (int h = 0; h < 2; ++h) {
      uint64_t v[16];
      load_w8_half<TAIL>(col, base, lane, h, nvalid, v, cap);
      uint32_t mh = 0;
      if (L.pad & kLeafBitmap) {
        const uint64_t sp = span_tab[L.iv_begin];
        mh = (bm_sbase != kNoStage && (L.pad & kLeafStaged))
                 ? bitmap_test_smem<16>(v, bm_sbase + (uint32_t)(sp >> 32), (uint32_t)sp)
                 : bitmap_test<16>(v, lo_tab[L.iv_begin], (uint32_t)sp);
      } else {
        for (int t = 0; t < L.iv_count; ++t) {
          const uint64_t lo = lo_tab[L.iv_begin + t], sp = span_tab[L.iv_begin + t];
#pragma unroll
          for (int i = 0; i < 16; ++i) mh |= (v[i] - lo <= sp) ? (1u << i) : 0u;
        }
      }
      m |= mh << (16 * h);
    }
    return (L.pad & kLeafNegate) ? ~m : m;
  }
  uint32_t v[32];
  if (L.wclass == W4) {
    load_w4<TAIL>(col, base, lane, nvalid, v, cap);
    if (L.fkey) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = fkey(v[i]);
    }
  } else if (L.wclass == W1) {
    load_w1<TAIL>(col, base, lane, nvalid, v, cap);
  } else {
    load_w2<TAIL>(col, base, lane, nvalid, v, cap);
  }
  if (L.pad & kLeafBitmap) {
    const uint64_t sp = span_tab[L.iv_begin];
    m = (bm_sbase != kNoStage && (L.pad & kLeafStaged))
            ? bitmap_test_smem<32>(v, bm_sbase + (uint32_t)(sp >> 32), (uint32_t)sp)
            : bitmap_test<32>(v, lo_tab[L.iv_begin], (uint32_t)sp);
    return (L.pad & kLeafNegate) ? ~m : m;
  }
  for (int t = 0; t < L.iv_count; ++t) {
    const uint32_t lo = (uint32_t)lo_tab[L.iv_begin + t], sp = (uint32_t)span_tab[L.iv_begin + t];
    if (sp == 0) {            // an equality (=, IN value): one compare per row
#pragma unroll
      for (int i = 0; i < 32; ++i) m |= (v[i] == lo) ? (1u << i) : 0u;
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) m |= (v[i] - lo <= sp) ? (1u << i) : 0u;
    }
  }
  return m;
}

template <bool TAIL, bool CAP, class P>
__device__ __forceinline__ uint32_t eval_leaf(const P& p, const DevLeaf& L, uint64_t base,
                                              int lane, uint32_t nvalid, char* wsmem,
                                              uint32_t bm_sbase) {
  const void* col = p.col[L.slot];
  char* cap = (CAP && L.cap) ? wsmem + L.cap_off : nullptr;
  return leaf_mask<TAIL>(col, L, p.lo, p.span, base, lane, nvalid, cap, bm_sbase);
}

// The whole predicate over the lane's 32 rows of the chunk at `base` (nvalid rows valid).
// One eval_leaf call site (conjunctions just AND into an accumulator instead of using the stack),
// so each TAIL variant inlines a single copy of the interval loop (toolchain note above).
template <bool TAIL, bool CAP, class P>
__device__ __forceinline__ uint32_t eval_program(const P& p, uint64_t base, int lane,
                                                 uint32_t nvalid, char* wsmem,
                                                 uint32_t bm_sbase = kNoStage) {
  uint32_t st[kMaxDeviceStack];
  int sp = 0;
  uint32_t acc = 0xFFFFFFFFu;
  const bool conj = p.conj != 0;
#pragma unroll 1
  for (uint32_t i = 0; i < p.n_ops; ++i) {
    const uint8_t op = p.op[i];
    if (op == DOP_LEAF) {
      const uint32_t r = eval_leaf<TAIL, CAP>(p, p.leaf[p.arg[i]], base, lane, nvalid, wsmem, bm_sbase);
      if (conj) acc &= r;
      else st[sp++] = r;
    } else if (!conj) {
      --sp;
      st[sp - 1] = op == DOP_AND ? (st[sp - 1] & st[sp]) : (st[sp - 1] | st[sp]);
    }
  }
  uint32_t m = conj ? acc : st[0];
  if (TAIL) m &= valid_mask(lane, nvalid);
  return m;
}

// ---- count fast path: conjunctions of 1..4 leaves of known kinds --------------------------------
// Straight-line evaluation of a full chunk (no interval loop, no postfix walk): the leaf
// parameters sit in the constant bank at compile-time offsets, so they are hoisted out of the
// chunk loop (uniform registers). One copy per (slot, kind); none contains a dynamic interval loop
// (the toolchain note above concerns that loop).

// 1-byte column, 1..4 point keys, four rows per 32-bit word (SWAR): byte e of x equals the key
// byte iff the high bit of byte e of ~(((t & 0x7F..) + 0x7F..) | t), t = x ^ key, is set (exact:
// no carries cross bytes). The four high bits are gathered into a nibble by one multiply.
__device__ __forceinline__ uint32_t s1_nibble(uint32_t x, const uint32_t (&pts)[4], int npts) {
  uint32_t hit = 0;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    if (t < npts) {
      const uint32_t d = x ^ pts[t];
      hit |= ~(((d & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | d);
    }
  }
  return ((hit & 0x80808080u) * 0x00204081u) >> 28;   // byte e's high bit -> bit e
}

// The coded leaf (p.fast_code; two points) also returns which rows matched point 1 (*wm).
__device__ __forceinline__ uint32_t s1_zero_bytes(uint32_t x, uint32_t pt) {
  const uint32_t d = x ^ pt;
  return ~(((d & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | d);
}
__device__ __forceinline__ uint32_t s1_gather_nibble(uint32_t h) {
  return ((h & 0x80808080u) * 0x00204081u) >> 28;
}

template <bool CAP>
__device__ __forceinline__ uint32_t fast_s1(const void* col, uint64_t base, int lane,
                                            const uint32_t (&pts)[4], int npts, char* cap,
                                            uint32_t* wm) {
  const uint8_t* c = static_cast<const uint8_t*>(col) + base;
  uint32_t x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = ld_stream_u32(c + 4u * (32u * k + lane));
  uint32_t m = 0;
  if (wm) {
    uint32_t w = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (CAP && cap) reinterpret_cast<uint32_t*>(cap)[32 * k + lane] = x[k];
      const uint32_t z1 = s1_zero_bytes(x[k], pts[1]);
      m |= s1_gather_nibble(s1_zero_bytes(x[k], pts[0]) | z1) << (4 * k);
      w |= s1_gather_nibble(z1) << (4 * k);
    }
    *wm = w;
    return m;
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if (CAP && cap) reinterpret_cast<uint32_t*>(cap)[32 * k + lane] = x[k];
    m |= s1_nibble(x[k], pts, npts) << (4 * k);
  }
  return m;
}

// The coded leaf's point-1 matches over a partial (tail) chunk, for keep_chunk.
__device__ __forceinline__ uint32_t which_tail(const void* col, uint64_t base, int lane,
                                               uint32_t nvalid, uint32_t pt1, bool w4) {
  uint32_t v[32];
  if (w4) load_w4<true>(col, base, lane, nvalid, v, nullptr);
  else load_w1<true>(col, base, lane, nvalid, v, nullptr);
  uint32_t m = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) m |= (v[i] == pt1) ? (1u << i) : 0u;
  return m & valid_mask(lane, nvalid);
}

// 4-byte column: one point (E4), one interval (R4) or 2..4 intervals (S4, n = iv_count).
// The coded leaf (S4 with two points) also returns which rows matched point 1 (*wm).
template <int KIND, bool CAP>
__device__ __forceinline__ uint32_t fast_w4(const void* col, uint64_t base, int lane,
                                            const uint64_t* lo, const uint64_t* span, int n,
                                            char* cap, uint32_t* wm = nullptr) {
  uint32_t v[32];
  load_w4<false>(col, base, lane, kChunkRows, v, CAP ? cap : nullptr);
  uint32_t m = 0;
  if (KIND == FK_S4 && wm) {   // two points
    const uint32_t a = (uint32_t)lo[0], b = (uint32_t)lo[1];
    uint32_t m1 = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      m |= (v[i] == a) ? (1u << i) : 0u;
      m1 |= (v[i] == b) ? (1u << i) : 0u;
    }
    *wm = m1;
    return m | m1;
  }
  if (KIND == FK_E4) {
    const uint32_t a = (uint32_t)lo[0];
#pragma unroll
    for (int i = 0; i < 32; ++i) m |= (v[i] == a) ? (1u << i) : 0u;
  } else if (KIND == FK_R4) {
    const uint32_t a = (uint32_t)lo[0], b = (uint32_t)span[0];
#pragma unroll
    for (int i = 0; i < 32; ++i) m |= (v[i] - a <= b) ? (1u << i) : 0u;
  } else {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if (t < n) {
        const uint32_t a = (uint32_t)lo[t], b = (uint32_t)span[t];
#pragma unroll
        for (int i = 0; i < 32; ++i) m |= (v[i] - a <= b) ? (1u << i) : 0u;
      }
    }
  }
  return m;
}

// 8-byte column, one interval.
template <bool CAP>
__device__ __forceinline__ uint32_t fast_r8(const void* col, uint64_t base, int lane, uint64_t a,
                                            uint64_t b, char* cap) {
  uint32_t m = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    uint64_t v[16];
    load_w8_half<false>(col, base, lane, h, kChunkRows, v, CAP ? cap : nullptr);
#pragma unroll
    for (int i = 0; i < 16; ++i) m |= (v[i] - a <= b) ? (1u << (16 * h + i)) : 0u;
  }
  return m;
}

template <int FASTN, bool CAP, class P>
__device__ __forceinline__ uint32_t eval_fast(const P& p, uint64_t base, int lane, char* wsmem,
                                              uint32_t* wm) {
  uint32_t acc = 0xFFFFFFFFu;
#pragma unroll
  for (int s = 0; s < FASTN; ++s) {
    const DevLeaf& L = p.leaf[s];
    const void* col = p.col[L.slot];
    char* cap = (CAP && L.cap) ? wsmem + L.cap_off : nullptr;
    const uint64_t* lo = p.lo + L.iv_begin;
    const uint64_t* sp = p.span + L.iv_begin;
    uint32_t r;
    switch (p.fast_kind[s]) {
      case FK_E4: r = fast_w4<FK_E4, CAP>(col, base, lane, lo, sp, 1, cap); break;
      case FK_R4: r = fast_w4<FK_R4, CAP>(col, base, lane, lo, sp, 1, cap); break;
      case FK_S4:
        r = fast_w4<FK_S4, CAP>(col, base, lane, lo, sp, L.iv_count, cap,
                                p.fast_code == s ? wm : nullptr);
        break;
      case FK_R8: r = fast_r8<CAP>(col, base, lane, lo[0], sp[0], cap); break;
      default:
        r = fast_s1<CAP>(col, base, lane, p.fast_pts[s], p.fast_npts[s], cap,
                         p.fast_code == s ? wm : nullptr);
        break;
    }
    acc &= r;
  }
  return acc;
}

// L2 prefetch of a chunk's predicate columns, fast path (compile-time leaf count).
template <int FASTN, class P>
__device__ __forceinline__ void prefetch_chunk_fast(const P& p, uint64_t c) {
#pragma unroll
  for (int s = 0; s < FASTN; ++s) {
    const uint32_t w = 1u << p.leaf[s].wclass;
    prefetch_l2(static_cast<const char*>(p.col[p.leaf[s].slot]) + c * kChunkRows * w, kChunkRows * w);
  }
}

// ---- push-down ------------------------------------------------------------------------------
constexpr uint64_t kFlagAgg = 1, kFlagPrefix = 2;
__device__ __forceinline__ uint64_t pack_status(uint32_t epoch, uint64_t flag, uint32_t value) {
  return ((uint64_t)epoch << 34) | (flag << 32) | value;
}

// Write-out of a projected column gathered from global memory (non-predicate columns): the
// chunk-local rows s_idx[0..lim) ascending; batches of 8 loads in flight per lane before stores.
#ifndef SEL_GATHER_BATCH
#define SEL_GATHER_BATCH 8   // loads in flight per lane (A/B: 4 equal, 16 slower on C2)
#endif
template <class T, bool MASK = false>
__device__ __forceinline__ void gather_global(const void* src_v, void* dst_v, uint64_t cbase,
                                              uint64_t gbase, const uint16_t* s_idx, uint32_t lim,
                                              int lane) {
  constexpr int B = SEL_GATHER_BATCH;
  const T* __restrict__ src = static_cast<const T*>(src_v) + cbase;
  T* __restrict__ dst = static_cast<T*>(dst_v) + gbase;
  uint32_t q = lane;
  for (; q + (B - 1) * 32 < lim; q += B * 32) {
    T v[B];
#pragma unroll
    for (int u = 0; u < B; ++u) v[u] = __ldg(src + (MASK ? (s_idx[q + 32 * u] & (kCodeBit - 1u)) : s_idx[q + 32 * u]));
#pragma unroll
    for (int u = 0; u < B; ++u) dst[q + 32 * u] = v[u];
  }
  for (; q < lim; q += 32) dst[q] = __ldg(src + (MASK ? (s_idx[q] & (kCodeBit - 1u)) : s_idx[q]));
}

// Write-out of a projected predicate column from its shared-memory capture.
template <class T>
__device__ __forceinline__ void gather_smem(const char* cap, void* dst_v, uint64_t gbase,
                                            const uint16_t* s_idx, uint32_t lim, int lane) {
  const T* src = reinterpret_cast<const T*>(cap);
  T* __restrict__ dst = static_cast<T*>(dst_v) + gbase;
#pragma unroll 4
  for (uint32_t q = lane; q < lim; q += 32) dst[q] = src[s_idx[q]];
}

// Coalesced write-out of one chunk's compacted rows: output positions [gbase, gbase + cnt) receive
// the chunk-local rows s_idx[0..cnt) (ascending), truncated at the capacity (Algorithm 1's gate).
template <class T>
__device__ __forceinline__ void copy_slot(const void* slot_v, void* dst_v, uint64_t cbase,
                                          uint64_t gbase, uint32_t lim, int lane) {
  const T* __restrict__ src = static_cast<const T*>(slot_v) + cbase;
  T* __restrict__ dst = static_cast<T*>(dst_v) + gbase;
#pragma unroll 4
  for (uint32_t q = lane; q < lim; q += 32) dst[q] = src[q];
}

// Output positions [gbase, gbase + lim) of a constant projection receive its value.
template <class T>
__device__ __forceinline__ void fill_const(uint64_t bits, void* dst_v, uint64_t gbase, uint32_t lim,
                                           int lane) {
  T* __restrict__ dst = static_cast<T*>(dst_v) + gbase;
  const T v = (T)bits;
#pragma unroll 4
  for (uint32_t q = lane; q < lim; q += 32) dst[q] = v;
}
__device__ __forceinline__ void fill_proj(uint8_t wclass, const void* bits, void* dst, uint64_t gbase,
                                          uint32_t lim, int lane) {
  const uint64_t b = (uint64_t)(uintptr_t)bits;
  switch (wclass) {
    case W1: fill_const<uint8_t>(b, dst, gbase, lim, lane); break;
    case W2: fill_const<uint16_t>(b, dst, gbase, lim, lane); break;
    case W4: fill_const<uint32_t>(b, dst, gbase, lim, lane); break;
    default: fill_const<uint64_t>(b, dst, gbase, lim, lane); break;
  }
}

// proj_cap_off >= kKeptBase: projection j comes from kept slot (proj_cap_off - kKeptBase).
template <class P>
__device__ __forceinline__ void write_out(const P& p, uint64_t cbase, uint64_t gbase, uint32_t cnt,
                                          const uint16_t* my, const char* wsmem, int lane,
                                          uint32_t* __restrict__ out_ids,
                                          const SelectionBufs* kept = nullptr) {
  if (gbase >= p.capacity) return;
  const uint32_t lim = (uint32_t)min((uint64_t)cnt, p.capacity - gbase);
  const uint32_t idbase = (uint32_t)(p.row_offset + cbase);
#pragma unroll 4
  for (uint32_t q = lane; q < lim; q += 32) out_ids[gbase + q] = idbase + my[q];
#pragma unroll 1
  for (uint32_t j = 0; j < p.n_proj; ++j) {
    const uint16_t co = p.proj_cap_off[j];
    if (co == kConstProj) {
      fill_proj(p.proj_wclass[j], p.proj_src[j], p.proj_dst[j], gbase, lim, lane);
    } else if (kept && co != kNoCapture) {
      const void* slot = kept->keep_slot[co - kKeptBase];
      switch (p.proj_wclass[j]) {
        case W1: copy_slot<uint8_t>(slot, p.proj_dst[j], cbase, gbase, lim, lane); break;
        case W2: copy_slot<uint16_t>(slot, p.proj_dst[j], cbase, gbase, lim, lane); break;
        case W4: copy_slot<uint32_t>(slot, p.proj_dst[j], cbase, gbase, lim, lane); break;
        default: copy_slot<uint64_t>(slot, p.proj_dst[j], cbase, gbase, lim, lane); break;
      }
    } else if (co != kNoCapture) {
      const char* cap = wsmem + co;
      switch (p.proj_wclass[j]) {
        case W1: gather_smem<uint8_t>(cap, p.proj_dst[j], gbase, my, lim, lane); break;
        case W2: gather_smem<uint16_t>(cap, p.proj_dst[j], gbase, my, lim, lane); break;
        case W4: gather_smem<uint32_t>(cap, p.proj_dst[j], gbase, my, lim, lane); break;
        default: gather_smem<uint64_t>(cap, p.proj_dst[j], gbase, my, lim, lane); break;
      }
    } else {
      switch (p.proj_wclass[j]) {
        case W1: gather_global<uint8_t>(p.proj_src[j], p.proj_dst[j], cbase, gbase, my, lim, lane); break;
        case W2: gather_global<uint16_t>(p.proj_src[j], p.proj_dst[j], cbase, gbase, my, lim, lane); break;
        case W4: gather_global<uint32_t>(p.proj_src[j], p.proj_dst[j], cbase, gbase, my, lim, lane); break;
        default: gather_global<uint64_t>(p.proj_src[j], p.proj_dst[j], cbase, gbase, my, lim, lane); break;
      }
    }
  }
}

// Stage the chunk-local indices of the rows selected by the lanes' masks, ascending; returns the
// chunk's count. Positions come from a warp scan of per-quad-stripe popcounts, 4 stripes of 8 bits
// per word (fields <= 128 never carry).
__device__ __forceinline__ uint32_t stage_indices(uint32_t m, int lane, uint16_t* my) {
  uint32_t cw0 = 0, cw1 = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    cw0 |= (uint32_t)__popc((m >> (4 * k)) & 0xFu) << (8 * k);
    cw1 |= (uint32_t)__popc((m >> (4 * (k + 4))) & 0xFu) << (8 * k);
  }
  uint32_t ex0 = cw0, ex1 = cw1;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t t0 = __shfl_up_sync(0xFFFFFFFFu, ex0, d);
    const uint32_t t1 = __shfl_up_sync(0xFFFFFFFFu, ex1, d);
    if (lane >= d) { ex0 += t0; ex1 += t1; }
  }
  const uint32_t tot0 = __shfl_sync(0xFFFFFFFFu, ex0, 31), tot1 = __shfl_sync(0xFFFFFFFFu, ex1, 31);
  ex0 -= cw0;
  ex1 -= cw1;
  uint32_t acc = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t nib = (m >> (4 * k)) & 0xFu;
    uint32_t pos = acc + (((k < 4 ? ex0 : ex1) >> (8 * (k & 3))) & 0xFFu);
    acc += ((k < 4 ? tot0 : tot1) >> (8 * (k & 3))) & 0xFFu;
    if (nib == 0) continue;
    const uint32_t r0 = 4u * (32u * k + lane);
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (nib & (1u << e)) my[pos++] = (uint16_t)(r0 + e);
  }
  return acc;
}

// ---- count ----------------------------------------------------------------------------------
// Persistent grid-stride over warp-chunks; per-lane popc, warp redux, CTA reduction, one partial
// per CTA; the last CTA to finish sums the partials (self-resetting: no memset between probes).
// KEEP (sel_count_ex with SEL_KEEP_SELECTION): the chunk's row mask (one u32 per lane, 128 B per
// 1024 rows) and its count are also kept, plus per-64-chunk sums, so that a following push-down
// of the same predicate materialises from the selection without re-evaluating it (PAPER.md:329:
// materialise right after the count, reusing the scan already done on the GPU). With kept value
// columns (the compound's projected predicate columns, known before the count: ExtractPushDown
// returns conditions AND columns) the values loaded for the predicate are
// captured in shared memory and the chunk's selected ones written, compacted, to its slot.
// Stage the rows of one chunk from its ROW-MAJOR kept masks (lane L: rows 32L..32L+31) at
// my[base..] as block-relative rows, ascending: one warp scan of per-lane popcounts, then each lane
// walks its set bits.
__device__ __forceinline__ void stage_rows_rm(uint32_t t, int lane, uint16_t* my, uint32_t base,
                                              uint32_t row_base) {
  const uint32_t c = (uint32_t)__popc(t);
  uint32_t incl = c;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, d);
    if (lane >= d) incl += v;
  }
  uint32_t pos = base + incl - c;
  const uint32_t r0 = row_base + 32u * lane;
  while (t) {
    const uint32_t b = (uint32_t)(__ffs(t) - 1);
    t &= t - 1;
    my[pos++] = (uint16_t)(r0 + b);
  }
}

// stage_rows_rm carrying each row's code bit (row-major word w of the coded leaf) in kCodeBit.
__device__ __forceinline__ void stage_rows_rm_coded(uint32_t t, uint32_t w, int lane, uint16_t* my,
                                                    uint32_t base, uint32_t row_base) {
  const uint32_t c = (uint32_t)__popc(t);
  uint32_t incl = c;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, d);
    if (lane >= d) incl += v;
  }
  uint32_t pos = base + incl - c;
  const uint32_t r0 = row_base + 32u * lane;
  while (t) {
    const uint32_t b = (uint32_t)(__ffs(t) - 1);
    t &= t - 1;
    my[pos++] = (uint16_t)((r0 + b) | (((w >> b) & 1u) ? kCodeBit : 0u));
  }
}

// Quad layout (bit 4k+e of lane l = row 4(32k+l)+e) -> row-major (bit b of lane L = row 32L+b):
// lane L = 4k + j gathers nibble k of lanes 8j..8j+7 (row 128k + 32j + 4i + e = 32L + 4i + e).
__device__ __forceinline__ uint32_t to_row_major(uint32_t m, int lane) {
  const int k = lane >> 2, j = lane & 3;
  uint32_t t = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t v = __shfl_sync(0xFFFFFFFFu, m, 8 * j + i);
    t |= ((v >> (4 * k)) & 0xFu) << (4 * i);
  }
  return t;
}

__device__ __forceinline__ void st_evict_last(uint32_t* p, uint32_t v) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
}

// coded: also keep the coded leaf's point-1 matches (wm, the count's quad layout) row-major.
template <class P, bool KEEP>
// Returns the chunk's selected-row count (every lane; 0 without KEEP).
__device__ __forceinline__ uint32_t keep_chunk(const SelectionBufs& sb, uint32_t* sbs, uint64_t c, int lane,
                                               uint32_t m, char* wsmem, uint32_t wm = 0u,
                                               bool coded = false) {
  if (!KEEP) return 0u;
  if (coded) st_evict_last(sb.which + c * 32 + lane, to_row_major(wm, lane));
  const uint32_t t = to_row_major(m, lane);          // the push-down stages from row-major masks
  if (sb.n_keep) {
    sb.bits[c * 32 + lane] = t;
  } else {
    // Selection only: the masks (n/8 bytes) stay in L2 for the push-down that follows instead of
    // being written back while the scan streams its columns (measured: C5 count 0.638 -> 0.629
    // ms, C4 push-down 0.176 -> 0.160 ms). With kept values the slots compete for L2 and the
    // policy hurt (C2 0.913 -> 0.968 ms), so it is not used there.
    st_evict_last(sb.bits + c * 32 + lane, t);
  }
  uint32_t cc;
  if (sb.n_keep) {
    uint16_t* my = reinterpret_cast<uint16_t*>(wsmem);
    stage_rows_rm(t, lane, my, 0u, 0u);
    cc = __reduce_add_sync(0xFFFFFFFFu, (uint32_t)__popc(t));
    __syncwarp();
#pragma unroll 1
    for (uint32_t k = 0; k < sb.n_keep; ++k) {
      const char* cap = wsmem + sb.keep_cap_off[k];
      switch (sb.keep_wclass[k]) {
        case W1: gather_smem<uint8_t>(cap, sb.keep_slot[k], c * kChunkRows, my, cc, lane); break;
        case W2: gather_smem<uint16_t>(cap, sb.keep_slot[k], c * kChunkRows, my, cc, lane); break;
        case W4: gather_smem<uint32_t>(cap, sb.keep_slot[k], c * kChunkRows, my, cc, lane); break;
        default: gather_smem<uint64_t>(cap, sb.keep_slot[k], c * kChunkRows, my, cc, lane); break;
      }
    }
    __syncwarp();
  } else {
    cc = __reduce_add_sync(0xFFFFFFFFu, (uint32_t)__popc(m));
  }
  if (lane == 0) {
    sb.chunk_cnt[c] = (uint16_t)cc;
    if (cc) atomicAdd(sbs + (c >> kSbShift), cc);
  }
  return cc;
}

// NW warps per CTA: 8 normally; 32 when staged key sets leave room for one CTA per SM only.
// FASTN > 0: the program is a conjunction of FASTN fast-path leaves (p.fast_n == FASTN).
template <class P, bool KEEP, int NW, int FASTN = 0>
#ifndef SEL_FAST_MINB
#define SEL_FAST_MINB 3   // fast path: <= 85 registers (A/B: 2-6; 3 best on C2, C4, C5)
#endif
__global__ void __launch_bounds__(NW * 32, NW == kWarpsPerCta ? (FASTN ? SEL_FAST_MINB : 4) : 1) count_kernel(const __grid_constant__ P p, uint64_t n,
                                                         uint64_t* __restrict__ partials,
                                                         unsigned int* __restrict__ done,
                                                         uint64_t* __restrict__ out,
                                                         SelectionBufs sb, const PeerXchg xg,
                                                         const ExecFinish fin) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t nfull = n / kChunkRows;
  const uint32_t rem = (uint32_t)(n % kChunkRows);
  const uint64_t gw = (uint64_t)blockIdx.x * NW + warp;
  const uint64_t nw = (uint64_t)gridDim.x * NW;
  extern __shared__ __align__(16) char s_dyn[];
  char* wsmem = KEEP ? s_dyn + (size_t)warp * sb.warp_smem : nullptr;
  uint32_t cnt = 0;
  bool full = false;   // this warp kept a fully selected chunk (raises the flag once, below)
  // keeping counts: this count's half of the superblock sums (zero: the count before the last one
  // used it), and the other half — the previous selection's, dead from here on — zeroed for the
  // next count while this one runs
  uint32_t epoch = 0;
  uint32_t* my_sb = nullptr;
  if constexpr (KEEP) {
    epoch = *(volatile const uint32_t*)sb.state;
    my_sb = sb.sb_sum + (size_t)(epoch & 1u) * sb.sb_stride;
    uint32_t* other = sb.sb_sum + (size_t)((epoch + 1u) & 1u) * sb.sb_stride;
    const uint32_t ext = sb.state[1 + ((epoch + 1u) & 1u)];
    for (uint32_t i = blockIdx.x * (NW * 32) + threadIdx.x; i < ext; i += gridDim.x * (NW * 32))
      other[i] = 0u;
  }
  // Stage the program's key sets in shared memory (after the warps' areas), once per CTA.
  uint32_t bm_sbase = kNoStage;
  if (p.bm_smem) {
    char* area = s_dyn + (KEEP ? (size_t)NW * sb.warp_smem : 0);
#pragma unroll 1
    for (uint32_t l = 0; l < p.n_leaves; ++l) {
      const DevLeaf& L = p.leaf[l];
      if (!(L.pad & kLeafStaged)) continue;
      const uint64_t sp = p.span[L.iv_begin];
      const uint64_t* src = reinterpret_cast<const uint64_t*>(p.lo[L.iv_begin]);
      uint64_t* dst = reinterpret_cast<uint64_t*>(area + (uint32_t)(sp >> 32));
      const uint32_t nwords = ((uint32_t)sp + 63u) >> 6;
#pragma unroll 8
      for (uint32_t i = threadIdx.x; i < nwords; i += (NW * 32)) dst[i] = __ldg(src + i);
    }
    __syncthreads();
    bm_sbase = (uint32_t)__cvta_generic_to_shared(area);
  }
  // Chunks scanned: c = phase + s * stride (stride 1, phase 0: every chunk). A stride > 1 is the
  // block sample of sel_count_sampled; keeping a selection needs stride 1.
  const uint64_t stride = p.chunk_stride, phase = p.chunk_phase;
  const uint64_t ns_full = nfull > phase ? (nfull - phase + stride - 1) / stride : 0;
  const bool tail_sampled = rem != 0 && nfull >= phase && (nfull - phase) % stride == 0;
  if constexpr (FASTN > 0) {
    if (lane == 0 && p.prefetch && gw < ns_full) prefetch_chunk_fast<FASTN>(p, phase + gw * stride);
    for (uint64_t s = gw; s < ns_full; s += nw) {
      const uint64_t c = phase + s * stride;
      if (lane == 0 && p.prefetch && s + nw < ns_full) prefetch_chunk_fast<FASTN>(p, c + nw * stride);
      uint32_t wm = 0;
      const uint32_t m = eval_fast<FASTN, KEEP>(p, c * kChunkRows, lane, wsmem, &wm);
      cnt += __popc(m);
      full |= keep_chunk<P, KEEP>(sb, my_sb, c, lane, m, wsmem, wm, KEEP && p.fast_code >= 0) == kChunkRows;
    }
  } else {
    if (lane == 0 && p.prefetch && gw < ns_full) prefetch_chunk(p, phase + gw * stride);
    for (uint64_t s = gw; s < ns_full; s += nw) {
      const uint64_t c = phase + s * stride;
      if (lane == 0 && p.prefetch && s + nw < ns_full) prefetch_chunk(p, c + nw * stride);
      const uint32_t m = eval_program<false, KEEP>(p, c * kChunkRows, lane, kChunkRows, wsmem, bm_sbase);
      cnt += __popc(m);
      full |= keep_chunk<P, KEEP>(sb, my_sb, c, lane, m, wsmem) == kChunkRows;
    }
  }
  if (tail_sampled && gw == ns_full % nw) {
    const uint32_t m = eval_program<true, KEEP>(p, nfull * kChunkRows, lane, rem, wsmem, bm_sbase);
    cnt += __popc(m);
    uint32_t wm = 0;
    const bool coded = KEEP && FASTN > 0 && p.fast_code >= 0;
    if (coded) {
      const int s = p.fast_code;
      const bool w4 = p.fast_kind[s] == FK_S4;
      const uint32_t pt1 = w4 ? (uint32_t)p.lo[p.leaf[s].iv_begin + 1] : (p.fast_pts[s][1] & 0xFFu);
      wm = which_tail(p.col[p.leaf[s].slot], nfull * kChunkRows, lane, rem, pt1, w4);
    }
    keep_chunk<P, KEEP>(sb, my_sb, nfull, lane, m, wsmem, wm, coded);   // a tail chunk is never full
  }
  // dense_chunks_kernel has work: one store per warp (one per chunk contended on the word: C5 at
  // s = 1 count 0.62 -> 1.36 ms)
  if (KEEP && full && lane == 0) sb.state[3] = 1u;
  cnt = __reduce_add_sync(0xFFFFFFFFu, cnt);
  // the superblock atomics and the full-chunk flag (lane 0 of each warp) are read by the last CTA
  // (finish_selection); the masks are read by later kernels only
  if (KEEP && lane == 0) __threadfence();

  __shared__ uint32_t s_warp[NW];
  __shared__ bool s_last;
  if (lane == 0) s_warp[warp] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t s = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += s_warp[w];
    partials[blockIdx.x] = s;
    __threadfence();
    s_last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    uint64_t local;
    if constexpr (KEEP) {
      // keeping counts: the hyperblock prefix the push-down starts from (no kernel in between);
      // its total is the local count
      local = finish_selection<NW>(sb, n, epoch, my_sb);
      if (threadIdx.x == 0) {
        *out = local;
        *done = 0u;
      }
    } else {
      uint64_t s = 0;
      for (uint32_t b = threadIdx.x; b < gridDim.x; b += (NW * 32)) s += ((volatile uint64_t*)partials)[b];
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
      __shared__ uint64_t s_sum[NW];
      __shared__ uint64_t s_total;
      if (lane == 0) s_sum[warp] = s;
      __syncthreads();
      if (threadIdx.x == 0) {
        uint64_t t = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) t += s_sum[w];
        *out = t;
        *done = 0u;
        s_total = t;
      }
      __syncthreads();
      local = s_total;
    }
    if (fin.result) {
      // a device-gated Execute: its result words (and, with peers, the exchange) right here
      __syncthreads();
      finish_execute(fin, xg, local);
    } else {
      if (xg.n > 0) {
        // sel_count with peers: the count's collective fused into the same kernel — the last CTA
        // exchanges the local count over peer memory and leaves the global sum in *out
        __syncthreads();
        peer_gather_block(xg, out, 1, nullptr, out);
      }
      // sel_count: the count straight into the pinned host word (no copy after the kernel)
      if (fin.host && threadIdx.x == 0) fin.host[0] = *out;
    }
  }
}

// Warp-granular single-pass compaction. Every warp runs independently (no CTA barriers): it draws
// a 1024-row tile from a global ticket counter (tickets are handed out in order, so every tile a
// warp waits on belongs to a warp that is already running: forward progress), evaluates the
// predicate (capturing projected predicate columns into its shared-memory area), scans its
// per-stripe counts, publishes its aggregate, resolves its exclusive prefix by decoupled
// look-back over up to 32 predecessors per step, publishes the inclusive prefix, stages the
// ascending chunk-local indices of the selected rows and writes row ids + projected columns with
// coalesced stores. Dynamic shared memory per warp: [u16 s_idx[1024] | captures].
template <class P>
__global__ void __launch_bounds__(kThreads, 3) pushdown_kernel(
    const __grid_constant__ P p, uint64_t n, uint32_t* __restrict__ out_ids,
    unsigned long long* __restrict__ ticket, uint64_t ticket_base, uint64_t* __restrict__ status,
    uint32_t epoch, uint64_t* __restrict__ out_count) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t ntiles = (n + kChunkRows - 1) / kChunkRows;
  extern __shared__ __align__(16) char s_dyn[];
  char* wsmem = s_dyn + (size_t)warp * p.warp_smem;
  uint16_t* my = reinterpret_cast<uint16_t*>(wsmem);

  for (;;) {
    unsigned long long tk = 0;
    if (lane == 0) tk = atomicAdd(ticket, 1ull);
    const uint64_t tile = __shfl_sync(0xFFFFFFFFu, tk, 0) - ticket_base;
    if (tile >= ntiles) break;
    const uint64_t cbase = tile * kChunkRows;
    const uint32_t nvalid = n - cbase >= (uint64_t)kChunkRows ? (uint32_t)kChunkRows : (uint32_t)(n - cbase);

    // 1. evaluate (and capture)
    const uint32_t m = nvalid == kChunkRows ? eval_program<false, true>(p, cbase, lane, kChunkRows, wsmem)
                                            : eval_program<true, true>(p, cbase, lane, nvalid, wsmem);

    // 2. stage the chunk-local indices of the selected rows (ascending) and count them
    const uint32_t acc = stage_indices(m, lane, my);
    __syncwarp();

    // 3. publish the aggregate, look back for the exclusive prefix, publish the inclusive prefix
    uint64_t excl = 0;
    if (tile == 0) {
      if (lane == 0) st_relaxed_u64(&status[0], pack_status(epoch, kFlagPrefix, acc));
    } else {
      if (lane == 0) st_relaxed_u64(&status[tile], pack_status(epoch, kFlagAgg, acc));
      int64_t j = (int64_t)tile - 1;
      for (;;) {
        const int64_t idx = j - lane;
        const uint64_t sw = idx >= 0 ? ld_relaxed_u64(&status[idx]) : pack_status(epoch, kFlagPrefix, 0);
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
      if (lane == 0) st_relaxed_u64(&status[tile], pack_status(epoch, kFlagPrefix, (uint32_t)(excl + acc)));
    }
    if (tile == ntiles - 1 && lane == 0) *out_count = excl + acc;
    // 4. coalesced write-out of the tile's slice, honouring the capacity gate
    if (acc != 0) write_out(p, cbase, excl, acc, my, wsmem, lane, out_ids);
    __syncwarp();  // `my` and the captures are rewritten by the next tile
  }
}


// ---- push-down from a kept selection ------------------------------------------------------------

// Exclusive prefix of the per-64-chunk sums kept by the count kernel (one CTA; <= 65536 sums).
__global__ void __launch_bounds__(256) peer_exchange_kernel(const PeerXchg x, const uint64_t* src,
                                                            int k, uint64_t* out, uint64_t* sums) {
  peer_gather_block(x, src, k, out, sums);
}

// The kept selection's local count into result[0] and the result words of ExecFinish (sel_execute
// with a communicator: after the all-gather of the per-rank counts; sel_pushdown from a kept
// selection: the local count only). One CTA.
__global__ void __launch_bounds__(256) selection_result_kernel(const uint32_t* __restrict__ hb_prefix,
                                                               uint32_t nhb, const ExecFinish f,
                                                               const PeerXchg xg) {
  const uint64_t local = hb_prefix[nhb];
  if (threadIdx.x == 0) f.result[0] = local;
  finish_execute(f, xg, local);
}

// Flush `k` staged rows (block-relative, ascending) to output positions [gbase, gbase + k): row
// ids and the projections gathered from global memory (kept-value projections were copied per
// chunk while staging).
template <bool CODED, class P>
__device__ __forceinline__ void flush_rows(const P& p, uint64_t bbase, uint64_t gbase, uint32_t k,
                                           const uint16_t* my, int lane,
                                           uint32_t* __restrict__ out_ids) {
  if (gbase >= p.capacity || k == 0) return;
  const uint32_t lim = (uint32_t)min((uint64_t)k, p.capacity - gbase);
  const uint32_t idbase = (uint32_t)(p.row_offset + bbase);
#pragma unroll 4
  for (uint32_t q = lane; q < lim; q += 32)
    out_ids[gbase + q] = idbase + (CODED ? (my[q] & (kCodeBit - 1u)) : my[q]);
#pragma unroll 1
  for (uint32_t j = 0; j < p.n_proj; ++j) {
    if (CODED && p.proj_cap_off[j] == kCodedProj) {   // the value from the row's code bit, nothing read
      const uint64_t pts = (uint64_t)(uintptr_t)p.proj_src[j];
      if (p.proj_wclass[j] == W1) {
        uint8_t* __restrict__ dst = static_cast<uint8_t*>(p.proj_dst[j]) + gbase;
#pragma unroll 4
        for (uint32_t q = lane; q < lim; q += 32) dst[q] = (uint8_t)(pts >> ((my[q] & kCodeBit) ? 8 : 0));
      } else {
        uint32_t* __restrict__ dst = static_cast<uint32_t*>(p.proj_dst[j]) + gbase;
#pragma unroll 4
        for (uint32_t q = lane; q < lim; q += 32) dst[q] = (uint32_t)(pts >> ((my[q] & kCodeBit) ? 32 : 0));
      }
      continue;
    }
    if (p.proj_cap_off[j] != kNoCapture) continue;
    switch (p.proj_wclass[j]) {
      case W1: gather_global<uint8_t, CODED>(p.proj_src[j], p.proj_dst[j], bbase, gbase, my, lim, lane); break;
      case W2: gather_global<uint16_t, CODED>(p.proj_src[j], p.proj_dst[j], bbase, gbase, my, lim, lane); break;
      case W4: gather_global<uint32_t, CODED>(p.proj_src[j], p.proj_dst[j], bbase, gbase, my, lim, lane); break;
      default: gather_global<uint64_t, CODED>(p.proj_src[j], p.proj_dst[j], bbase, gbase, my, lim, lane); break;
    }
  }
}

// Copy chunk c's kept values of the projections that have them to output positions [pos, pos+cnt).
template <class P>
__device__ __forceinline__ void copy_kept(const P& p, const SelectionBufs& sb, uint64_t c,
                                          uint64_t pos, uint32_t cnt, int lane) {
  if (pos >= p.capacity) return;
  const uint32_t lim = (uint32_t)min((uint64_t)cnt, p.capacity - pos);
#pragma unroll 1
  for (uint32_t j = 0; j < p.n_proj; ++j) {
    const uint16_t co = p.proj_cap_off[j];
    if (co == kNoCapture || co == kCodedProj) continue;
    if (co == kConstProj) {
      fill_proj(p.proj_wclass[j], p.proj_src[j], p.proj_dst[j], pos, lim, lane);
      continue;
    }
    const void* slot = sb.keep_slot[co - kKeptBase];
    switch (p.proj_wclass[j]) {
      case W1: copy_slot<uint8_t>(slot, p.proj_dst[j], c * kChunkRows, pos, lim, lane); break;
      case W2: copy_slot<uint16_t>(slot, p.proj_dst[j], c * kChunkRows, pos, lim, lane); break;
      case W4: copy_slot<uint32_t>(slot, p.proj_dst[j], c * kChunkRows, pos, lim, lane); break;
      default: copy_slot<uint64_t>(slot, p.proj_dst[j], c * kChunkRows, pos, lim, lane); break;
    }
  }
}

#ifndef SEL_STAGE_CAP
#define SEL_STAGE_CAP 1024
#endif
#ifndef SEL_PD_MINB
#define SEL_PD_MINB 8
#endif
constexpr int kBlockChunks = kSelBlockChunks;          // whole-chunk copy kernel: chunks per warp block
constexpr uint32_t kStageCap = SEL_STAGE_CAP;          // staged rows per warp before a flush

// Warp blocks of 4 contiguous chunks, grid-stride. All of a block's metadata — its 4 chunk counts,
// the lane's 4 mask words and the counts of the preceding chunks of its 64-chunk superblock —
// are independent loads issued together (one round trip). The block's output base is the
// superblock prefix plus that partial sum; empty chunks are skipped without touching any column;
// the selected rows of the block are staged and flushed with batched gathers into one contiguous
// output range. No ticket, no look-back, no predicate evaluation.
template <class P, bool CODED, int BC>
__global__ void __launch_bounds__(kThreads, SEL_PD_MINB) pushdown_sel_kernel(const __grid_constant__ P p,
                                                                   uint64_t n, SelectionBufs sb,
                                                                   uint32_t* __restrict__ out_ids,
                                                                   const uint64_t* __restrict__ gate_count) {
  // Algorithm 1's "throw" (nothing written), or a failed peer exchange (kXchgFailed)
  if (*gate_count == kXchgFailed || (p.gate && *gate_count > p.gate_max)) return;
  // sel_execute_to: positions in the global result start at this rank's offset (prefix kernel)
  const uint64_t goff = p.global_out ? gate_count[kOffsetSlot - kGateSlot] : 0ull;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  static_assert(BC * kChunkRows <= kCodeBit, "staged rows must leave the code bit free");
  __shared__ uint16_t s_stage[kWarpsPerCta][kStageCap];
  uint16_t* my = s_stage[warp];
  const uint64_t nchunks = (n + kChunkRows - 1) / kChunkRows;
  const uint64_t nblocks = (nchunks + BC - 1) / BC;
  const uint64_t gw = (uint64_t)blockIdx.x * kWarpsPerCta + warp;
  const uint64_t nw = (uint64_t)gridDim.x * kWarpsPerCta;
  const uint32_t* sbs = kept_sb(sb);
  for (uint64_t blk = gw; blk < nblocks; blk += nw) {
    const uint64_t c0 = blk * BC;
    // --- metadata, all loads independent ---
    const uint32_t cntv = (lane < BC && c0 + lane < nchunks) ? sb.chunk_cnt[c0 + lane] : 0u;
    uint32_t m[BC];
#pragma unroll
    for (int g = 0; g < BC; ++g) m[g] = c0 + g < nchunks ? sb.bits[(c0 + g) * 32 + lane] : 0u;
    // the count stored the masks evict_last (keep_chunk): hand their L2 lines back to the normal
    // replacement order once read (one 128-byte line per chunk)
    if (sb.n_keep == 0 && lane < BC && c0 + lane < nchunks)
      asm volatile("applypriority.global.L2::evict_normal [%0], 128;" ::"l"(sb.bits + (c0 + lane) * 32) : "memory");
    if (CODED && lane < BC && c0 + lane < nchunks)
      asm volatile("applypriority.global.L2::evict_normal [%0], 128;" ::"l"(sb.which + (c0 + lane) * 32) : "memory");
    const uint64_t kb = kept_base(sb, sbs, c0, lane);
    // --- offsets ---
    const uint32_t total = __reduce_add_sync(0xFFFFFFFFu, cntv);
    if (total == 0) continue;
    uint64_t gbase = goff + kb;
    const uint64_t bbase = c0 * kChunkRows;
    uint32_t staged = 0;
#pragma unroll
    for (int g = 0; g < BC; ++g) {
      const uint32_t cg = __shfl_sync(0xFFFFFFFFu, cntv, g);
      if (cg == 0) continue;
      if (p.dense_split && cg == kChunkRows && gbase + staged + kChunkRows <= p.capacity) {
        __syncwarp();   // a full chunk is copied whole by dense_chunks_kernel: skip its positions
        flush_rows<CODED>(p, bbase, gbase, staged, my, lane, out_ids);
        __syncwarp();
        gbase += staged + kChunkRows;
        staged = 0;
        continue;
      }
      if (staged + cg > kStageCap) {
        __syncwarp();
        flush_rows<CODED>(p, bbase, gbase, staged, my, lane, out_ids);
        __syncwarp();
        gbase += staged;
        staged = 0;
      }
      if (p.n_direct) copy_kept(p, sb, c0 + g, gbase + staged, cg, lane);  // kept / constant
      if (CODED)   // the coded leaf's word, read when the chunk is staged (L2: stored evict_last)
        stage_rows_rm_coded(m[g], sb.which[(c0 + g) * 32 + lane], lane, my, staged, (uint32_t)g * kChunkRows);
      else
        stage_rows_rm(m[g], lane, my, staged, (uint32_t)g * kChunkRows);
      staged += cg;
    }
    __syncwarp();
    flush_rows<CODED>(p, bbase, gbase, staged, my, lane, out_ids);
    __syncwarp();
  }
}


// ---- fully selected chunks: whole-chunk copies beside the push-down ---------------------------
// Dense selections and clustered layouts select whole 1024-row chunks; pushdown_sel leaves those
// (p.dense_split) to this kernel: ids are a run, gathered projections are copies (8 loads in
// flight per lane; 16-byte loads and stores when the output position is 16-byte aligned, else
// element-wise); kept slots and constants as in copy_kept. Its own
// kernel, so that the 32-register push-down kernel does not carry the copy's registers.
template <class T>
__device__ __forceinline__ void copy_chunk(const void* src_v, void* dst_v, uint64_t cbase,
                                           uint64_t gbase, int lane) {
  T* __restrict__ dst = static_cast<T*>(dst_v) + gbase;
  if ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0) {
    // output position 16-byte aligned (every full chunk of a run of them): 16-byte stores too
    constexpr int N16 = kChunkRows * sizeof(T) / 16;
    const uint4* src = reinterpret_cast<const uint4*>(static_cast<const T*>(src_v) + cbase);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll 1
    for (int h = 0; h < (N16 + 255) / 256; ++h) {
      uint4 v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int k = h * 256 + i * 32 + lane;
        if (k < N16) v[i] = ld_stream_v4(src + k);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int k = h * 256 + i * 32 + lane;
        if (k < N16) d4[k] = v[i];
      }
    }
  } else {
    // unaligned output: element-wise, both sides coalesced (16-byte loads with 4-byte-strided
    // stores touched every store sector PER times: 2.5x the written sectors in ncu)
    const T* __restrict__ src = static_cast<const T*>(src_v) + cbase;
#pragma unroll 1
    for (int h = 0; h < kChunkRows; h += 256) {
      T v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = __ldcs(src + h + i * 32 + lane);
#pragma unroll
      for (int i = 0; i < 8; ++i) dst[h + i * 32 + lane] = v[i];
    }
  }
}

template <class P>
__global__ void __launch_bounds__(kThreads) dense_chunks_kernel(const __grid_constant__ P p,
                                                                uint64_t n, SelectionBufs sb,
                                                                uint32_t* __restrict__ out_ids,
                                                                const uint64_t* __restrict__ gate_count) {
  if (*gate_count == kXchgFailed || (p.gate && *gate_count > p.gate_max)) return;  // as pushdown_sel
  const uint64_t nhb = ((n + kChunkRows - 1) / kChunkRows + kHbChunks - 1) / kHbChunks;
  if (sb.hb_prefix[nhb + 1] == 0u) return;   // the count saw no fully selected chunk
  const uint32_t* sbs = kept_sb(sb);
  const uint64_t goff = p.global_out ? gate_count[kOffsetSlot - kGateSlot] : 0ull;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t nchunks = (n + kChunkRows - 1) / kChunkRows;
  const uint64_t nblocks = (nchunks + kBlockChunks - 1) / kBlockChunks;
  const uint64_t gw = (uint64_t)blockIdx.x * kWarpsPerCta + warp;
  const uint64_t nw = (uint64_t)gridDim.x * kWarpsPerCta;
  for (uint64_t blk = gw; blk < nblocks; blk += nw) {
    const uint64_t c0 = blk * kBlockChunks;
    const uint32_t cntv = (lane < kBlockChunks && c0 + lane < nchunks) ? sb.chunk_cnt[c0 + lane] : 0u;
    if (!__ballot_sync(0xFFFFFFFFu, cntv == (uint32_t)kChunkRows && lane < kBlockChunks)) continue;
    uint64_t gbase = goff + kept_base(sb, sbs, c0, lane);
#pragma unroll 1
    for (int g = 0; g < kBlockChunks; ++g) {
      const uint32_t cg = __shfl_sync(0xFFFFFFFFu, cntv, g);
      if (cg == (uint32_t)kChunkRows && gbase + kChunkRows <= p.capacity) {
        const uint64_t c = c0 + g, cbase = c * kChunkRows;
        const uint32_t idbase = (uint32_t)(p.row_offset + cbase);
#pragma unroll 8
        for (uint32_t q = lane; q < (uint32_t)kChunkRows; q += 32) out_ids[gbase + q] = idbase + q;
        if (p.n_direct) copy_kept(p, sb, c, gbase, kChunkRows, lane);   // kept slots / constants
#pragma unroll 1
        for (uint32_t j = 0; j < p.n_proj; ++j) {
          if (p.proj_cap_off[j] == kCodedProj) {
            // the value from each row's code bit (the keeping count's row-major word: bit b of
            // word L = row 32L + b), as flush_rows does for staged rows; the column is not read
            const uint64_t pts = (uint64_t)(uintptr_t)p.proj_src[j];
            const uint32_t wl = sb.which[c * 32 + lane];
            if (p.proj_wclass[j] == W1) {
              uint8_t* __restrict__ dst = static_cast<uint8_t*>(p.proj_dst[j]) + gbase;
#pragma unroll 8
              for (int i = 0; i < 32; ++i) {
                const uint32_t w = __shfl_sync(0xFFFFFFFFu, wl, i);
                dst[32 * i + lane] = (uint8_t)(pts >> (((w >> lane) & 1u) ? 8 : 0));
              }
            } else {
              uint32_t* __restrict__ dst = static_cast<uint32_t*>(p.proj_dst[j]) + gbase;
#pragma unroll 8
              for (int i = 0; i < 32; ++i) {
                const uint32_t w = __shfl_sync(0xFFFFFFFFu, wl, i);
                dst[32 * i + lane] = (uint32_t)(pts >> (((w >> lane) & 1u) ? 32 : 0));
              }
            }
            continue;
          }
          if (p.proj_cap_off[j] != kNoCapture) continue;
          switch (p.proj_wclass[j]) {
            case W1: copy_chunk<uint8_t>(p.proj_src[j], p.proj_dst[j], cbase, gbase, lane); break;
            case W2: copy_chunk<uint16_t>(p.proj_src[j], p.proj_dst[j], cbase, gbase, lane); break;
            case W4: copy_chunk<uint32_t>(p.proj_src[j], p.proj_dst[j], cbase, gbase, lane); break;
            default: copy_chunk<uint64_t>(p.proj_src[j], p.proj_dst[j], cbase, gbase, lane); break;
          }
        }
      }
      gbase += cg;
    }
  }
}

// ---- batch of programs over one scan -------------------------------------
// Every column of the batch is loaded once per chunk; each distinct leaf on it is evaluated once
// into the warp's leaf-mask table (shared memory, one u32 per lane per leaf); each program's
// postfix then runs over leaf masks and DOP_EMIT(k) adds the warp's popcount to program k's
// counter. One instance of the interval loop per TAIL variant (toolchain note above).
template <bool TAIL>
__device__ __forceinline__ void batch_column(const BatchProgram& p, const BatchColumn& C,
                                             uint64_t base, int lane, uint32_t nvalid,
                                             uint32_t* lm /* [leaf][32] */) {
  if (C.wclass == W8) {
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      uint64_t v[16];
      load_w8_half<TAIL>(C.data, base, lane, h, nvalid, v, nullptr);
#pragma unroll 1
      for (uint32_t l = C.leaf_begin; l < (uint32_t)C.leaf_begin + C.leaf_count; ++l) {
        uint32_t mh = 0;
#pragma unroll 1
        for (int t = 0; t < p.leaf_iv_count[l]; ++t) {
          const uint64_t lo = p.lo[p.leaf_iv_begin[l] + t], sp = p.span[p.leaf_iv_begin[l] + t];
#pragma unroll
          for (int i = 0; i < 16; ++i) mh |= (v[i] - lo <= sp) ? (1u << i) : 0u;
        }
        if (h == 0) lm[l * 32 + lane] = mh;
        else lm[l * 32 + lane] |= mh << 16;
      }
    }
    return;
  }
  uint32_t v[32];
  if (C.wclass == W1 && C.swar) {
    // every leaf on this 1-byte column is 1..4 points: test four rows per 32-bit word (SWAR, the
    // count fast path's s1_nibble; bit 4k+e = byte e of word k, the layout of load_w1)
    uint32_t x[8];
    load_w1_words<TAIL>(C.data, base, lane, nvalid, x);
#pragma unroll 1
    for (uint32_t l = C.leaf_begin; l < (uint32_t)C.leaf_begin + C.leaf_count; ++l) {
      const int np = p.leaf_pts[l];
      uint32_t pts[4];
#pragma unroll
      for (int t = 0; t < 4; ++t)
        pts[t] = t < np ? (uint32_t)p.lo[p.leaf_iv_begin[l] + t] * 0x01010101u : 0u;
      uint32_t m = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) m |= s1_nibble(x[k], pts, np) << (4 * k);
      lm[l * 32 + lane] = m;
    }
    return;
  }
  if (C.wclass == W1) {
    load_w1<TAIL>(C.data, base, lane, nvalid, v, nullptr);
  } else if (C.wclass == W4) {
    load_w4<TAIL>(C.data, base, lane, nvalid, v, nullptr);
    if (C.fkey) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = fkey(v[i]);
    }
  } else {
    load_w2<TAIL>(C.data, base, lane, nvalid, v, nullptr);
  }
#pragma unroll 1
  for (uint32_t l = C.leaf_begin; l < (uint32_t)C.leaf_begin + C.leaf_count; ++l) {
    uint32_t m = 0;
    const int niv = p.leaf_iv_count[l];
    if (niv == 1 && p.span[p.leaf_iv_begin[l]] == 0) {   // one point: an equality per row
      const uint32_t a = (uint32_t)p.lo[p.leaf_iv_begin[l]];
#pragma unroll
      for (int i = 0; i < 32; ++i) m |= (v[i] == a) ? (1u << i) : 0u;
    } else {
#pragma unroll 1
      for (int t = 0; t < niv; ++t) {
        const uint32_t lo = (uint32_t)p.lo[p.leaf_iv_begin[l] + t];
        const uint32_t sp = (uint32_t)p.span[p.leaf_iv_begin[l] + t];
#pragma unroll
        for (int i = 0; i < 32; ++i) m |= (v[i] - lo <= sp) ? (1u << i) : 0u;
      }
    }
    lm[l * 32 + lane] = m;
  }
}

template <bool TAIL>
__device__ __forceinline__ void batch_chunk(const BatchProgram& p, uint64_t base, int lane,
                                            uint32_t nvalid, uint32_t* lm, uint32_t* cnt /* [k] */,
                                            uint32_t (&acc)[8]) {
#if SEL_BATCH_PREFETCH
  // the chunk's other columns are loaded only after the first one is evaluated: start their DRAM
  // reads now (TMA bulk prefetch into L2), so that their loads later hit L2
  if (!TAIL && lane == 0) {
#pragma unroll 1
    for (uint32_t c = 1; c < p.n_cols; ++c) {
      const uint32_t w = 1u << p.col[c].wclass;
      prefetch_l2(static_cast<const char*>(p.col[c].data) + base * w, kChunkRows * w);
    }
  }
#endif
#pragma unroll 1
  for (uint32_t c = 0; c < p.n_cols; ++c) batch_column<TAIL>(p, p.col[c], base, lane, nvalid, lm);
  __syncwarp();
  const uint32_t valid = TAIL ? valid_mask(lane, nvalid) : 0xFFFFFFFFu;
  if (p.all_conj && p.n_progs <= 8) {   // and up to 8 programs: per-lane counts in registers
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (k < (int)p.n_progs && ((p.prog_live >> k) & 1u)) {
        uint32_t m = valid, bits = p.conj_set[k];
        while (bits) {
          const int l = __ffs(bits) - 1;
          bits &= bits - 1;
          m &= lm[l * 32 + lane];
        }
        acc[k] += (uint32_t)__popc(m);
      }
    }
    __syncwarp();
    return;
  }
  if (p.all_conj) {   // conjunctions: AND each program's leaf masks, no postfix stack
#pragma unroll 1
    for (uint32_t k = 0; k < p.n_progs; ++k) {
      if (!((p.prog_live >> k) & 1u)) continue;
      uint32_t m = valid, bits = p.conj_set[k];
      while (bits) {
        const int l = __ffs(bits) - 1;
        bits &= bits - 1;
        m &= lm[l * 32 + lane];
      }
      const uint32_t c = __reduce_add_sync(0xFFFFFFFFu, (uint32_t)__popc(m));
      if (lane == 0) cnt[k] += c;
    }
    __syncwarp();
    return;
  }
  uint32_t st[kMaxDeviceStack];
  int sp = 0;
#pragma unroll 1
  for (uint32_t i = 0; i < p.n_ops; ++i) {
    const uint8_t op = p.op[i];
    if (op == DOP_LEAF) {
      st[sp++] = lm[p.arg[i] * 32 + lane];
    } else if (op == DOP_EMIT) {
      const uint32_t m = sp > 0 ? st[--sp] : 0xFFFFFFFFu;    // an empty program is TRUE
      const uint32_t c = __reduce_add_sync(0xFFFFFFFFu, (uint32_t)__popc(m & valid));
      if (lane == 0) cnt[p.arg[i]] += c;
      sp = 0;
    } else {
      --sp;
      st[sp - 1] = op == DOP_AND ? (st[sp - 1] & st[sp]) : (st[sp - 1] | st[sp]);
    }
  }
  __syncwarp();
}

__global__ void __launch_bounds__(kThreads, SEL_BATCH_MINB) count_batch_kernel(const __grid_constant__ BatchProgram p,
                                                               uint64_t n, uint64_t* __restrict__ out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ uint32_t s_lm[kWarpsPerCta][kBatchMaxLeaves * 32];
  __shared__ uint32_t s_cnt[kWarpsPerCta][kBatchMaxProgs];
  for (int k = lane; k < kBatchMaxProgs; k += 32) s_cnt[warp][k] = 0;
  __syncwarp();
  const uint64_t nfull = n / kChunkRows;
  const uint32_t rem = (uint32_t)(n % kChunkRows);
  const uint64_t gw = (uint64_t)blockIdx.x * kWarpsPerCta + warp;
  const uint64_t nw = (uint64_t)gridDim.x * kWarpsPerCta;
  uint32_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (uint64_t c = gw; c < nfull; c += nw)
    batch_chunk<false>(p, c * kChunkRows, lane, kChunkRows, s_lm[warp], s_cnt[warp], acc);
  if (rem != 0 && gw == nfull % nw)
    batch_chunk<true>(p, nfull * kChunkRows, lane, rem, s_lm[warp], s_cnt[warp], acc);
#pragma unroll
  for (int k = 0; k < 8; ++k) {   // register counts of the <= 8-program conjunctive path
    const uint32_t c = __reduce_add_sync(0xFFFFFFFFu, acc[k]);
    if (lane == 0 && c) s_cnt[warp][k] += c;
  }
  __syncthreads();
  for (uint32_t k = threadIdx.x; k < p.n_progs; k += kThreads) {
    uint64_t s = 0;
#pragma unroll
    for (int w = 0; w < kWarpsPerCta; ++w) s += s_cnt[w][k];
    if (s) atomicAdd(reinterpret_cast<unsigned long long*>(out + k), (unsigned long long)s);
  }
}

// Memoised per (kernel, threads, shared memory, device): the grid of every probe is sized from it,
// and the runtime query costs microseconds of host time per launch.
template <class Kern>
int occupancy_of(Kern k, size_t dyn_smem, int threads = kThreads) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, size_t, int, int>, int> memo;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(reinterpret_cast<const void*>(k), dyn_smem, threads, dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    const auto it = memo.find(key);
    if (it != memo.end()) return it->second;
  }
  int blocks = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k, threads, dyn_smem) != cudaSuccess) return 1;
  blocks = blocks > 0 ? blocks : 1;
  std::lock_guard<std::mutex> lk(mu);
  memo[key] = blocks;
  return blocks;
}

}  // namespace

template <int FASTN>
void launch_count_fast(const DevProgramSmall& p, uint64_t n, int grid, const Scratch& s,
                       const SelectionBufs* keep, cudaStream_t stream, const ExecFinish& fin) {
  if (keep)
    count_kernel<DevProgramSmall, true, kWarpsPerCta, FASTN><<<grid, kThreads, (size_t)keep->warp_smem * kWarpsPerCta, stream>>>(p, n, s.partials, s.done, s.result, *keep, s.xg, fin);
  else
    count_kernel<DevProgramSmall, false, kWarpsPerCta, FASTN><<<grid, kThreads, 0, stream>>>(p, n, s.partials, s.done, s.result, SelectionBufs{}, s.xg, fin);
}

template <class P>
int launch_count_t(const P& p, uint64_t n, int grid, const Scratch& s, const SelectionBufs* keep,
                   int nw, void* st, const ExecFinish* finp) {
  cudaStream_t stream = (cudaStream_t)st;
  const ExecFinish fin = finp ? *finp : ExecFinish{};
  if constexpr (std::is_same<P, DevProgramSmall>::value) {
    if (p.fast_n > 0 && nw == kWarpsPerCta && !p.bm_smem) {
      switch (p.fast_n) {
        case 1: launch_count_fast<1>(p, n, grid, s, keep, stream, fin); break;
        case 2: launch_count_fast<2>(p, n, grid, s, keep, stream, fin); break;
        case 3: launch_count_fast<3>(p, n, grid, s, keep, stream, fin); break;
        default: launch_count_fast<4>(p, n, grid, s, keep, stream, fin); break;
      }
      return (int)cudaGetLastError();
    }
  }
  if (nw == 32) {
    if (keep)
      count_kernel<P, true, 32><<<grid, 32 * 32, (size_t)keep->warp_smem * 32 + p.bm_smem, stream>>>(p, n, s.partials, s.done, s.result, *keep, s.xg, fin);
    else
      count_kernel<P, false, 32><<<grid, 32 * 32, p.bm_smem, stream>>>(p, n, s.partials, s.done, s.result, SelectionBufs{}, s.xg, fin);
  } else {
    if (keep)
      count_kernel<P, true, kWarpsPerCta><<<grid, kThreads, (size_t)keep->warp_smem * kWarpsPerCta + p.bm_smem, stream>>>(p, n, s.partials, s.done, s.result, *keep, s.xg, fin);
    else
      count_kernel<P, false, kWarpsPerCta><<<grid, kThreads, p.bm_smem, stream>>>(p, n, s.partials, s.done, s.result, SelectionBufs{}, s.xg, fin);
  }
  return (int)cudaGetLastError();
}
int launch_count_small(const DevProgramSmall& p, uint64_t n, int grid, const Scratch& s,
                       const SelectionBufs* keep, void* st, int nw, const ExecFinish* fin) {
  return launch_count_t(p, n, grid, s, keep, nw, st, fin);
}
int launch_count_large(const DevProgramLarge& p, uint64_t n, int grid, const Scratch& s,
                       const SelectionBufs* keep, void* st, int nw, const ExecFinish* fin) {
  return launch_count_t(p, n, grid, s, keep, nw, st, fin);
}
template <class P>
int launch_pushdown_sel_t(const P& p, uint64_t n, uint32_t* out_ids, int grid, const Scratch& s,
                          const SelectionBufs& sb, void* st, int gate_ranks, const PeerXchg* xg,
                          int rank, bool finished, uint64_t* host, int block_chunks) {
  cudaStream_t stream = (cudaStream_t)st;
  if (!finished) {
    const uint64_t nchunks = (n + kChunkRows - 1) / kChunkRows;
    const uint32_t nhb = (uint32_t)((nchunks + kHbChunks - 1) / kHbChunks);
    selection_result_kernel<<<1, 256, 0, stream>>>(sb.hb_prefix, nhb,
                                                   ExecFinish{s.result, host, gate_ranks, rank},
                                                   xg ? *xg : PeerXchg{});
  }
  if (block_chunks == 1) {
    if (p.coded)
      pushdown_sel_kernel<P, true, 1><<<grid, kThreads, 0, stream>>>(p, n, sb, out_ids, s.result + kGateSlot);
    else
      pushdown_sel_kernel<P, false, 1><<<grid, kThreads, 0, stream>>>(p, n, sb, out_ids, s.result + kGateSlot);
  } else if (block_chunks == 2) {
    if (p.coded)
      pushdown_sel_kernel<P, true, 2><<<grid, kThreads, 0, stream>>>(p, n, sb, out_ids, s.result + kGateSlot);
    else
      pushdown_sel_kernel<P, false, 2><<<grid, kThreads, 0, stream>>>(p, n, sb, out_ids, s.result + kGateSlot);
  } else {
    if (p.coded)
      pushdown_sel_kernel<P, true, 4><<<grid, kThreads, 0, stream>>>(p, n, sb, out_ids, s.result + kGateSlot);
    else
      pushdown_sel_kernel<P, false, 4><<<grid, kThreads, 0, stream>>>(p, n, sb, out_ids, s.result + kGateSlot);
  }
  if (p.dense_split)
    dense_chunks_kernel<P><<<grid, kThreads, 0, stream>>>(p, n, sb, out_ids, s.result + kGateSlot);
  return (int)cudaGetLastError();
}
int launch_pushdown_sel_small(const DevProgramSmall& p, uint64_t n, uint32_t* out_ids, int grid,
                              const Scratch& s, const SelectionBufs& sb, void* st, int gate_ranks,
                              const PeerXchg* xg, int rank, bool finished, uint64_t* host,
                              int block_chunks) {
  return launch_pushdown_sel_t(p, n, out_ids, grid, s, sb, st, gate_ranks, xg, rank, finished, host,
                               block_chunks);
}
int launch_pushdown_sel_large(const DevProgramLarge& p, uint64_t n, uint32_t* out_ids, int grid,
                              const Scratch& s, const SelectionBufs& sb, void* st, int gate_ranks,
                              const PeerXchg* xg, int rank, bool finished, uint64_t* host,
                              int block_chunks) {
  return launch_pushdown_sel_t(p, n, out_ids, grid, s, sb, st, gate_ranks, xg, rank, finished, host,
                               block_chunks);
}
int launch_pushdown_small(const DevProgramSmall& p, uint64_t n, uint32_t* out_ids, int grid,
                          const Scratch& s, uint64_t ticket_base, uint32_t epoch, void* st) {
  pushdown_kernel<DevProgramSmall><<<grid, kThreads, (size_t)p.warp_smem * kWarpsPerCta, (cudaStream_t)st>>>(
      p, n, out_ids, s.ticket, ticket_base, s.status, epoch, s.result);
  return (int)cudaGetLastError();
}
int launch_pushdown_large(const DevProgramLarge& p, uint64_t n, uint32_t* out_ids, int grid,
                          const Scratch& s, uint64_t ticket_base, uint32_t epoch, void* st) {
  pushdown_kernel<DevProgramLarge><<<grid, kThreads, (size_t)p.warp_smem * kWarpsPerCta, (cudaStream_t)st>>>(
      p, n, out_ids, s.ticket, ticket_base, s.status, epoch, s.result);
  return (int)cudaGetLastError();
}
int prepare_kernels() {
  const int bytes = (int)kMaxPushdownSmem;
  cudaError_t e = cudaFuncSetAttribute(pushdown_kernel<DevProgramSmall>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(pushdown_kernel<DevProgramLarge>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  const int cbytes = (int)kMaxCountSmem;  // warp areas + staged key sets
  const void* counts[] = {(const void*)count_kernel<DevProgramSmall, true, kWarpsPerCta>,
                          (const void*)count_kernel<DevProgramLarge, true, kWarpsPerCta>,
                          (const void*)count_kernel<DevProgramSmall, false, kWarpsPerCta>,
                          (const void*)count_kernel<DevProgramLarge, false, kWarpsPerCta>,
                          (const void*)count_kernel<DevProgramSmall, true, 32>,
                          (const void*)count_kernel<DevProgramLarge, true, 32>,
                          (const void*)count_kernel<DevProgramSmall, false, 32>,
                          (const void*)count_kernel<DevProgramLarge, false, 32>};
  for (const void* f : counts)
    if (e == cudaSuccess) e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, cbytes);
  const void* fasts[] = {(const void*)count_kernel<DevProgramSmall, true, kWarpsPerCta, 1>,
                         (const void*)count_kernel<DevProgramSmall, true, kWarpsPerCta, 2>,
                         (const void*)count_kernel<DevProgramSmall, true, kWarpsPerCta, 3>,
                         (const void*)count_kernel<DevProgramSmall, true, kWarpsPerCta, 4>};
  for (const void* f : fasts)
    if (e == cudaSuccess) e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, cbytes);
  return (int)e;
}
int occupancy_count_fast(int fast_n, bool keep, size_t dyn) {
  switch (fast_n * 2 + (keep ? 1 : 0)) {
    case 2: return occupancy_of(count_kernel<DevProgramSmall, false, kWarpsPerCta, 1>, dyn);
    case 3: return occupancy_of(count_kernel<DevProgramSmall, true, kWarpsPerCta, 1>, dyn);
    case 4: return occupancy_of(count_kernel<DevProgramSmall, false, kWarpsPerCta, 2>, dyn);
    case 5: return occupancy_of(count_kernel<DevProgramSmall, true, kWarpsPerCta, 2>, dyn);
    case 6: return occupancy_of(count_kernel<DevProgramSmall, false, kWarpsPerCta, 3>, dyn);
    case 7: return occupancy_of(count_kernel<DevProgramSmall, true, kWarpsPerCta, 3>, dyn);
    case 8: return occupancy_of(count_kernel<DevProgramSmall, false, kWarpsPerCta, 4>, dyn);
    default: return occupancy_of(count_kernel<DevProgramSmall, true, kWarpsPerCta, 4>, dyn);
  }
}
// ---- equi-depth histogram over a block sample -----------
// Keys of the sampled chunks (c = phase + s * stride) of a 1/2/4-byte integer column, in the
// unsigned order of the values (INT32/DATE32: bits ^ 2^31), packed: sampled chunk s at s * 1024
// (only the last sampled chunk can be partial). One warp per chunk, grid-stride.
__global__ void __launch_bounds__(kThreads) sample_keys_kernel(const void* col, int wclass,
                                                               uint32_t flip, uint64_t n,
                                                               uint64_t stride, uint64_t phase,
                                                               uint64_t nsamp, uint32_t* keys) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (uint64_t)blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5);
  const uint64_t nw = (uint64_t)gridDim.x * kWarpsPerCta;
  for (uint64_t s = gw; s < nsamp; s += nw) {
    const uint64_t base = (phase + s * stride) * kChunkRows;
    const uint32_t rows = (uint32_t)min((uint64_t)kChunkRows, n - base);
    for (uint32_t i = lane; i < rows; i += 32) {
      uint32_t v;
      if (wclass == W4) v = __ldg(static_cast<const uint32_t*>(col) + base + i);
      else if (wclass == W2) v = __ldg(static_cast<const uint16_t*>(col) + base + i);
      else v = __ldg(static_cast<const uint8_t*>(col) + base + i);
      keys[s * kChunkRows + i] = v ^ flip;
    }
  }
}

// Bucket b of B over the m sorted keys: positions [floor(b m / B), floor((b+1) m / B)); its
// lowest and highest key, row count and number of distinct keys. One warp per bucket.
__global__ void __launch_bounds__(kThreads) bucket_stats_kernel(const uint32_t* __restrict__ s,
                                                                uint64_t m, uint32_t nb,
                                                                uint32_t* lo, uint32_t* hi,
                                                                uint64_t* rows, uint64_t* distinct) {
  const int lane = threadIdx.x & 31;
  const uint64_t b = (uint64_t)blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5);
  if (b >= nb) return;
  const uint64_t start = b * m / nb, end = (b + 1) * m / nb;
  uint64_t changes = 0;
  for (uint64_t i = start + 1 + lane; i < end; i += 32) changes += s[i] != s[i - 1] ? 1u : 0u;
  for (int o = 16; o > 0; o >>= 1) changes += __shfl_xor_sync(0xFFFFFFFFu, changes, o);
  if (lane == 0) {
    rows[b] = end - start;
    distinct[b] = end > start ? changes + 1 : 0;
    lo[b] = end > start ? s[start] : 0u;
    hi[b] = end > start ? s[end - 1] : 0u;
  }
}

__global__ void set_u64_kernel(uint64_t* p, uint64_t v) { *p = v; }
int launch_histogram(const void* col, int wclass, uint32_t flip, uint64_t n, uint64_t stride,
                     uint64_t phase, uint64_t nsamp, uint64_t m, uint32_t nb, uint32_t* keys,
                     uint32_t* sorted, void* temp, size_t temp_bytes, uint32_t* lo, uint32_t* hi,
                     uint64_t* rows, uint64_t* distinct, void* st) {
  cudaStream_t stream = (cudaStream_t)st;
  const uint64_t units = (nsamp + kWarpsPerCta - 1) / kWarpsPerCta;
  const uint64_t grid = units < 1 ? 1 : (units > 148ull * 16 ? 148ull * 16 : units);
  sample_keys_kernel<<<(unsigned)grid, kThreads, 0, stream>>>(col, wclass, flip, n, stride, phase,
                                                              nsamp, keys);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && m > 0)
    e = cub::DeviceRadixSort::SortKeys(temp, temp_bytes, keys, sorted, (int)m, 0, 32, stream);
  if (e == cudaSuccess)
    bucket_stats_kernel<<<(nb + kWarpsPerCta - 1) / kWarpsPerCta, kThreads, 0, stream>>>(
        m > 0 ? sorted : keys, m, nb, lo, hi, rows, distinct);
  return e != cudaSuccess ? (int)e : (int)cudaGetLastError();
}
size_t histogram_temp_bytes(uint64_t m) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                 (int)m, 0, 32);
  return bytes;
}
int launch_set_u64(uint64_t* p, uint64_t v, void* st) {
  set_u64_kernel<<<1, 1, 0, (cudaStream_t)st>>>(p, v);
  return (int)cudaGetLastError();
}
int launch_peer_exchange(const PeerXchg& x, const uint64_t* src, int k, uint64_t* out,
                         uint64_t* sums, void* st) {
  peer_exchange_kernel<<<1, 256, 0, (cudaStream_t)st>>>(x, src, k, out, sums);
  return (int)cudaGetLastError();
}
int launch_count_batch(const BatchProgram& p, uint64_t n, int grid, uint64_t* out, void* st) {
  count_batch_kernel<<<grid, kThreads, 0, (cudaStream_t)st>>>(p, n, out);
  return (int)cudaGetLastError();
}
int occupancy_count_batch() { return occupancy_of(count_batch_kernel, 0); }
int occupancy_count_small() { return occupancy_of(count_kernel<DevProgramSmall, false, kWarpsPerCta>, 0); }
int occupancy_count_keep_small(size_t dyn) { return occupancy_of(count_kernel<DevProgramSmall, true, kWarpsPerCta>, dyn); }
int occupancy_count_keep_large(size_t dyn) { return occupancy_of(count_kernel<DevProgramLarge, true, kWarpsPerCta>, dyn); }
int occupancy_count_large() { return occupancy_of(count_kernel<DevProgramLarge, false, kWarpsPerCta>, 0); }
int occupancy_count_dyn_small(size_t dyn) { return occupancy_of(count_kernel<DevProgramSmall, false, kWarpsPerCta>, dyn); }
int occupancy_count_dyn_large(size_t dyn) { return occupancy_of(count_kernel<DevProgramLarge, false, kWarpsPerCta>, dyn); }
int occupancy_pushdown_sel_small() { return occupancy_of(pushdown_sel_kernel<DevProgramSmall, false, kSelBlockChunks>, 0); }
int occupancy_pushdown_sel_large() { return occupancy_of(pushdown_sel_kernel<DevProgramLarge, false, kSelBlockChunks>, 0); }
int occupancy_pushdown_small(size_t dyn_smem) { return occupancy_of(pushdown_kernel<DevProgramSmall>, dyn_smem); }
int occupancy_pushdown_large(size_t dyn_smem) { return occupancy_of(pushdown_kernel<DevProgramLarge>, dyn_smem); }

}  // namespace sel
