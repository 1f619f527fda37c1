// jz_sort.cu -- A1 ingest/validate/frame, A2 Morton encode, A3 LSD radix sort + gather
// (PAPER.md L67-114 z-order sort, here with integer keys as BASELINE.json asks).
//
// Keys: 21 bits per axis, bit b of axis d at key bit 3b + (2 - d): x most significant
// ("differences in earlier coordinates are more significant").
// Sort: one-sweep LSD radix sort, 8-bit digits. A single histogram kernel reads the
// positions once and produces all eight digit histograms; every pass then ranks a tile
// of 3072 keys per CTA with warp match_any, publishes per-digit tile counts with
// decoupled look-back (dynamic tile ids => forward progress), stages the tile in shared
// memory in digit order, and writes contiguous runs. Pass 0 computes keys from positions
// (no key/val read); the last pass gathers float4 {x, y, z, bits(gidx)} (no separate
// gather kernel). Passes whose digit is constant over all keys are skipped.
#include <cstdlib>
#include <cstring>
#include <vector>

#include "jz_common.cuh"
#include "jz_internal.h"

namespace jz {

constexpr int kSortThreads = 256;
constexpr int kSortIPT = 12;
constexpr int kSortTile = kSortThreads * kSortIPT;
constexpr int kRadix = 256;
constexpr int kPasses = 8;
constexpr unsigned long long kFlagAgg = 1ull << 62, kFlagPre = 2ull << 62, kValMask = (1ull << 62) - 1;

__device__ __forceinline__ uint64_t spread21(uint32_t v) {
  uint64_t x = v & 0x1fffffu;
  x = (x | x << 32) & 0x1f00000000ffffull;
  x = (x | x << 16) & 0x1f0000ff0000ffull;
  x = (x | x << 8) & 0x100f00f00f00f00full;
  x = (x | x << 4) & 0x10c30c30c30c30c3ull;
  x = (x | x << 2) & 0x1249249249249249ull;
  return x;
}

__device__ __forceinline__ uint32_t quant(float x, float o, float s) {
  float v = __fmul_rn(__fsub_rn(x, o), s);
  v = fminf(fmaxf(v, 0.f), 2097151.f);
  return (uint32_t)v;  // v >= 0: truncation == floor
}

__device__ __forceinline__ uint64_t morton(float x, float y, float z, const Frame &f) {
  return (spread21(quant(x, f.o[0], f.s[0])) << 2) | (spread21(quant(y, f.o[1], f.s[1])) << 1) |
         spread21(quant(z, f.o[2], f.s[2]));
}

// ---------------------------------------------------------------- A1: validate + bbox
struct FrameStats {
  unsigned int lo[3], hi[3];  // order-preserving uint encoding of floats
  int bad;                    // 1: non-finite, 2: periodic coordinate outside [0, L)
};

__device__ __forceinline__ unsigned int f2ord(float f) {
  unsigned int u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__global__ void k_frame(const float *__restrict__ pos, int64_t n, int stride, Dom D, FrameStats *st) {
  float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  int bad = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      float v = pos[i * stride + d];
      if (!isfinite(v)) bad |= 1;
      else if (D.periodic && !(v >= 0.f && v < D.L[d])) bad |= 2;
      lo[d] = fminf(lo[d], v);
      hi[d] = fmaxf(hi[d], v);
    }
  }
#pragma unroll
  for (int d = 0; d < 3; ++d) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo[d] = fminf(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
      hi[d] = fmaxf(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
    }
  }
  bad = __reduce_or_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      atomicMin(&st->lo[d], f2ord(lo[d]));
      atomicMax(&st->hi[d], f2ord(hi[d]));
    }
    if (bad) atomicOr(&st->bad, bad);
  }
}

// ---------------------------------------------------------------- A2: all digit histograms
__global__ void __launch_bounds__(256) k_sort_hist(const float *__restrict__ pos, int64_t n, int stride, Frame f,
                                                   unsigned int *__restrict__ hist /*[8][256]*/) {
  __shared__ unsigned int s_h[kPasses][kRadix];
  for (int i = threadIdx.x; i < kPasses * kRadix; i += blockDim.x) (&s_h[0][0])[i] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float *p = pos + i * stride;
    uint64_t key = morton(p[0], p[1], p[2], f);
#pragma unroll
    for (int ps = 0; ps < kPasses; ++ps) atomicAdd(&s_h[ps][(key >> (8 * ps)) & 255], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kPasses * kRadix; i += blockDim.x) {
    unsigned int v = (&s_h[0][0])[i];
    if (v) atomicAdd(&hist[i], v);
  }
}

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ---------------------------------------------------------------- A3: one-sweep pass
// FIRST: keys computed from positions, vals = input index.  LAST: gather float4 output.
template <bool FIRST, bool LAST>
__global__ void __launch_bounds__(kSortThreads, 3) k_onesweep(
    const float *__restrict__ pos, int stride, int gidx_mode, int64_t gidx_base, Frame f, float4 *__restrict__ pos4,
    const uint64_t *__restrict__ kin, const uint32_t *__restrict__ vin, uint64_t *__restrict__ kout,
    uint32_t *__restrict__ vout, float4 *__restrict__ pts_out, int64_t n, int shift,
    const unsigned int *__restrict__ digit_base, unsigned long long *status, int *tile_counter) {
  __shared__ unsigned int s_wcnt[kSortThreads / 32][kRadix];
  __shared__ uint64_t s_keys[kSortTile];
  __shared__ uint32_t s_vals[kSortTile];
  __shared__ unsigned int s_tstart[kRadix];
  __shared__ unsigned long long s_gbase[kRadix];
  __shared__ int s_tile;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (kSortThreads / 32) * kRadix; i += kSortThreads) (&s_wcnt[0][0])[i] = 0;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1);
  __syncthreads();
  const int tile = s_tile;
  const int64_t base = (int64_t)tile * kSortTile;

  uint64_t key[kSortIPT];
  uint32_t val[kSortIPT];
  uint32_t rank[kSortIPT];
#pragma unroll
  for (int i = 0; i < kSortIPT; ++i) {
    int64_t idx = base + (int64_t)warp * 32 * kSortIPT + i * 32 + lane;
    if (idx < n) {
      if (FIRST) {
        const float *p = pos + idx * stride;
        key[i] = morton(p[0], p[1], p[2], f);
        val[i] = (uint32_t)idx;
        // aligned float4 copy {x, y, z, bits(gidx)} for the final gather (one 16-byte load per point)
        if (pos4) pos4[idx] = make_float4(p[0], p[1], p[2], __int_as_float((int)(gidx_base + idx)));
      } else {
        key[i] = kin[idx];
        val[i] = vin[idx];
      }
    } else {
      key[i] = ~0ull;
      val[i] = 0;
    }
  }
  const unsigned lt_mask = (1u << lane) - 1u;
#pragma unroll
  for (int i = 0; i < kSortIPT; ++i) {
    int64_t idx = base + (int64_t)warp * 32 * kSortIPT + i * 32 + lane;
    unsigned d = idx < n ? (unsigned)((key[i] >> shift) & 255) : 256u;
    unsigned peers = __match_any_sync(0xffffffffu, d);
    unsigned before = d < 256 ? s_wcnt[warp][d] : 0u;
    rank[i] = before + __popc(peers & lt_mask);
    __syncwarp();
    if (d < 256 && lane == 31 - __clz(peers)) s_wcnt[warp][d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // per digit: warp offsets and tile total
  const int t = threadIdx.x;
  unsigned tot = 0;
#pragma unroll
  for (int w = 0; w < kSortThreads / 32; ++w) {
    unsigned c = s_wcnt[w][t];
    s_wcnt[w][t] = tot;
    tot += c;
  }
  unsigned long long *my_status = status + (size_t)tile * kRadix + t;
  st_relaxed(my_status, (tile == 0 ? kFlagPre : kFlagAgg) | (unsigned long long)tot);
  // exclusive scan of digit totals within the tile
  {
    unsigned v = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    __shared__ unsigned s_ws[kSortThreads / 32];
    if (lane == 31) s_ws[warp] = v;
    __syncthreads();
    unsigned wpre = 0;
#pragma unroll
    for (int w = 0; w < kSortThreads / 32; ++w) wpre += (w < warp) ? s_ws[w] : 0u;
    s_tstart[t] = wpre + v - tot;
  }
  // decoupled look-back over previous tiles for digit t
  unsigned long long excl = 0;
  if (tile > 0) {
    int j = tile - 1;
    while (true) {
      unsigned long long s = ld_relaxed(status + (size_t)j * kRadix + t);
      unsigned long long flag = s & ~kValMask;
      if (flag == 0) continue;
      excl += s & kValMask;
      if (flag == kFlagPre) break;
      --j;
    }
    st_relaxed(my_status, kFlagPre | (excl + tot));
  }
  s_gbase[t] = (unsigned long long)digit_base[t] + excl;
  __syncthreads();
  // stage tile in digit order
#pragma unroll
  for (int i = 0; i < kSortIPT; ++i) {
    int64_t idx = base + (int64_t)warp * 32 * kSortIPT + i * 32 + lane;
    if (idx < n) {
      unsigned d = (unsigned)((key[i] >> shift) & 255);
      unsigned lp = s_tstart[d] + s_wcnt[warp][d] + rank[i];
      s_keys[lp] = key[i];
      s_vals[lp] = val[i];
    }
  }
  __syncthreads();
  const int cnt = (int)min((int64_t)kSortTile, n - base);
  for (int j = threadIdx.x; j < cnt; j += kSortThreads) {
    uint64_t k = s_keys[j];
    uint32_t v = s_vals[j];
    unsigned d = (unsigned)((k >> shift) & 255);
    int64_t gp = (int64_t)s_gbase[d] + (j - (int)s_tstart[d]);
    kout[gp] = k;
    vout[gp] = v;
    if (LAST) {
      if (gidx_mode) {
        pts_out[gp] = reinterpret_cast<const float4 *>(pos)[v];  // input rows are float4 {x, y, z, gidx}
      } else if (pos4 && !FIRST) {
        pts_out[gp] = pos4[v];
      } else {
        const float *p = pos + (int64_t)v * stride;
        pts_out[gp] = make_float4(p[0], p[1], p[2], __int_as_float((int)(gidx_base + v)));
      }
    }
  }
}

// ---------------------------------------------------------------- A3 (default): 40-bit key sort, 8-byte items
// The LSD passes sort key bits 23..62 (the 40 most significant of the 63 key bits) with 8-byte
// (key part, index) items instead of 12-byte (key, index) pairs, five 8-bit passes instead of
// eight: pass 0 ranks bits 23..30, computed from the positions; passes 1-4 rank hi = key >> 31.
// The last pass gathers the positions, recomputes the full 63-bit keys and writes keys +
// float4 points + perm. Points whose bits 23..62 agree (cells of 2^-13.3 of the box side: rare
// even at halo centres) are then in input order; a fix-up orders each such run by (key, index),
// which makes the result the stable argsort of the full keys. Runs longer than
// kSegBlock (massive duplicates) fall back to the 8-pass sort of the full keys.
#ifndef JZ_S32_IPT
#define JZ_S32_IPT 16
#endif
#ifndef JZ_S32_MINB
#define JZ_S32_MINB 3
#endif
constexpr int kS32Threads = 256;
constexpr int kS32IPT = JZ_S32_IPT;
constexpr int kS32Tile = kS32Threads * kS32IPT;
constexpr int kS32Passes = 5;     // pass 0: key bits 23..30; passes 1-4: the bytes of hi = key >> 31
constexpr int kLoShift = 23;
constexpr int kSegThread = 32;    // runs up to this length: one thread, insertion sort in place
constexpr int kSegBlock = 2048;   // runs up to this length: one CTA, bitonic sort in shared memory

__device__ __forceinline__ uint32_t hi32(uint64_t k) { return (uint32_t)(k >> 31); }
__device__ __forceinline__ uint64_t runkey(uint64_t k) { return k >> kLoShift; }  // equal => fix-up run

__global__ void __launch_bounds__(256) k_hist32(const float *__restrict__ pos, int64_t n, int stride, Frame f,
                                                unsigned int *__restrict__ hist /*[4][256]*/) {
  __shared__ unsigned int s_h[kS32Passes][kRadix];
  for (int i = threadIdx.x; i < kS32Passes * kRadix; i += blockDim.x) (&s_h[0][0])[i] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float *p = pos + i * stride;
    const uint64_t k = morton(p[0], p[1], p[2], f);
    const uint32_t h = hi32(k);
    atomicAdd(&s_h[0][(k >> kLoShift) & 255], 1u);
#pragma unroll
    for (int ps = 1; ps < kS32Passes; ++ps) atomicAdd(&s_h[ps][(h >> (8 * (ps - 1))) & 255], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kS32Passes * kRadix; i += blockDim.x) {
    const unsigned v = (&s_h[0][0])[i];
    if (v) atomicAdd(&hist[i], v);
  }
}

__device__ __forceinline__ void cpa16(void *sdst, const void *gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gsrc) : "memory");
}

// input point v as float4 {x, y, z, bits(gidx)} (gidx_mode: input rows are float4 {x, y, z, gidx})
__device__ __forceinline__ float4 load_point(const float *__restrict__ pos, int stride, int gidx_mode, int64_t gidx_base,
                                             uint32_t v) {
  if (gidx_mode) return reinterpret_cast<const float4 *>(pos)[v];
  const float *p = pos + (int64_t)v * stride;
  return make_float4(p[0], p[1], p[2], __int_as_float((int)(gidx_base + v)));
}

// One-sweep pass over (hi, index) pairs. Non-first passes bring the tile into shared memory with
// 16-byte asynchronous copies (every load of the tile in flight at once), then rank as above.
template <bool FIRST, bool LAST>
__global__ void __launch_bounds__(kS32Threads, JZ_S32_MINB) k_onesweep32(
    const float *__restrict__ pos, int stride, int gidx_mode, int64_t gidx_base, Frame f,
    const uint32_t *__restrict__ kin, const uint32_t *__restrict__ vin, uint32_t *__restrict__ kout,
    uint32_t *__restrict__ vout, uint64_t *__restrict__ keys_out, float4 *__restrict__ pts_out, int64_t n, int shift,
    int lo, const unsigned int *__restrict__ digit_base, unsigned long long *status, int *tile_counter) {
  // FIRST && lo: the item key is (key >> 23) mod 2^32 (digit = bits 23..30, shift 0) and the hi
  // part written for the next pass is recomputed from the position; otherwise items carry hi
  __shared__ unsigned int s_wcnt[kS32Threads / 32][kRadix];
  __shared__ __align__(16) uint32_t s_keys[kS32Tile];
  __shared__ __align__(16) uint32_t s_vals[kS32Tile];
  __shared__ unsigned int s_tstart[kRadix];
  __shared__ unsigned long long s_gbase[kRadix];
  __shared__ unsigned s_ws[kS32Threads / 32];
  __shared__ int s_tile;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (kS32Threads / 32) * kRadix; i += kS32Threads) (&s_wcnt[0][0])[i] = 0;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1);
  __syncthreads();
  const int tile = s_tile;
  const int64_t base = (int64_t)tile * kS32Tile;
  const int cnt = (int)min((int64_t)kS32Tile, n - base);

  uint32_t key[kS32IPT], val[kS32IPT], rank[kS32IPT];
  if (!FIRST) {
    if (cnt == kS32Tile) {  // full tile: 16-byte copies of keys and values
#pragma unroll
      for (int c = threadIdx.x; c < kS32Tile / 4; c += kS32Threads) {
        cpa16(&s_keys[4 * c], kin + base + 4 * c);
        cpa16(&s_vals[4 * c], vin + base + 4 * c);
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
    } else {
      for (int j = threadIdx.x; j < cnt; j += kS32Threads) {
        s_keys[j] = kin[base + j];
        s_vals[j] = vin[base + j];
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < kS32IPT; ++i) {
    const int j = warp * 32 * kS32IPT + i * 32 + lane;  // warp-striped: stable ranking order
    if (j < cnt) {
      if (FIRST) {
        const float *p = pos + (base + j) * stride;
        const uint64_t k64 = morton(p[0], p[1], p[2], f);
        key[i] = lo ? (uint32_t)(k64 >> kLoShift) : hi32(k64);
        val[i] = (uint32_t)(base + j);
      } else {
        key[i] = s_keys[j];
        val[i] = s_vals[j];
      }
    } else {
      key[i] = 0xffffffffu;
      val[i] = 0;
    }
  }
  if (!FIRST) __syncthreads();  // s_keys / s_vals are reused for the digit-ordered tile below
  const unsigned lt_mask = (1u << lane) - 1u;
#pragma unroll
  for (int i = 0; i < kS32IPT; ++i) {
    const int j = warp * 32 * kS32IPT + i * 32 + lane;
    const unsigned d = j < cnt ? (key[i] >> shift) & 255u : 256u;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const unsigned before = d < 256 ? s_wcnt[warp][d] : 0u;
    rank[i] = before + __popc(peers & lt_mask);
    __syncwarp();
    if (d < 256 && lane == 31 - __clz(peers)) s_wcnt[warp][d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  const int t = threadIdx.x;
  unsigned tot = 0;
#pragma unroll
  for (int w = 0; w < kS32Threads / 32; ++w) {
    const unsigned c = s_wcnt[w][t];
    s_wcnt[w][t] = tot;
    tot += c;
  }
  unsigned long long *my_status = status + (size_t)tile * kRadix + t;
  st_relaxed(my_status, (tile == 0 ? kFlagPre : kFlagAgg) | (unsigned long long)tot);
  {
    unsigned v = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    if (lane == 31) s_ws[warp] = v;
    __syncthreads();
    unsigned wpre = 0;
#pragma unroll
    for (int w = 0; w < kS32Threads / 32; ++w) wpre += (w < warp) ? s_ws[w] : 0u;
    s_tstart[t] = wpre + v - tot;
  }
  unsigned long long excl = 0;
  if (tile > 0) {
    int jt = tile - 1;
    while (true) {
      const unsigned long long sv = ld_relaxed(status + (size_t)jt * kRadix + t);
      const unsigned long long flag = sv & ~kValMask;
      if (flag == 0) continue;
      excl += sv & kValMask;
      if (flag == kFlagPre) break;
      --jt;
    }
    st_relaxed(my_status, kFlagPre | (excl + tot));
  }
  s_gbase[t] = (unsigned long long)digit_base[t] + excl;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kS32IPT; ++i) {
    const int j = warp * 32 * kS32IPT + i * 32 + lane;
    if (j < cnt) {
      const unsigned d = (key[i] >> shift) & 255u;
      const unsigned lp = s_tstart[d] + s_wcnt[warp][d] + rank[i];
      s_keys[lp] = key[i];
      s_vals[lp] = val[i];
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < cnt; j += kS32Threads) {
    const uint32_t k = s_keys[j];
    const uint32_t v = s_vals[j];
    const unsigned d = (k >> shift) & 255u;
    const int64_t gp = (int64_t)s_gbase[d] + (j - (int)s_tstart[d]);
    if (LAST) {
      vout[gp] = v;  // perm
      const float4 p = load_point(pos, stride, gidx_mode, gidx_base, v);
      keys_out[gp] = morton(p.x, p.y, p.z, f);
      pts_out[gp] = p;
    } else {
      if (FIRST && lo) {  // the tile's points were just read: the position is in L1 / L2
        const float *p = pos + (int64_t)v * stride;
        kout[gp] = hi32(morton(p[0], p[1], p[2], f));
      } else {
        kout[gp] = k;
      }
      vout[gp] = v;
    }
  }
}

__device__ __forceinline__ bool key_less(uint64_t ka, uint32_t pa, uint64_t kb, uint32_t pb) {
  return ka < kb || (ka == kb && pa < pb);
}

// Fix-up of runs of equal hi parts (in input order after the passes): every run of length >= 2
// is sorted by (key, index). Runs up to kSegThread: the thread at the run start, insertion sort
// in place (key, perm and point move together); longer runs are queued for k_seg_block.
__global__ void k_seg_fix(uint64_t *__restrict__ keys, int32_t *__restrict__ perm, float4 *__restrict__ pts, int64_t n,
                          int64_t *__restrict__ big, int *__restrict__ nbig, int big_cap, int *__restrict__ fallback) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i + 1 < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t h = runkey(keys[i]);
    if (runkey(keys[i + 1]) != h) continue;
    if (i > 0 && runkey(keys[i - 1]) == h) continue;  // not the run start
    int64_t e = i + 2;
    while (e < n && e - i <= kSegThread && runkey(keys[e]) == h) ++e;
    const int64_t len = e - i;
    if (len > kSegThread) {
      const int b = atomicAdd(nbig, 1);
      if (b < big_cap) big[b] = i;
      else atomicOr(fallback, 1);
      continue;
    }
    for (int64_t a = i + 1; a < e; ++a) {  // insertion sort by (key, index)
      const uint64_t ka = keys[a];
      const int32_t pa = perm[a];
      const float4 qa = pts[a];
      int64_t b = a - 1;
      while (b >= i && key_less(ka, (uint32_t)pa, keys[b], (uint32_t)perm[b])) {
        keys[b + 1] = keys[b];
        perm[b + 1] = perm[b];
        pts[b + 1] = pts[b];
        --b;
      }
      keys[b + 1] = ka;
      perm[b + 1] = pa;
      pts[b + 1] = qa;
    }
  }
}

// one CTA per queued long run: bitonic sort of (key, index) pairs in shared memory, then the
// points are re-gathered from the input by the sorted indices
__global__ void __launch_bounds__(512) k_seg_block(uint64_t *__restrict__ keys, int32_t *__restrict__ perm,
                                                   float4 *__restrict__ pts, int64_t n, const int64_t *__restrict__ big,
                                                   const int *__restrict__ nbig, int big_cap, const float *__restrict__ pos,
                                                   int stride, int gidx_mode, int64_t gidx_base,
                                                   int *__restrict__ fallback) {
  __shared__ uint64_t s_k[kSegBlock];
  __shared__ uint32_t s_p[kSegBlock];
  __shared__ int s_len;
  const int nb = min(*nbig, big_cap);
  for (int b = blockIdx.x; b < nb; b += gridDim.x) {
    const int64_t i0 = big[b];
    if (threadIdx.x == 0) {
      const uint64_t h = runkey(keys[i0]);
      int64_t e = i0 + 1;
      while (e < n && e - i0 <= kSegBlock && runkey(keys[e]) == h) ++e;
      s_len = (int)(e - i0);
      if (e - i0 > kSegBlock) atomicOr(fallback, 1);
    }
    __syncthreads();
    const int len = s_len;
    if (len <= kSegBlock) {
      int P = 1;
      while (P < len) P <<= 1;
      for (int j = threadIdx.x; j < P; j += blockDim.x) {
        s_k[j] = j < len ? keys[i0 + j] : ~0ull;
        s_p[j] = j < len ? (uint32_t)perm[i0 + j] : 0xffffffffu;
      }
      __syncthreads();
      for (int size = 2; size <= P; size <<= 1) {
        for (int stride2 = size >> 1; stride2 > 0; stride2 >>= 1) {
          for (int j = threadIdx.x; j < P; j += blockDim.x) {
            const int o = j ^ stride2;
            if (o > j) {
              const bool asc = (j & size) == 0;
              const bool gt = key_less(s_k[o], s_p[o], s_k[j], s_p[j]);
              if (gt == asc) {
                const uint64_t tk = s_k[j];
                s_k[j] = s_k[o];
                s_k[o] = tk;
                const uint32_t tp = s_p[j];
                s_p[j] = s_p[o];
                s_p[o] = tp;
              }
            }
          }
          __syncthreads();
        }
      }
      for (int j = threadIdx.x; j < len; j += blockDim.x) {
        keys[i0 + j] = s_k[j];
        perm[i0 + j] = (int32_t)s_p[j];
        pts[i0 + j] = load_point(pos, stride, gidx_mode, gidx_base, s_p[j]);
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- host driver
void compute_frame(const float *pos, int64_t n, int stride, const Dom &D, const jz_knn_params_t &prm,
                   Frame *frame, cudaStream_t st) {
  FrameStats h;
  for (int d = 0; d < 3; ++d) {
    h.lo[d] = 0xffffffffu;
    h.hi[d] = 0u;
  }
  h.bad = 0;
  FrameStats *dst = nullptr;
  JZ_CUDA(cudaMallocAsync(&dst, sizeof(FrameStats), st));
  JZ_CUDA(cudaMemcpyAsync(dst, &h, sizeof(h), cudaMemcpyHostToDevice, st));
  k_frame<<<grid_for(n, 256, 148 * 8), 256, 0, st>>>(pos, n, stride, D, dst);
  JZ_LAUNCH_CHECK();
  JZ_CUDA(cudaMemcpyAsync(&h, dst, sizeof(h), cudaMemcpyDeviceToHost, st));
  JZ_CUDA(cudaFreeAsync(dst, st));
  JZ_CUDA(cudaStreamSynchronize(st));
  if (h.bad & 1) throw Error(3, "non-finite coordinate in input");
  if (h.bad & 2) throw Error(3, "periodic coordinate outside [0, L)");
  auto ord2f = [](unsigned u) {
    unsigned b = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
    float f;
    memcpy(&f, &b, 4);
    return f;
  };
  if (D.periodic) {
    for (int d = 0; d < 3; ++d) {
      frame->o[d] = 0.f;
      frame->s[d] = (float)(2097152.0 / (double)D.L[d]);
    }
  } else if (prm.flags & 1u /* JZ_FLAG_FRAME */) {
    for (int d = 0; d < 3; ++d) {
      frame->o[d] = prm.frame_origin[d];
      frame->s[d] = (float)(2097152.0 / (double)prm.frame_extent);
    }
  } else {
    float lo[3], hi[3], e = 0.f;
    for (int d = 0; d < 3; ++d) {
      lo[d] = ord2f(h.lo[d]);
      hi[d] = ord2f(h.hi[d]);
      float sp = hi[d] - lo[d];
      if (sp > e) e = sp;
    }
    if (!(e > 0.f)) e = 1.f;
    for (int d = 0; d < 3; ++d) {
      frame->o[d] = lo[d];
      frame->s[d] = (float)(2097152.0 / (double)e);
    }
  }
}

// validation + bounding box of this rank's points (multi-GPU frame: all-reduced by the caller);
// n = 0: lo = +inf, hi = -inf
void local_bbox(const float *pos, int64_t n, int stride, const Dom &D, float lo[3], float hi[3], cudaStream_t st) {
  for (int d = 0; d < 3; ++d) {
    lo[d] = INFINITY;
    hi[d] = -INFINITY;
  }
  if (n <= 0) return;
  FrameStats h;
  for (int d = 0; d < 3; ++d) {
    h.lo[d] = 0xffffffffu;
    h.hi[d] = 0u;
  }
  h.bad = 0;
  FrameStats *dst = nullptr;
  JZ_CUDA(cudaMallocAsync(&dst, sizeof(FrameStats), st));
  JZ_CUDA(cudaMemcpyAsync(dst, &h, sizeof(h), cudaMemcpyHostToDevice, st));
  k_frame<<<grid_for(n, 256, 148 * 8), 256, 0, st>>>(pos, n, stride, D, dst);
  JZ_LAUNCH_CHECK();
  JZ_CUDA(cudaMemcpyAsync(&h, dst, sizeof(h), cudaMemcpyDeviceToHost, st));
  JZ_CUDA(cudaFreeAsync(dst, st));
  JZ_CUDA(cudaStreamSynchronize(st));
  if (h.bad & 1) throw Error(3, "non-finite coordinate in input");
  if (h.bad & 2) throw Error(3, "periodic coordinate outside [0, L)");
  for (int d = 0; d < 3; ++d) {
    const unsigned a = (h.lo[d] & 0x80000000u) ? (h.lo[d] & 0x7fffffffu) : ~h.lo[d];
    const unsigned b = (h.hi[d] & 0x80000000u) ? (h.hi[d] & 0x7fffffffu) : ~h.hi[d];
    memcpy(&lo[d], &a, 4);
    memcpy(&hi[d], &b, 4);
  }
}

// 8-pass sort of the full 63-bit keys (fallback for runs of equal high keys > kSegBlock)
static void sort_points8(const float *pos, int64_t n, int stride, int gidx_mode, int64_t gidx_base, const Frame &frame,
                         uint64_t *keys_out, int32_t *perm_out, float4 *pts_out, cudaStream_t st) {
  unsigned int *dhist = nullptr;
  JZ_CUDA(cudaMallocAsync(&dhist, kPasses * kRadix * sizeof(unsigned), st));
  JZ_CUDA(cudaMemsetAsync(dhist, 0, kPasses * kRadix * sizeof(unsigned), st));
  k_sort_hist<<<grid_for(n, 256, 148 * 4), 256, 0, st>>>(pos, n, stride, frame, dhist);
  JZ_LAUNCH_CHECK();
  std::vector<unsigned> hist(kPasses * kRadix);
  JZ_CUDA(cudaMemcpyAsync(hist.data(), dhist, hist.size() * sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  JZ_CUDA(cudaStreamSynchronize(st));
  std::vector<unsigned> bases(kPasses * kRadix);
  std::vector<int> passes;
  for (int p = 0; p < kPasses; ++p) {
    unsigned acc = 0;
    bool trivial = false;
    for (int b = 0; b < kRadix; ++b) {
      bases[p * kRadix + b] = acc;
      if (hist[p * kRadix + b] == (unsigned)n) trivial = true;
      acc += hist[p * kRadix + b];
    }
    if (!trivial) passes.push_back(p);
  }
  if (passes.empty()) passes.push_back(0);
  JZ_CUDA(cudaMemcpyAsync(dhist, bases.data(), bases.size() * sizeof(unsigned), cudaMemcpyHostToDevice, st));

  const int64_t ntiles = ceil_div(n, kSortTile);
  unsigned long long *status = nullptr;
  int *counters = nullptr;
  uint64_t *kbuf[2] = {nullptr, nullptr};
  uint32_t *vbuf[2] = {nullptr, nullptr};
  JZ_CUDA(cudaMallocAsync(&status, (size_t)ntiles * kRadix * sizeof(unsigned long long), st));
  JZ_CUDA(cudaMallocAsync(&counters, kPasses * sizeof(int), st));
  JZ_CUDA(cudaMemsetAsync(counters, 0, kPasses * sizeof(int), st));
  JZ_CUDA(cudaMallocAsync(&kbuf[0], n * sizeof(uint64_t), st));
  JZ_CUDA(cudaMallocAsync(&vbuf[0], n * sizeof(uint32_t), st));
  const int np = (int)passes.size();
  float4 *pos4 = nullptr;  // aligned float4 copy written by the first pass (xyz input, >= 2 passes)
  if (!gidx_mode && np > 1) JZ_CUDA(cudaMallocAsync(&pos4, n * sizeof(float4), st));
  if (np > 1) {
    JZ_CUDA(cudaMallocAsync(&kbuf[1], n * sizeof(uint64_t), st));
    JZ_CUDA(cudaMallocAsync(&vbuf[1], n * sizeof(uint32_t), st));
  }
  for (int i = 0; i < np; ++i) {
    const int p = passes[i];
    const bool first = i == 0, last = i == np - 1;
    JZ_CUDA(cudaMemsetAsync(status, 0, (size_t)ntiles * kRadix * sizeof(unsigned long long), st));
    const uint64_t *ki = first ? nullptr : kbuf[(i - 1) & 1];
    const uint32_t *vi = first ? nullptr : vbuf[(i - 1) & 1];
    uint64_t *ko = last ? keys_out : kbuf[i & 1];
    uint32_t *vo = last ? (uint32_t *)perm_out : vbuf[i & 1];
    const unsigned *db = dhist + p * kRadix;
    int *tc = counters + i;
    dim3 g((unsigned)ntiles);
#define JZ_PASS(F, L)                                                                                          \
  k_onesweep<F, L><<<g, kSortThreads, 0, st>>>(pos, stride, gidx_mode, gidx_base, frame, pos4, ki, vi, ko, vo, pts_out, \
                                               n, 8 * p, db, status, tc)
    if (first && last) JZ_PASS(true, true);
    else if (first) JZ_PASS(true, false);
    else if (last) JZ_PASS(false, true);
    else JZ_PASS(false, false);
#undef JZ_PASS
    JZ_LAUNCH_CHECK();
  }
  JZ_CUDA(cudaFreeAsync(status, st));
  JZ_CUDA(cudaFreeAsync(counters, st));
  if (pos4) JZ_CUDA(cudaFreeAsync(pos4, st));
  JZ_CUDA(cudaFreeAsync(kbuf[0], st));
  JZ_CUDA(cudaFreeAsync(vbuf[0], st));
  if (kbuf[1]) JZ_CUDA(cudaFreeAsync(kbuf[1], st));
  if (vbuf[1]) JZ_CUDA(cudaFreeAsync(vbuf[1], st));
  JZ_CUDA(cudaFreeAsync(dhist, st));
}

static bool g_force8 = getenv("JZ_SORT8") != nullptr;  // diagnostics: always the 8-pass sort

void sort_points(const float *pos, int64_t n, int stride, int gidx_mode, int64_t gidx_base, const Frame &frame,
                 uint64_t *keys_out, int32_t *perm_out, float4 *pts_out, cudaStream_t st) {
  if (g_force8) {
    sort_points8(pos, n, stride, gidx_mode, gidx_base, frame, keys_out, perm_out, pts_out, st);
    return;
  }
  // scratch: histograms [4][256], fix-up counters {nbig, fallback}, big-run queue
  constexpr int kBigCap = 1 << 16;
  unsigned int *dhist = nullptr;
  int *dcnt = nullptr;
  int64_t *big = nullptr;
  JZ_CUDA(cudaMallocAsync(&dhist, kS32Passes * kRadix * sizeof(unsigned), st));
  JZ_CUDA(cudaMemsetAsync(dhist, 0, kS32Passes * kRadix * sizeof(unsigned), st));
  k_hist32<<<grid_for(n, 256, 148 * 4), 256, 0, st>>>(pos, n, stride, frame, dhist);
  JZ_LAUNCH_CHECK();
  std::vector<unsigned> hist(kS32Passes * kRadix);
  JZ_CUDA(cudaMemcpyAsync(hist.data(), dhist, hist.size() * sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  JZ_CUDA(cudaStreamSynchronize(st));
  std::vector<unsigned> bases(kS32Passes * kRadix);
  std::vector<int> passes;
  for (int p = 0; p < kS32Passes; ++p) {
    unsigned acc = 0;
    bool trivial = false;
    for (int b = 0; b < kRadix; ++b) {
      bases[p * kRadix + b] = acc;
      if (hist[p * kRadix + b] == (unsigned)n) trivial = true;
      acc += hist[p * kRadix + b];
    }
    if (!trivial) passes.push_back(p);
  }
  if (passes.empty()) passes.push_back(0);
  JZ_CUDA(cudaMemcpyAsync(dhist, bases.data(), bases.size() * sizeof(unsigned), cudaMemcpyHostToDevice, st));
  const int64_t ntiles = ceil_div(n, kS32Tile);
  unsigned long long *status = nullptr;
  int *counters = nullptr;
  uint32_t *kbuf[2] = {nullptr, nullptr}, *vbuf[2] = {nullptr, nullptr};
  const int np = (int)passes.size();
  JZ_CUDA(cudaMallocAsync(&status, (size_t)ntiles * kRadix * sizeof(unsigned long long), st));
  JZ_CUDA(cudaMallocAsync(&counters, (kS32Passes + 2) * sizeof(int), st));
  JZ_CUDA(cudaMemsetAsync(counters, 0, (kS32Passes + 2) * sizeof(int), st));
  for (int b = 0; b < (np > 2 ? 2 : np - 1); ++b) {
    JZ_CUDA(cudaMallocAsync(&kbuf[b], n * sizeof(uint32_t), st));
    JZ_CUDA(cudaMallocAsync(&vbuf[b], n * sizeof(uint32_t), st));
  }
  for (int i = 0; i < np; ++i) {
    const int p = passes[i];
    const bool first = i == 0, last = i == np - 1;
    JZ_CUDA(cudaMemsetAsync(status, 0, (size_t)ntiles * kRadix * sizeof(unsigned long long), st));
    const uint32_t *ki = first ? nullptr : kbuf[(i - 1) & 1];
    const uint32_t *vi = first ? nullptr : vbuf[(i - 1) & 1];
    uint32_t *ko = last ? nullptr : kbuf[i & 1];
    uint32_t *vo = last ? (uint32_t *)perm_out : vbuf[i & 1];
#define JZ_PASS32(F, L)                                                                                            \
  k_onesweep32<F, L><<<(unsigned)ntiles, kS32Threads, 0, st>>>(pos, stride, gidx_mode, gidx_base, frame, ki, vi, ko, vo, \
                                                             keys_out, pts_out, n, p == 0 ? 0 : 8 * (p - 1),      \
                                                             p == 0, dhist + p * kRadix, status, counters + i)
    if (first && last) JZ_PASS32(true, true);
    else if (first) JZ_PASS32(true, false);
    else if (last) JZ_PASS32(false, true);
    else JZ_PASS32(false, false);
#undef JZ_PASS32
    JZ_LAUNCH_CHECK();
  }
  // fix-up of runs of equal high keys
  JZ_CUDA(cudaMallocAsync(&big, kBigCap * sizeof(int64_t), st));
  int *nbig = counters + kS32Passes, *fallback = counters + kS32Passes + 1;
  k_seg_fix<<<grid_for(n, 256, 148 * 8), 256, 0, st>>>(keys_out, perm_out, pts_out, n, big, nbig, kBigCap, fallback);
  JZ_LAUNCH_CHECK();
  k_seg_block<<<148 * 2, 512, 0, st>>>(keys_out, perm_out, pts_out, n, big, nbig, kBigCap, pos, stride, gidx_mode,
                                       gidx_base, fallback);
  JZ_LAUNCH_CHECK();
  int fb = 0;
  JZ_CUDA(cudaMemcpyAsync(&fb, fallback, sizeof(int), cudaMemcpyDeviceToHost, st));
  JZ_CUDA(cudaFreeAsync(status, st));
  JZ_CUDA(cudaFreeAsync(counters, st));
  JZ_CUDA(cudaFreeAsync(big, st));
  for (int b = 0; b < 2; ++b) {
    if (kbuf[b]) JZ_CUDA(cudaFreeAsync(kbuf[b], st));
    if (vbuf[b]) JZ_CUDA(cudaFreeAsync(vbuf[b], st));
  }
  JZ_CUDA(cudaFreeAsync(dhist, st));
  JZ_CUDA(cudaStreamSynchronize(st));
  // a run of > kSegBlock equal high keys (heavy duplicates): redo with the full-key passes
  if (fb) sort_points8(pos, n, stride, gidx_mode, gidx_base, frame, keys_out, perm_out, pts_out, st);
}

// ---------------------------------------------------------------- stable sort of 32-bit (key, value) pairs
// (friends-of-friends group order): the one-sweep passes above over the key bytes
__global__ void __launch_bounds__(256) k_hist_u32(const uint32_t *__restrict__ k, int64_t n,
                                                  unsigned int *__restrict__ hist /*[4][256]*/) {
  __shared__ unsigned int s_h[4][kRadix];
  for (int i = threadIdx.x; i < 4 * kRadix; i += blockDim.x) (&s_h[0][0])[i] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t v = k[i];
#pragma unroll
    for (int ps = 0; ps < 4; ++ps) atomicAdd(&s_h[ps][(v >> (8 * ps)) & 255], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 4 * kRadix; i += blockDim.x) {
    const unsigned v = (&s_h[0][0])[i];
    if (v) atomicAdd(&hist[i], v);
  }
}

void sort_pairs_u32(const uint32_t *keys, const uint32_t *vals, int64_t n, uint32_t *keys_out, uint32_t *vals_out,
                    cudaStream_t st) {
  if (n <= 0) return;
  unsigned int *dhist = nullptr;
  JZ_CUDA(cudaMallocAsync(&dhist, 4 * kRadix * sizeof(unsigned), st));
  JZ_CUDA(cudaMemsetAsync(dhist, 0, 4 * kRadix * sizeof(unsigned), st));
  k_hist_u32<<<grid_for(n, 256, 148 * 4), 256, 0, st>>>(keys, n, dhist);
  JZ_LAUNCH_CHECK();
  std::vector<unsigned> hist(4 * kRadix), bases(4 * kRadix);
  JZ_CUDA(cudaMemcpyAsync(hist.data(), dhist, hist.size() * sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  JZ_CUDA(cudaStreamSynchronize(st));
  std::vector<int> passes;
  for (int p = 0; p < 4; ++p) {
    unsigned acc = 0;
    bool trivial = false;
    for (int b = 0; b < kRadix; ++b) {
      bases[p * kRadix + b] = acc;
      if (hist[p * kRadix + b] == (unsigned)n) trivial = true;
      acc += hist[p * kRadix + b];
    }
    if (!trivial) passes.push_back(p);
  }
  JZ_CUDA(cudaMemcpyAsync(dhist, bases.data(), bases.size() * sizeof(unsigned), cudaMemcpyHostToDevice, st));
  const int64_t ntiles = ceil_div(n, kS32Tile);
  unsigned long long *status = nullptr;
  int *counters = nullptr;
  uint32_t *tk = nullptr, *tv = nullptr;
  JZ_CUDA(cudaMallocAsync(&status, (size_t)ntiles * kRadix * sizeof(unsigned long long), st));
  JZ_CUDA(cudaMallocAsync(&counters, 4 * sizeof(int), st));
  JZ_CUDA(cudaMemsetAsync(counters, 0, 4 * sizeof(int), st));
  JZ_CUDA(cudaMallocAsync(&tk, n * sizeof(uint32_t), st));
  JZ_CUDA(cudaMallocAsync(&tv, n * sizeof(uint32_t), st));
  const uint32_t *ki = keys, *vi = vals;
  const int np = (int)passes.size();
  for (int i = 0; i < np; ++i) {
    // ping-pong so that the last pass lands in keys_out / vals_out
    const bool to_out = ((np - 1 - i) & 1) == 0;
    uint32_t *ko = to_out ? keys_out : tk, *vo = to_out ? vals_out : tv;
    JZ_CUDA(cudaMemsetAsync(status, 0, (size_t)ntiles * kRadix * sizeof(unsigned long long), st));
    k_onesweep32<false, false><<<(unsigned)ntiles, kS32Threads, 0, st>>>(nullptr, 0, 0, 0, Frame{}, ki, vi, ko, vo,
                                                                          nullptr, nullptr, n, 8 * passes[i], 0,
                                                                          dhist + passes[i] * kRadix, status, counters + i);
    JZ_LAUNCH_CHECK();
    ki = ko;
    vi = vo;
  }
  if (np == 0) {  // already sorted (one key value)
    JZ_CUDA(cudaMemcpyAsync(keys_out, keys, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
    JZ_CUDA(cudaMemcpyAsync(vals_out, vals, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
  }
  JZ_CUDA(cudaFreeAsync(status, st));
  JZ_CUDA(cudaFreeAsync(counters, st));
  JZ_CUDA(cudaFreeAsync(tk, st));
  JZ_CUDA(cudaFreeAsync(tv, st));
  JZ_CUDA(cudaFreeAsync(dhist, st));
}

// Morton keys only (multi-GPU splitter step)
__global__ void k_keys(const float *__restrict__ pos, int64_t n, Frame f, uint64_t *__restrict__ keys) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    keys[i] = morton(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], f);
}

void morton_keys(const float *pos, int64_t n, const Frame &f, uint64_t *keys, cudaStream_t st) {
  k_keys<<<grid_for(n, 256), 256, 0, st>>>(pos, n, f, keys);
  JZ_LAUNCH_CHECK();
}

}  // namespace jz
