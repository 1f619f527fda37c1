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

void sort_points(const float *pos, int64_t n, int stride, int gidx_mode, int64_t gidx_base, const Frame &frame,
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
