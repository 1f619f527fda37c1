// jz_build.cu -- plane-based tree hierarchy (§2.3).
//
//  A4 levels        lvl_g = bitlen(key_{g-1} xor key_g) for gaps g in [1, N-1]; lvl_0 = lvl_N = 64
//                    (integer-key reading DESIGN.md R4/R5), computed on the fly.
//  A5 k_leaf_flags   gap g is a leaf split iff n_g > N_max^(0), where n_g is the size of the Morton
//                    cell at level lvl_g holding points g-1 and g (= the distance between the
//                    nearest gaps with a strictly greater level, = the paper's binary-search
//                    definition; pinned by tests/test_oracle_tree.py). Decided inside a
//                    +-N_max^(0) window of keys staged in shared memory with two binary searches
//                    (P:L253 step (2) "range search").
//     compaction     scan + scatter -> spl^(0).
//  A6 k_split_n      exact n at every leaf split by the paper's two binary searches on the
//                    sorted keys (P:L147-155, P:L253 step (3)).
//  A7 planes         spl^(p) = leaf splits with n > N_max^(0) c^p, stored as positions in plane
//                    p-1's split array (Fig. 3); plane p >= 1 exists iff
//                    2N / N_max^(p) >= N_target.
//  A8 boxes          exact FP32 AABB + point count per node; leaves reduce over their points,
//                    coarser planes over their children (R7: AABBs instead of
//                    Morton-cell centre/level boxes).
#include <climits>
#include <vector>

#include "jz_common.cuh"
#include "jz_internal.h"

namespace jz {

constexpr int kFlagBlock = 512;

// Leaf-split test (P:L253 step (2)): gap g is a split iff the Morton cell at level
// lvl_g = bitlen(key_{g-1} ^ key_g) holding points g-1 and g has more than W = N_max^(0) points.
// The cell is the contiguous run of keys sharing key >> lvl_g (a node is the set of
// points sharing the leading bits), so n <= W can be decided inside a +-W window of keys staged
// in shared memory with two binary searches (<= 2 log2 W probes per gap).
__global__ void __launch_bounds__(kFlagBlock) k_leaf_flags(const uint64_t *__restrict__ keys, int64_t n, int W,
                                                           int32_t *__restrict__ flag) {
  extern __shared__ uint64_t s_k[];
  const int64_t b0 = (int64_t)blockIdx.x * kFlagBlock;
  const int64_t w0 = b0 - W - 1;
  const int len = kFlagBlock + 2 * W + 2;
  for (int i = threadIdx.x; i < len; i += blockDim.x) {
    const int64_t g = w0 + i;
    s_k[i] = (g < 0 || g >= n) ? 0ull : keys[g];
  }
  __syncthreads();
  const int64_t g = b0 + threadIdx.x;
  if (g > n) return;
  int f = 1;
  if (g > 0 && g < n) {
    const uint64_t kg = s_k[g - w0], kg1 = s_k[g - 1 - w0];
    const int l = 64 - __clzll((long long)(kg1 ^ kg));
    const uint64_t p = l >= 64 ? 0ull : (kg >> l);
    auto pre = [&](int64_t i) { return l >= 64 ? 0ull : (s_k[i - w0] >> l); };
    // L_b: first index of the cell; if it starts before g - W the cell has > W points
    const int64_t lo_lim = g - W > 0 ? g - W : 0;
    if (!(g - W >= 1 && pre(g - W) == p)) {
      int64_t lo = lo_lim, hi = g - 1;  // smallest a in [lo, g-1] with prefix == p (true at g-1)
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (pre(mid) == p) hi = mid;
        else lo = mid + 1;
      }
      const int64_t Lb = lo;
      // R_b: first index after the cell; n = R_b - L_b <= W iff R_b <= L_b + W
      const int64_t rmax = Lb + W < n ? Lb + W : n;  // R_b = n if the cell reaches the end
      if (rmax >= n) {
        f = (n - Lb) > W;
        if (f == 0) {
          // the cell ends at n only if every key up to n-1 shares the prefix
          int64_t lo2 = g, hi2 = n;
          while (lo2 < hi2) {
            const int64_t mid = (lo2 + hi2) >> 1;
            if (pre(mid) != p) hi2 = mid;
            else lo2 = mid + 1;
          }
          f = (lo2 - Lb) > W;
        }
      } else {
        f = pre(rmax) == p;  // cell still continues at L_b + W => n > W
      }
    }
  }
  flag[g] = f;
}

__global__ void k_compact_gaps(const int32_t *__restrict__ flag, const int64_t *__restrict__ pos, int64_t m,
                               int32_t *__restrict__ out) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < m; g += (int64_t)gridDim.x * blockDim.x)
    if (flag[g]) out[pos[g]] = (int32_t)g;
}

// n at every leaf split by binary search on keys.
__global__ void k_split_n(const uint64_t *__restrict__ keys, int64_t n, const int32_t *__restrict__ spl,
                          int64_t nspl, int32_t *__restrict__ nsplit) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nspl; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = spl[j];
    if (g <= 0 || g >= n) {
      nsplit[j] = INT_MAX;
      continue;
    }
    const uint64_t kg = keys[g], kg1 = keys[g - 1];
    const int l = 64 - __clzll((long long)(kg1 ^ kg));
    // l_b: smallest a in [0, g-1] with bitlen(key_a ^ key_g) <= l
    int64_t lo = 0, hi = g - 1;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (64 - __clzll((long long)(keys[mid] ^ kg)) <= l) hi = mid;
      else lo = mid + 1;
    }
    const int64_t lb = lo;
    // r_b: smallest r in [g, N) with bitlen(key_{g-1} ^ key_r) > l, N if none
    lo = g;
    hi = n;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (64 - __clzll((long long)(kg1 ^ keys[mid])) > l) hi = mid;
      else lo = mid + 1;
    }
    int64_t v = lo - lb;
    nsplit[j] = v > INT_MAX ? INT_MAX : (int32_t)v;
  }
}

__global__ void k_plane_flags(const int32_t *__restrict__ leafspl_prev, int64_t m, const int32_t *__restrict__ nsplit,
                              int64_t nmax, int32_t *__restrict__ flag) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x)
    flag[j] = (int64_t)nsplit[leafspl_prev[j]] > nmax;
}

__global__ void k_plane_compact(const int32_t *__restrict__ flag, const int64_t *__restrict__ pos,
                                const int32_t *__restrict__ leafspl_prev, int64_t m, int32_t *__restrict__ beg,
                                int32_t *__restrict__ leafspl) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x)
    if (flag[j]) {
      int64_t p = pos[j];
      beg[p] = (int32_t)j;
      leafspl[p] = leafspl_prev[j];
    }
}

__global__ void k_iota(int32_t *__restrict__ a, int64_t m) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x)
    a[j] = (int32_t)j;
}

// one warp per leaf: AABB of its points (all types) + number of SOURCE points (gidx >= 0):
// the count heap of FindRmax counts neighbour candidates (P:L276-279 joint tree over types)
__global__ void k_leaf_boxes(const float4 *__restrict__ pts, const int32_t *__restrict__ beg, int64_t nleaf,
                             NodeBox *__restrict__ box) {
  const int lane = threadIdx.x & 31;
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (; w < nleaf; w += nw) {
    const int b = beg[w], e = beg[w + 1];
    float lx = INFINITY, ly = INFINITY, lz = INFINITY, hx = -INFINITY, hy = -INFINITY, hz = -INFINITY;
    int ns = 0;
    for (int i = b + lane; i < e; i += 32) {
      float4 p = pts[i];
      ns += __float_as_int(p.w) >= 0;
      lx = fminf(lx, p.x);
      ly = fminf(ly, p.y);
      lz = fminf(lz, p.z);
      hx = fmaxf(hx, p.x);
      hy = fmaxf(hy, p.y);
      hz = fmaxf(hz, p.z);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lx = fminf(lx, __shfl_xor_sync(0xffffffffu, lx, o));
      ly = fminf(ly, __shfl_xor_sync(0xffffffffu, ly, o));
      lz = fminf(lz, __shfl_xor_sync(0xffffffffu, lz, o));
      hx = fmaxf(hx, __shfl_xor_sync(0xffffffffu, hx, o));
      hy = fmaxf(hy, __shfl_xor_sync(0xffffffffu, hy, o));
      hz = fmaxf(hz, __shfl_xor_sync(0xffffffffu, hz, o));
      ns += __shfl_xor_sync(0xffffffffu, ns, o);
    }
    if (lane == 0) {
      NodeBox nb;
      nb.lo = make_float4(lx, ly, lz, __int_as_float(ns));
      nb.hi = make_float4(hx, hy, hz, 0.f);
      box[w] = nb;
    }
  }
}

// one warp per node of plane p: AABB over its children in plane p-1
__global__ void k_node_boxes(const NodeBox *__restrict__ child, const int32_t *__restrict__ beg, int64_t nnodes,
                             NodeBox *__restrict__ box) {
  const int lane = threadIdx.x & 31;
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (; w < nnodes; w += nw) {
    const int b = beg[w], e = beg[w + 1];
    float lx = INFINITY, ly = INFINITY, lz = INFINITY, hx = -INFINITY, hy = -INFINITY, hz = -INFINITY;
    int cnt = 0;
    for (int i = b + lane; i < e; i += 32) {
      NodeBox c = child[i];
      lx = fminf(lx, c.lo.x);
      ly = fminf(ly, c.lo.y);
      lz = fminf(lz, c.lo.z);
      hx = fmaxf(hx, c.hi.x);
      hy = fmaxf(hy, c.hi.y);
      hz = fmaxf(hz, c.hi.z);
      cnt += __float_as_int(c.lo.w);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lx = fminf(lx, __shfl_xor_sync(0xffffffffu, lx, o));
      ly = fminf(ly, __shfl_xor_sync(0xffffffffu, ly, o));
      lz = fminf(lz, __shfl_xor_sync(0xffffffffu, lz, o));
      hx = fmaxf(hx, __shfl_xor_sync(0xffffffffu, hx, o));
      hy = fmaxf(hy, __shfl_xor_sync(0xffffffffu, hy, o));
      hz = fmaxf(hz, __shfl_xor_sync(0xffffffffu, hz, o));
      cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    }
    if (lane == 0) {
      NodeBox nb;
      nb.lo = make_float4(lx, ly, lz, __int_as_float(cnt));
      nb.hi = make_float4(hx, hy, hz, 0.f);
      box[w] = nb;
    }
  }
}

// ---------------------------------------------------------------- regularisation
// PAPER.md §2.4 "Regularization", readings DESIGN.md R18-R20: node volume 2^lvl with
// lvl = bitlen(first key ^ last key); V_90% over the count-based nodes of the plane in (volume,
// index) order until 90% of the points are covered (the crossing node included); lvl_max = the
// largest l with 2^l <= f_max V_90% (exact integer arithmetic); non-decreasing over planes; every
// gap (leaf plane) or leaf split (plane p >= 1) with a level above lvl_max becomes a split.
__device__ __forceinline__ int gap_level(const uint64_t *__restrict__ keys, int64_t n, int64_t g) {
  return (g <= 0 || g >= n) ? kLevelSentinel : 64 - __clzll((long long)(keys[g - 1] ^ keys[g]));
}

// node i = sorted points [beg[s(i)], beg[s(i+1)]) with s = leafspl (planes >= 1) or identity
__global__ void k_node_levels(const uint64_t *__restrict__ keys, const int32_t *__restrict__ beg,
                              const int32_t *__restrict__ leafspl, int64_t nnodes, uint8_t *__restrict__ lvl,
                              int32_t *__restrict__ cnt, unsigned long long *__restrict__ hist) {
  __shared__ unsigned long long s_h[kLevelSentinel + 1];
  for (int i = threadIdx.x; i <= kLevelSentinel; i += blockDim.x) s_h[i] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnodes; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = beg[leafspl ? leafspl[i] : i], b = beg[leafspl ? leafspl[i + 1] : i + 1];
    const int c = (int)(b - a);
    const int l = c >= 2 ? 64 - __clzll((long long)(keys[a] ^ keys[b - 1])) : 0;
    lvl[i] = (uint8_t)l;
    cnt[i] = c;
    atomicAdd(&s_h[l], (unsigned long long)c);
  }
  __syncthreads();
  for (int i = threadIdx.x; i <= kLevelSentinel; i += blockDim.x)
    if (s_h[i]) atomicAdd(&hist[i], s_h[i]);
}

__global__ void k_level_select(const uint8_t *__restrict__ lvl, const int32_t *__restrict__ cnt, int64_t m, int b,
                               int32_t *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = lvl[i] == b ? cnt[i] : 0;
}

// first node (index order) of level b whose inclusive prefix count reaches rem
__global__ void k_first_reach(const uint8_t *__restrict__ lvl, const int32_t *__restrict__ cnt,
                              const int64_t *__restrict__ pre, int64_t m, int b, int64_t rem,
                              unsigned long long *__restrict__ best) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    if (lvl[i] == b && pre[i] + cnt[i] >= rem) atomicMin(best, (unsigned long long)i);
}

__global__ void k_force_gaps(const uint64_t *__restrict__ keys, int64_t n, int lm, int32_t *__restrict__ flag) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g <= n; g += (int64_t)gridDim.x * blockDim.x)
    if (gap_level(keys, n, g) > lm) flag[g] = 1;
}

__global__ void k_force_splits(const uint64_t *__restrict__ keys, int64_t n, const int32_t *__restrict__ leafbeg,
                               const int32_t *__restrict__ leafspl_prev, int64_t m, int lm,
                               int32_t *__restrict__ flag) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x)
    if (gap_level(keys, n, leafbeg[leafspl_prev[j]]) > lm) flag[j] = 1;
}

// lvl_max of the nodes [beg[s(i)], beg[s(i+1)]), host-side exact arithmetic
static int level_max_of(const uint64_t *keys, const int32_t *beg, const int32_t *leafspl, int64_t nnodes, int fmax,
                        cudaStream_t st) {
  typedef unsigned __int128 u128;
  uint8_t *lvl = nullptr;
  int32_t *cnt = nullptr, *sel = nullptr;
  int64_t *pre = nullptr;
  unsigned long long *hist = nullptr;
  JZ_CUDA(cudaMallocAsync(&lvl, nnodes, st));
  JZ_CUDA(cudaMallocAsync(&cnt, nnodes * sizeof(int32_t), st));
  JZ_CUDA(cudaMallocAsync(&hist, (kLevelSentinel + 2) * sizeof(unsigned long long), st));
  JZ_CUDA(cudaMemsetAsync(hist, 0, (kLevelSentinel + 1) * sizeof(unsigned long long), st));
  k_node_levels<<<grid_for(nnodes, 256), 256, 0, st>>>(keys, beg, leafspl, nnodes, lvl, cnt, hist);
  JZ_LAUNCH_CHECK();
  unsigned long long h[kLevelSentinel + 1];
  JZ_CUDA(cudaMemcpyAsync(h, hist, sizeof(h), cudaMemcpyDeviceToHost, st));
  JZ_CUDA(cudaStreamSynchronize(st));
  u128 total = 0;
  for (int l = 0; l <= kLevelSentinel; ++l) total += h[l];
  u128 cum = 0, num = 0;
  int b = 0;
  for (; b <= kLevelSentinel; ++b) {
    if (10 * (cum + h[b]) >= 9 * total) break;
    cum += h[b];
    num += (u128)h[b] << b;
  }
  // part of level b: the shortest index-order prefix of its nodes reaching the 90% mark
  const int64_t rem = (int64_t)((9 * total - 10 * cum + 9) / 10);
  u128 part = 0;
  if (rem > 0) {
    JZ_CUDA(cudaMallocAsync(&sel, nnodes * sizeof(int32_t), st));
    JZ_CUDA(cudaMallocAsync(&pre, (nnodes + 1) * sizeof(int64_t), st));
    k_level_select<<<grid_for(nnodes, 256), 256, 0, st>>>(lvl, cnt, nnodes, b, sel);
    JZ_LAUNCH_CHECK();
    exclusive_scan_i32_to_i64(sel, pre, nnodes, st);
    unsigned long long *best = hist + kLevelSentinel + 1;
    const unsigned long long inf = ~0ull;
    JZ_CUDA(cudaMemcpyAsync(best, &inf, sizeof(inf), cudaMemcpyHostToDevice, st));
    k_first_reach<<<grid_for(nnodes, 256), 256, 0, st>>>(lvl, cnt, pre, nnodes, b, rem, best);
    JZ_LAUNCH_CHECK();
    unsigned long long ib = 0;
    JZ_CUDA(cudaMemcpyAsync(&ib, best, sizeof(ib), cudaMemcpyDeviceToHost, st));
    JZ_CUDA(cudaStreamSynchronize(st));
    int64_t pv = 0;
    int32_t cv = 0;
    JZ_CUDA(cudaMemcpy(&pv, pre + ib, sizeof(pv), cudaMemcpyDeviceToHost));
    JZ_CUDA(cudaMemcpy(&cv, cnt + ib, sizeof(cv), cudaMemcpyDeviceToHost));
    part = (u128)(pv + cv);
    JZ_CUDA(cudaFreeAsync(sel, st));
    JZ_CUDA(cudaFreeAsync(pre, st));
  }
  num += part << b;
  const u128 den = cum + part;
  int lm = 0;
  while (lm < 120 && ((u128)1 << (lm + 1)) * den <= (u128)fmax * num) ++lm;
  JZ_CUDA(cudaFreeAsync(lvl, st));
  JZ_CUDA(cudaFreeAsync(cnt, st));
  JZ_CUDA(cudaFreeAsync(hist, st));
  return lm;
}

void free_planes(std::vector<Plane> &planes, cudaStream_t st) {
  for (auto &p : planes) {
    if (p.beg) cudaFreeAsync(p.beg, st);
    if (p.leafspl) cudaFreeAsync(p.leafspl, st);
    if (p.box) cudaFreeAsync(p.box, st);
    p = Plane();
  }
  planes.clear();
}

void build_planes(const uint64_t *keys, const float4 *pts, int64_t n, const jz_knn_params_t &prm,
                  std::vector<Plane> &planes, cudaStream_t st) {
  const int W = prm.nmax0;
  int32_t *flag = nullptr;
  int64_t *pos = nullptr;
  JZ_CUDA(cudaMallocAsync(&flag, (n + 1) * sizeof(int32_t), st));
  JZ_CUDA(cudaMallocAsync(&pos, (n + 2) * sizeof(int64_t), st));
  const unsigned fb = (unsigned)ceil_div(n + 1, kFlagBlock);
  k_leaf_flags<<<fb, kFlagBlock, (kFlagBlock + 2 * W + 2) * sizeof(uint64_t), st>>>(keys, n, W, flag);
  JZ_LAUNCH_CHECK();
  exclusive_scan_i32_to_i64(flag, pos, n + 1, st);
  int64_t nspl = read_i64(pos + (n + 1), st);  // = N_leaf + 1
  Plane leaf;
  leaf.nnodes = nspl - 1;
  leaf.nmax = W;
  JZ_CUDA(cudaMallocAsync(&leaf.beg, nspl * sizeof(int32_t), st));
  k_compact_gaps<<<grid_for(n + 1, 256), 256, 0, st>>>(flag, pos, n + 1, leaf.beg);
  JZ_LAUNCH_CHECK();
  const int fmax = prm.reg_fmax;
  if (fmax > 0) {  // regularisation of the leaf plane
    leaf.lvl_max = level_max_of(keys, leaf.beg, nullptr, leaf.nnodes, fmax, st);
    k_force_gaps<<<grid_for(n + 1, 256), 256, 0, st>>>(keys, n, leaf.lvl_max, flag);
    JZ_LAUNCH_CHECK();
    exclusive_scan_i32_to_i64(flag, pos, n + 1, st);
    const int64_t nspl2 = read_i64(pos + (n + 1), st);
    if (nspl2 != nspl) {
      JZ_CUDA(cudaFreeAsync(leaf.beg, st));
      nspl = nspl2;
      leaf.nnodes = nspl - 1;
      JZ_CUDA(cudaMallocAsync(&leaf.beg, nspl * sizeof(int32_t), st));
      k_compact_gaps<<<grid_for(n + 1, 256), 256, 0, st>>>(flag, pos, n + 1, leaf.beg);
      JZ_LAUNCH_CHECK();
    }
  }
  JZ_CUDA(cudaMallocAsync(&leaf.leafspl, nspl * sizeof(int32_t), st));
  JZ_CUDA(cudaMallocAsync(&leaf.box, leaf.nnodes * sizeof(NodeBox), st));
  k_iota<<<grid_for(nspl, 256), 256, 0, st>>>(leaf.leafspl, nspl);
  JZ_LAUNCH_CHECK();
  int32_t *nsplit = nullptr;
  JZ_CUDA(cudaMallocAsync(&nsplit, nspl * sizeof(int32_t), st));
  k_split_n<<<grid_for(nspl, 128), 128, 0, st>>>(keys, n, leaf.beg, nspl, nsplit);
  JZ_LAUNCH_CHECK();
  k_leaf_boxes<<<grid_for(leaf.nnodes * 32, 256), 256, 0, st>>>(pts, leaf.beg, leaf.nnodes, leaf.box);
  JZ_LAUNCH_CHECK();
  planes.push_back(leaf);
  // coarser planes
  int64_t nmax = W;
  while (true) {
    if (nmax > (int64_t)INT_MAX / prm.coarsen) break;
    nmax *= prm.coarsen;
    if (2.0 * (double)n / (double)nmax < (double)prm.ntarget) break;
    const Plane &pv = planes.back();
    const int64_t m = pv.nnodes + 1;
    k_plane_flags<<<grid_for(m, 256), 256, 0, st>>>(pv.leafspl, m, nsplit, nmax, flag);
    JZ_LAUNCH_CHECK();
    exclusive_scan_i32_to_i64(flag, pos, m, st);
    int64_t np1 = read_i64(pos + m, st);
    Plane pl;
    pl.nnodes = np1 - 1;
    pl.nmax = nmax;
    JZ_CUDA(cudaMallocAsync(&pl.beg, np1 * sizeof(int32_t), st));
    JZ_CUDA(cudaMallocAsync(&pl.leafspl, np1 * sizeof(int32_t), st));
    k_plane_compact<<<grid_for(m, 256), 256, 0, st>>>(flag, pos, pv.leafspl, m, pl.beg, pl.leafspl);
    JZ_LAUNCH_CHECK();
    if (fmax > 0) {  // regularisation of plane p, lvl_max non-decreasing (nesting)
      const int lm = level_max_of(keys, planes[0].beg, pl.leafspl, pl.nnodes, fmax, st);
      pl.lvl_max = lm > pv.lvl_max ? lm : pv.lvl_max;
      k_force_splits<<<grid_for(m, 256), 256, 0, st>>>(keys, n, planes[0].beg, pv.leafspl, m, pl.lvl_max, flag);
      JZ_LAUNCH_CHECK();
      exclusive_scan_i32_to_i64(flag, pos, m, st);
      const int64_t np2 = read_i64(pos + m, st);
      if (np2 != np1) {
        JZ_CUDA(cudaFreeAsync(pl.beg, st));
        JZ_CUDA(cudaFreeAsync(pl.leafspl, st));
        np1 = np2;
        pl.nnodes = np1 - 1;
        JZ_CUDA(cudaMallocAsync(&pl.beg, np1 * sizeof(int32_t), st));
        JZ_CUDA(cudaMallocAsync(&pl.leafspl, np1 * sizeof(int32_t), st));
        k_plane_compact<<<grid_for(m, 256), 256, 0, st>>>(flag, pos, pv.leafspl, m, pl.beg, pl.leafspl);
        JZ_LAUNCH_CHECK();
      }
    }
    JZ_CUDA(cudaMallocAsync(&pl.box, pl.nnodes * sizeof(NodeBox), st));
    k_node_boxes<<<grid_for(pl.nnodes * 32, 256), 256, 0, st>>>(pv.box, pl.beg, pl.nnodes, pl.box);
    JZ_LAUNCH_CHECK();
    planes.push_back(pl);
  }
  JZ_CUDA(cudaFreeAsync(nsplit, st));
  JZ_CUDA(cudaFreeAsync(flag, st));
  JZ_CUDA(cudaFreeAsync(pos, st));
}

}  // namespace jz
