// jz_dist.cu -- per-rank compute of the multi-GPU path (PAPER.md L112-114
// sample-splitter partition, L388-393 distributed kNN). The exchanges themselves are
// all-gathers / all-to-allv issued by the caller through torch.distributed (NCCL).
//
//   jz_morton_keys          keys in one global frame (every rank gets identical keys)
//   jz_bucket_by_splitters  dest rank = #splitters <= key (Morton-range partition)
//   jz_pack_by_rank         float4 {x, y, z, bits(gidx)} grouped by destination rank
//   jz_knn_query_boxes      per node of a plane: AABB + max R_max^2 of its leaves (default: the
//                           NodeToNode walk to the leaf plane, Alg. 1 l. 1-5; JZ_FLAG_QBOX_DIAG:
//                           the AABB diagonal of the smallest ancestor holding k points)
//   jz_knn_select_ghosts    bitmask of peer ranks whose query boxes a local leaf reaches
//                           (exact monotone box bound d_low^2 <= r2; leaf granularity is a
//                           superset of the required points, so no neighbour can be missed)
//   jz_knn_pack_ghosts      pack flagged points per destination rank
//   jz_pack_rows            F2: result rows (idx[k], bits(d2)[k], gidx) grouped by the rank that
//                           owns their input row (reverse all-to-all-v)
//   jz_scatter_rows         F2: received rows written to input order (row = gidx - base)
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <ctime>
#include <vector>

#include "jz_comm.h"

#include "jz_common.cuh"
#include "jz_internal.h"


namespace jz {

__global__ void k_bucket(const uint64_t *__restrict__ keys, int64_t n, const uint64_t *__restrict__ spl, int nspl,
                         int32_t *__restrict__ dest, unsigned long long *__restrict__ counts) {
  __shared__ unsigned long long s_c[1024];
  for (int i = threadIdx.x; i <= nspl; i += blockDim.x) s_c[i] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[i];
    int lo = 0, hi = nspl;  // number of splitters <= k
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (spl[mid] <= k) lo = mid + 1;
      else hi = mid;
    }
    dest[i] = lo;
    atomicAdd(&s_c[lo], 1ull);
  }
  __syncthreads();
  for (int i = threadIdx.x; i <= nspl; i += blockDim.x)
    if (s_c[i]) atomicAdd(&counts[i], s_c[i]);
}

// Slot for this lane in destination r's group: one atomic per (warp, destination) instead of one
// per point (1e8 same-address atomics cost 65 ms at R = 1); order inside a group unspecified.
__device__ __forceinline__ unsigned long long warp_slot(unsigned long long *cursor, int r) {
  const unsigned act = __activemask();
  const unsigned peers = __match_any_sync(act, r);
  const int lane = threadIdx.x & 31, leader = __ffs(peers) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(&cursor[r], (unsigned long long)__popc(peers));
  base = __shfl_sync(peers, base, leader);
  return base + (unsigned long long)__popc(peers & ((1u << lane) - 1u));
}

// slots per destination rank aggregated per CTA (1024 points per round: shared-memory counters,
// then one global atomic per rank and round; per-warp atomics on the R cursors serialised: 0.6 ms
// per rank at 1.25e7 points). The order inside a destination is arbitrary (the receiver sorts).
constexpr int kPackThreads = 256, kPackIPT = 4;
__global__ void __launch_bounds__(kPackThreads) k_pack(const float *__restrict__ pos, int64_t n, int64_t gbase,
                                                       const int32_t *__restrict__ dest,
                                                       const int64_t *__restrict__ off,
                                                       unsigned long long *__restrict__ cursor, float4 *__restrict__ out) {
  __shared__ unsigned s_cnt[32];
  __shared__ unsigned long long s_base[32];
  constexpr int T = kPackThreads * kPackIPT;
  for (int64_t b = (int64_t)blockIdx.x * T; b < n; b += (int64_t)gridDim.x * T) {
    if (threadIdx.x < 32) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    int r[kPackIPT];
    unsigned loc[kPackIPT];
#pragma unroll
    for (int u = 0; u < kPackIPT; ++u) {
      const int64_t i = b + u * kPackThreads + threadIdx.x;
      r[u] = i < n ? dest[i] : -1;
      loc[u] = r[u] >= 0 ? atomicAdd(&s_cnt[r[u]], 1u) : 0u;
    }
    __syncthreads();
    if (threadIdx.x < 32 && s_cnt[threadIdx.x] > 0)
      s_base[threadIdx.x] = atomicAdd(&cursor[threadIdx.x], (unsigned long long)s_cnt[threadIdx.x]);
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kPackIPT; ++u) {
      const int64_t i = b + u * kPackThreads + threadIdx.x;
      if (r[u] >= 0)
        out[off[r[u]] + (int64_t)(s_base[r[u]] + loc[u])] =
            make_float4(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], __int_as_float((int)(gbase + i)));
    }
    __syncthreads();
  }
}

// F2: slot of each result row in the send buffer (grouped by destination rank)
__global__ void k_row_slots(const int32_t *__restrict__ dest, int64_t m, const int64_t *__restrict__ off,
                            unsigned long long *__restrict__ cursor, int64_t *__restrict__ slot) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = dest[i];
    slot[i] = off[r] + (int64_t)warp_slot(cursor, r);
  }
}

// one thread per output word: row i -> words [idx[k], bits(d2)[k], gidx] at slot[i]
__global__ void k_pack_rows(const int32_t *__restrict__ idx, const float *__restrict__ d2,
                            const int32_t *__restrict__ rowg, int64_t m, int k, const int64_t *__restrict__ slot,
                            int32_t *__restrict__ out) {
  const int W = 2 * k + 1;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < m * W; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / W;
    const int w = (int)(t - i * W);
    const int32_t v = w < k ? idx[i * k + w] : (w < 2 * k ? __float_as_int(d2[i * k + (w - k)]) : rowg[i]);
    out[slot[i] * W + w] = v;
  }
}

// one thread per received word: row j goes to input row gidx - base (flag on a bad gidx)
__global__ void k_scatter_rows(const int32_t *__restrict__ rows, int64_t m, int k, int64_t base, int64_t n,
                               int32_t *__restrict__ out_idx, float *__restrict__ out_d2, int *__restrict__ bad) {
  const int W = 2 * k + 1;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < m * 2 * k; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t / (2 * k);
    const int w = (int)(t - j * 2 * k);
    const int64_t row = (int64_t)rows[j * W + 2 * k] - base;
    if (row < 0 || row >= n) {
      *bad = 1;
      continue;
    }
    const int32_t v = rows[j * W + w];
    if (w < k) out_idx[row * k + w] = v;
    else out_d2[row * k + (w - k)] = __int_as_float(v);
  }
}

// Cheap per-leaf bound on every contained query's local k-th distance (no walk): the smallest
// ancestor-or-self node holding >= k (source) points contains k candidates within its own AABB, so
// its self d_up^2 (the AABB diagonal, an exact upper bound on any canonical d2 inside, R8) bounds
// the k-th distance; +inf if no node holds k points. planes: beg/leafspl/box of every plane.
struct PlaneRef {
  const int32_t *leafspl;
  const NodeBox *box;
  int64_t nnodes;
};
__global__ void k_leaf_rdiag(const NodeBox *__restrict__ leafbox, int64_t nleaf, const PlaneRef *__restrict__ up,
                             int nup, Dom D, int k, float *__restrict__ r2) {
  for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < nleaf; l += (int64_t)gridDim.x * blockDim.x) {
    NodeBox b = leafbox[l];
    float r = INFINITY;
    if (box_count(b) >= k) {
      r = box_dup2(b, b, D);
    } else {
      for (int p = 0; p < nup; ++p) {  // ancestor on plane p+1: node i with leafspl[i] <= l < leafspl[i+1]
        const PlaneRef pr = up[p];
        int64_t lo = 0, hi = pr.nnodes - 1;
        while (lo < hi) {
          const int64_t mid = (lo + hi + 1) >> 1;
          if (pr.leafspl[mid] <= l) lo = mid;
          else hi = mid - 1;
        }
        b = pr.box[lo];
        if (box_count(b) >= k) {
          r = box_dup2(b, b, D);
          break;
        }
      }
    }
    r2[l] = r;
  }
}

// leaf R_max^2 -> plane-level boxes with max r2
__global__ void k_plane_qboxes(const NodeBox *__restrict__ box, const int32_t *__restrict__ leafspl, int64_t nnodes,
                               const float *__restrict__ rmax2_leaf, int rank, float *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnodes; i += (int64_t)gridDim.x * blockDim.x) {
    float r2 = 0.f;
    for (int j = leafspl[i]; j < leafspl[i + 1]; ++j) r2 = fmaxf(r2, rmax2_leaf[j]);
    const NodeBox b = box[i];
    float *o = out + 8 * i;
    o[0] = b.lo.x;
    o[1] = b.lo.y;
    o[2] = b.lo.z;
    o[3] = r2;
    o[4] = b.hi.x;
    o[5] = b.hi.y;
    o[6] = b.hi.z;
    o[7] = __int_as_float(rank);
  }
}

__device__ __forceinline__ NodeBox qbox_at(const float *__restrict__ q, int64_t j, float *r2, int *rk) {
  const float4 a = reinterpret_cast<const float4 *>(q)[2 * j];
  const float4 b = reinterpret_cast<const float4 *>(q)[2 * j + 1];
  NodeBox nb;
  nb.lo = make_float4(a.x, a.y, a.z, 0.f);
  nb.hi = make_float4(b.x, b.y, b.z, 0.f);
  *r2 = a.w;
  *rk = __float_as_int(b.w);
  return nb;
}

constexpr int kGhostCand = 2048;
constexpr int kQChunk = 32;          // query boxes per culling chunk (consecutive = Morton-ordered per rank)
#ifndef JZ_GHOST_GRID_MIN
#define JZ_GHOST_GRID_MIN 8192
#endif
constexpr int kGhostGridMin = JZ_GHOST_GRID_MIN;  // CTAs of the ghost selection: the coarsest plane with >= this many nodes

// one record per chunk of kQChunk consecutive query boxes: union AABB, largest radius^2, ranks
// present (bit r); a box of the chunk can only reach a node if the chunk does (d_low^2 is monotone
// under box inclusion, the radius is the chunk's largest)
__global__ void k_qchunks(const float *__restrict__ qb, int64_t nqb, float4 *__restrict__ ch) {
  const int64_t nch = (nqb + kQChunk - 1) / kQChunk;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nch; c += (int64_t)gridDim.x * blockDim.x) {
    float4 lo = make_float4(INFINITY, INFINITY, INFINITY, 0.f), hi = make_float4(-INFINITY, -INFINITY, -INFINITY, 0.f);
    float r2m = 0.f;
    unsigned rm = 0;
    for (int64_t j = c * kQChunk; j < min(nqb, (c + 1) * kQChunk); ++j) {
      const float4 a = reinterpret_cast<const float4 *>(qb)[2 * j];
      const float4 b = reinterpret_cast<const float4 *>(qb)[2 * j + 1];
      const int rk = __float_as_int(b.w);
      if (rk < 0 || rk > 31) continue;
      lo = make_float4(fminf(lo.x, a.x), fminf(lo.y, a.y), fminf(lo.z, a.z), 0.f);
      hi = make_float4(fmaxf(hi.x, b.x), fmaxf(hi.y, b.y), fmaxf(hi.z, b.z), 0.f);
      r2m = fmaxf(r2m, a.w);
      rm |= 1u << rk;
    }
    lo.w = r2m;
    hi.w = __uint_as_float(rm);
    ch[2 * c] = lo;
    ch[2 * c + 1] = hi;
  }
}

// the plane whose nodes are the CTAs of k_select_ghosts (enough CTAs for the chip)
static int ghost_grid_plane(const std::vector<Plane> &pl) {
  for (int p = (int)pl.size() - 1; p > 0; --p)
    if (pl[p].nnodes >= kGhostGridMin) return p;
  return 0;
}
constexpr int kGhostHit = 16;  // query boxes per leaf kept for the point-level filter

// one CTA per node of the top plane: candidate peer boxes (CTA-wide), then one warp per leaf:
// the lanes test the candidates against the leaf box (ballot-compacted hit list), then the
// leaf's points one per lane (point-level filter; flags of the receiver leaves reached)
__global__ void __launch_bounds__(256) k_select_ghosts(const float4 *__restrict__ pts,
                                                       const NodeBox *__restrict__ topbox,
                                                       const int32_t *__restrict__ top_leafspl,
                                                       const NodeBox *__restrict__ leafbox,
                                                       const int32_t *__restrict__ leafbeg, const float *__restrict__ qb,
                                                       int64_t nqb, int self, Dom D, int32_t *__restrict__ mask,
                                                       const int2 *__restrict__ box_leaves,
                                                       const float *__restrict__ leafqb, int32_t *__restrict__ hit_leaf,
                                                       int32_t *__restrict__ cand_g, const float4 *__restrict__ qch) {
  // cand_g (optional, [gridDim.x][nqb]): candidates beyond the kGhostCand kept in shared memory
  // hit_leaf (optional): receiver leaves that some sent point reaches. Query box j covers the
  // receiver's leaf boxes [box_leaves[j].x, box_leaves[j].y) of leafqb (AABB + the leaf's own
  // radius^2, same 8-float records); a point that passes box j is tested against those leaves
  // and flags the ones within their radius (the receiver re-walks only their queries,
  // jz_knn_query_dist)
  __shared__ int s_cand[kGhostCand];
  __shared__ int s_hit[8][kGhostHit];
  __shared__ int s_n;
  __shared__ int s_over;
  const int64_t T = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    s_n = 0;
    s_over = 0;
  }
  __syncthreads();
  const NodeBox tb = topbox[T];
  const int64_t nch = (nqb + kQChunk - 1) / kQChunk;
  for (int64_t c = threadIdx.x; c < nch; c += blockDim.x) {  // chunks first, then their boxes
    const float4 clo = qch[2 * c], chi = qch[2 * c + 1];
    if ((__float_as_uint(chi.w) & ~(1u << self)) == 0u) continue;
    NodeBox cb;
    cb.lo = make_float4(clo.x, clo.y, clo.z, 0.f);
    cb.hi = make_float4(chi.x, chi.y, chi.z, 0.f);
    if (!(box_dlow2(tb, cb, D) <= clo.w)) continue;
    for (int64_t j = c * kQChunk; j < min(nqb, (c + 1) * kQChunk); ++j) {
      float r2;
      int rk;
      const NodeBox b = qbox_at(qb, j, &r2, &rk);
      if (rk == self) continue;
      if (box_dlow2(tb, b, D) <= r2) {
        int p = atomicAdd(&s_n, 1);
        if (p < kGhostCand) s_cand[p] = (int)j;
        else if (cand_g) cand_g[T * nqb + p] = (int)j;
        else s_over = 1;
      }
    }
  }
  __syncthreads();
  const int nc = s_n;
  const bool over = s_over;
  const int64_t lim = over ? nqb : nc;
  auto cand = [&](int64_t c) -> int { return over ? (int)c : (c < kGhostCand ? s_cand[c] : cand_g[T * nqb + c]); };
  for (int l = top_leafspl[T] + warp; l < top_leafspl[T + 1]; l += 8) {
    const NodeBox lb = leafbox[l];
    int m = 0, nh = 0;
    for (int64_t c0 = 0; c0 < lim; c0 += 32) {  // candidates reaching this leaf, in order
      const int64_t c = c0 + lane;
      bool ok = false;
      int j = 0, rk = 0;
      if (c < lim) {
        j = cand(c);
        float r2;
        const NodeBox b = qbox_at(qb, j, &r2, &rk);
        ok = rk != self && rk >= 0 && rk <= 31 && box_dlow2(lb, b, D) <= r2;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, ok);
      m |= (int)__reduce_or_sync(0xffffffffu, ok ? 1u << rk : 0u);
      const int pos = nh + __popc(bal & ((1u << lane) - 1u));
      if (ok && pos < kGhostHit) s_hit[warp][pos] = j;
      nh += __popc(bal);
    }
    __syncwarp();
    const int i0 = leafbeg[l], i1 = leafbeg[l + 1];
    if (m == 0 || nh > kGhostHit) {  // nothing, or too many boxes: leaf granularity
      for (int i = i0 + lane; i < i1; i += 32) mask[i] = m;
      if (m != 0 && hit_leaf) {  // every leaf of every box reaching the leaf box (a superset)
        for (int64_t c = lane; c < lim; c += 32) {
          const int64_t j = cand(c);
          float r2;
          int rk;
          const NodeBox b = qbox_at(qb, j, &r2, &rk);
          if (rk != self && rk >= 0 && rk <= 31 && box_dlow2(lb, b, D) <= r2)
            for (int q = box_leaves[j].x; q < box_leaves[j].y; ++q) hit_leaf[q] = 1;
        }
      }
      __syncwarp();
      continue;
    }
    // point granularity: a point goes to rank r only if one of r's boxes reaches the point itself
    // (exact point-box bound, the same test as the box test with a degenerate box)
    for (int i = i0 + lane; i < i1; i += 32) {
      const float4 p = pts[i];
      NodeBox pb;
      pb.lo = make_float4(p.x, p.y, p.z, 0.f);
      pb.hi = pb.lo;
      int pm = 0;
      for (int h = 0; h < nh; ++h) {
        const int j = s_hit[warp][h];
        float r2;
        int rk;
        const NodeBox b = qbox_at(qb, j, &r2, &rk);
        if ((hit_leaf || !((pm >> rk) & 1)) && box_dlow2(pb, b, D) <= r2) {
          pm |= 1 << rk;
          if (hit_leaf) {
            for (int q = box_leaves[j].x; q < box_leaves[j].y; ++q) {
              float lr2;
              int lrk;
              const NodeBox lbx = qbox_at(leafqb, q, &lr2, &lrk);
              if (box_dlow2(pb, lbx, D) <= lr2) hit_leaf[q] = 1;
            }
          }
        }
      }
      mask[i] = pm;
    }
    __syncwarp();
  }
}

__global__ void k_ghost_count(const int32_t *__restrict__ mask, int64_t n, int nranks,
                              unsigned long long *__restrict__ counts) {
  __shared__ unsigned long long s_c[32];
  if (threadIdx.x < 32) s_c[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int m = mask[i];
    while (m) {
      int r = __ffs(m) - 1;
      m &= m - 1;
      if (r < nranks) atomicAdd(&s_c[r], 1ull);
    }
  }
  __syncthreads();
  if (threadIdx.x < nranks && s_c[threadIdx.x]) atomicAdd(&counts[threadIdx.x], s_c[threadIdx.x]);
}

__global__ void k_ghost_pack(const float4 *__restrict__ pts, const int32_t *__restrict__ mask, int64_t n, int nranks,
                             const int64_t *__restrict__ off, unsigned long long *__restrict__ cursor,
                             float4 *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int m = mask[i];
    for (int r = 0; r < nranks; ++r) {  // rank-uniform loop: lanes flagged for r share one atomic
      if ((m >> r) & 1) {
        const unsigned long long p = warp_slot(cursor, r);
        out[off[r] + (int64_t)p] = pts[i];
      }
    }
  }
}

}  // namespace jz

namespace {

}

extern "C" {

int jz_morton_keys(const float *pos, int64_t n, const float *box, const float *origin, float extent, uint64_t *keys,
                   jz_stream_t s) {
  try {
    jz::Frame f;
    for (int d = 0; d < 3; ++d) {
      if (box) {
        f.o[d] = 0.f;
        f.s[d] = (float)(2097152.0 / (double)box[d]);
      } else {
        f.o[d] = origin ? origin[d] : 0.f;
        f.s[d] = (float)(2097152.0 / (double)(extent > 0.f ? extent : 1.f));
      }
    }
    jz::morton_keys(pos, n, f, keys, (cudaStream_t)s);
    return JZ_OK;
  } catch (const jz::Error &e) {
    return e.code;
  }
}

int jz_bucket_by_splitters(const uint64_t *keys, int64_t n, const uint64_t *splitters, int32_t nsplit, int32_t *dest,
                           int64_t *counts, jz_stream_t s) {
  if (nsplit < 0 || nsplit > 1023) return JZ_EINVAL;
  try {
    cudaStream_t st = (cudaStream_t)s;
    JZ_CUDA(cudaMemsetAsync(counts, 0, (nsplit + 1) * sizeof(int64_t), st));
    if (n > 0) {
      jz::k_bucket<<<jz::grid_for(n, 256, 148 * 4), 256, 0, st>>>(keys, n, splitters, nsplit, dest,
                                                                   (unsigned long long *)counts);
      JZ_LAUNCH_CHECK();
    }
    return JZ_OK;
  } catch (const jz::Error &e) {
    return e.code;
  }
}

int jz_pack_by_rank(const float *pos, int64_t n, int64_t gidx_base, const int32_t *dest, const int64_t *offsets,
                    int32_t nranks, float *out4, jz_stream_t s) {
  try {
    cudaStream_t st = (cudaStream_t)s;
    unsigned long long *cur = nullptr;
    JZ_CUDA(cudaMallocAsync(&cur, nranks * sizeof(unsigned long long), st));
    JZ_CUDA(cudaMemsetAsync(cur, 0, nranks * sizeof(unsigned long long), st));
    if (n > 0) {
      jz::k_pack<<<jz::grid_for(n, jz::kPackThreads * jz::kPackIPT), jz::kPackThreads, 0, st>>>(pos, n, gidx_base, dest, offsets, cur, (float4 *)out4);
      JZ_LAUNCH_CHECK();
    }
    JZ_CUDA(cudaFreeAsync(cur, st));
    return JZ_OK;
  } catch (const jz::Error &e) {
    return e.code;
  }
}

int jz_pack_rows(const int32_t *idx, const float *d2, const int32_t *row_gidx, int64_t m, int32_t k,
                 const int32_t *dest, const int64_t *offsets, int32_t nranks, int32_t *out, jz_stream_t s) {
  if (m < 0 || k < 1 || nranks < 1 || (m > 0 && (!idx || !d2 || !row_gidx || !dest || !offsets || !out)))
    return JZ_EINVAL;
  try {
    cudaStream_t st = (cudaStream_t)s;
    if (m == 0) return JZ_OK;
    unsigned long long *cur = nullptr;
    int64_t *slot = nullptr;
    JZ_CUDA(cudaMallocAsync(&cur, nranks * sizeof(unsigned long long), st));
    JZ_CUDA(cudaMallocAsync(&slot, m * sizeof(int64_t), st));
    JZ_CUDA(cudaMemsetAsync(cur, 0, nranks * sizeof(unsigned long long), st));
    jz::k_row_slots<<<jz::grid_for(m, 256), 256, 0, st>>>(dest, m, offsets, cur, slot);
    JZ_LAUNCH_CHECK();
    jz::k_pack_rows<<<jz::grid_for(m * (2 * k + 1), 256), 256, 0, st>>>(idx, d2, row_gidx, m, k, slot, out);
    JZ_LAUNCH_CHECK();
    JZ_CUDA(cudaFreeAsync(cur, st));
    JZ_CUDA(cudaFreeAsync(slot, st));
    return JZ_OK;
  } catch (const jz::Error &e) {
    jz::set_last_error(e.what());
    return e.code;
  }
}

int jz_scatter_rows(const int32_t *rows, int64_t m, int32_t k, int64_t gidx_base, int64_t n, int32_t *out_idx,
                    float *out_d2, jz_stream_t s) {
  if (m < 0 || k < 1 || n < 0 || (m > 0 && (!rows || !out_idx || !out_d2))) return JZ_EINVAL;
  try {
    cudaStream_t st = (cudaStream_t)s;
    if (m == 0) return JZ_OK;
    int *bad = nullptr;
    JZ_CUDA(cudaMallocAsync(&bad, sizeof(int), st));
    JZ_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
    jz::k_scatter_rows<<<jz::grid_for(m * 2 * k, 256), 256, 0, st>>>(rows, m, k, gidx_base, n, out_idx, out_d2, bad);
    JZ_LAUNCH_CHECK();
    int h = 0;
    JZ_CUDA(cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    JZ_CUDA(cudaFreeAsync(bad, st));
    JZ_CUDA(cudaStreamSynchronize(st));
    if (h) {
      jz::set_last_error("jz_scatter_rows: a row's global index is outside [gidx_base, gidx_base + n)");
      return JZ_EDATA;
    }
    return JZ_OK;
  } catch (const jz::Error &e) {
    jz::set_last_error(e.what());
    return e.code;
  }
}

int jz_knn_plane_nodes(const jz_knn_index *ix, int plane, int64_t *nnodes) {
  if (!ix || !nnodes) return JZ_EINVAL;
  jz::IndexView v = jz::view_of(ix);
  if (plane < 0) plane = (int)v.planes->size() - 1;
  if (plane >= (int)v.planes->size()) return JZ_EINVAL;
  *nnodes = (*v.planes)[plane].nnodes;
  return JZ_OK;
}

int jz_knn_query_boxes(jz_knn_index *ix, int k, int plane, int rank, float *boxes, jz_stream_t s) {
  if (!ix || !boxes || k < 1) return JZ_EINVAL;
  try {
    cudaStream_t st = (cudaStream_t)s;
    jz::IndexView v = jz::view_of(ix);
    const auto &pl = *v.planes;
    if (plane < 0) plane = (int)pl.size() - 1;
    if (plane >= (int)pl.size()) return JZ_EINVAL;
    jz::IList il;
    float *rmax2 = nullptr;
    if (k > v.n) {
      // fewer than k local points: unbounded radius (peers must send everything reachable)
      JZ_CUDA(cudaMallocAsync(&rmax2, pl[0].nnodes * sizeof(float), st));
      std::vector<float> inf(pl[0].nnodes, INFINITY);
      JZ_CUDA(cudaMemcpyAsync(rmax2, inf.data(), inf.size() * sizeof(float), cudaMemcpyHostToDevice, st));
      JZ_CUDA(cudaStreamSynchronize(st));
    } else if (!(v.flags & JZ_FLAG_QBOX_DIAG)) {  // default: R_max from the NodeToNode walk to the leaf plane
      int32_t *sb = nullptr;
      jz::walk_to(pl, v.D, k, v.ngr, v.flags, 0, il, &rmax2, &sb, st);
      il.release(st);
    } else {  // the diagonal of the smallest ancestor holding k points (no walk; far looser on clustered data)
      const int nup = (int)pl.size() - 1;
      std::vector<jz::PlaneRef> h(nup > 0 ? nup : 1);
      for (int p = 1; p < (int)pl.size(); ++p) h[p - 1] = jz::PlaneRef{pl[p].leafspl, pl[p].box, pl[p].nnodes};
      jz::PlaneRef *dup = nullptr;
      JZ_CUDA(cudaMallocAsync(&dup, h.size() * sizeof(jz::PlaneRef), st));
      JZ_CUDA(cudaMemcpyAsync(dup, h.data(), h.size() * sizeof(jz::PlaneRef), cudaMemcpyHostToDevice, st));
      JZ_CUDA(cudaMallocAsync(&rmax2, pl[0].nnodes * sizeof(float), st));
      jz::k_leaf_rdiag<<<jz::grid_for(pl[0].nnodes, 256), 256, 0, st>>>(pl[0].box, pl[0].nnodes, dup, nup, v.D, k, rmax2);
      JZ_LAUNCH_CHECK();
      JZ_CUDA(cudaFreeAsync(dup, st));
    }
    jz::k_plane_qboxes<<<jz::grid_for(pl[plane].nnodes, 128), 128, 0, st>>>(pl[plane].box, pl[plane].leafspl,
                                                                             pl[plane].nnodes, rmax2, rank, boxes);
    JZ_LAUNCH_CHECK();
    JZ_CUDA(cudaFreeAsync(rmax2, st));
    JZ_CUDA(cudaStreamSynchronize(st));
    return JZ_OK;
  } catch (const jz::Error &e) {
    jz::set_last_error(e.what());
    return e.code;
  }
}

int jz_knn_select_ghosts(jz_knn_index *ix, const float *boxes, int64_t nbox, int self_rank, int32_t nranks,
                         int32_t *mask, int64_t *counts, jz_stream_t s) {
  if (!ix || !mask || !counts || nranks < 1 || nranks > 32) return JZ_EINVAL;
  try {
    cudaStream_t st = (cudaStream_t)s;
    jz::IndexView v = jz::view_of(ix);
    const auto &pl = *v.planes;
    const int top = jz::ghost_grid_plane(pl);
    JZ_CUDA(cudaMemsetAsync(counts, 0, nranks * sizeof(int64_t), st));
    if (nbox > 0) {
      float4 *qch = nullptr;
      const int64_t nch = (nbox + jz::kQChunk - 1) / jz::kQChunk;
      JZ_CUDA(cudaMallocAsync(&qch, nch * 2 * sizeof(float4), st));
      jz::k_qchunks<<<jz::grid_for(nch, 256), 256, 0, st>>>(boxes, nbox, qch);
      jz::k_select_ghosts<<<(unsigned)pl[top].nnodes, 256, 0, st>>>(v.pts, pl[top].box, pl[top].leafspl, pl[0].box,
                                                                     pl[0].beg, boxes, nbox, self_rank, v.D, mask,
                                                                     nullptr, nullptr, nullptr, nullptr, qch);
      JZ_LAUNCH_CHECK();
      JZ_CUDA(cudaFreeAsync(qch, st));
      jz::k_ghost_count<<<jz::grid_for(v.n, 256, 148 * 4), 256, 0, st>>>(mask, v.n, nranks,
                                                                          (unsigned long long *)counts);
      JZ_LAUNCH_CHECK();
    } else {
      JZ_CUDA(cudaMemsetAsync(mask, 0, v.n * sizeof(int32_t), st));
    }
    return JZ_OK;
  } catch (const jz::Error &e) {
    jz::set_last_error(e.what());
    return e.code;
  }
}

int jz_knn_pack_ghosts(jz_knn_index *ix, const int32_t *mask, int32_t nranks, const int64_t *offsets, float *out4,
                       jz_stream_t s) {
  if (!ix || !mask || !offsets || !out4 || nranks < 1 || nranks > 32) return JZ_EINVAL;
  try {
    cudaStream_t st = (cudaStream_t)s;
    jz::IndexView v = jz::view_of(ix);
    unsigned long long *cur = nullptr;
    JZ_CUDA(cudaMallocAsync(&cur, nranks * sizeof(unsigned long long), st));
    JZ_CUDA(cudaMemsetAsync(cur, 0, nranks * sizeof(unsigned long long), st));
    jz::k_ghost_pack<<<jz::grid_for(v.n, 256), 256, 0, st>>>(v.pts, mask, v.n, nranks, offsets, cur, (float4 *)out4);
    JZ_LAUNCH_CHECK();
    JZ_CUDA(cudaFreeAsync(cur, st));
    return JZ_OK;
  } catch (const jz::Error &e) {
    jz::set_last_error(e.what());
    return e.code;
  }
}

}  // extern "C"

namespace jz {

// ---------------------------------------------------------------- distributed kNN (library-side orchestration)
// jz_knn_build_dist / jz_knn_query_dist: PAPER.md §3.3 (L388-393) distributed kNN with the
// sample-splitter Morton-range partition of L112-114, on a jz_comm (NCCL or logical ranks).
constexpr int kSampTotal = 16384;  // all ranks' key samples are sorted by one CTA
#ifndef JZ_QBOX_NODES
#define JZ_QBOX_NODES 65536
#endif
#ifndef JZ_REG_GHOST
#define JZ_REG_GHOST 50
#endif
constexpr int kQBoxNodes = JZ_QBOX_NODES;  // query boxes: the finest plane with at most this many nodes
constexpr int kRegGhost = JZ_REG_GHOST;    // f_max of the second (local + ghost) tree (paper: ~50)

__device__ __forceinline__ uint64_t smix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// N_samp keys drawn with replacement by a counter-based generator ("randomly sample")
__global__ void k_sample_keys(const uint64_t *__restrict__ keys, int64_t n, int ns, uint64_t seed,
                              uint64_t *__restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += gridDim.x * blockDim.x)
    out[i] = keys[(int64_t)(smix(seed * 0x100000001B3ull + (uint64_t)i) % (uint64_t)n)];
}

// one CTA: bitonic sort of the m gathered samples in shared memory, then R - 1 quantile
// splitters spl[i - 1] = sorted[(i m) / R] ("evenly partitioned"); identical on every rank
__global__ void __launch_bounds__(1024) k_splitters(const uint64_t *__restrict__ in, int m, int P, int R,
                                                    uint64_t *__restrict__ spl) {
  extern __shared__ uint64_t s_v[];
  for (int j = threadIdx.x; j < P; j += blockDim.x) s_v[j] = j < m ? in[j] : ~0ull;
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1) {
    for (int st = size >> 1; st > 0; st >>= 1) {
      for (int j = threadIdx.x; j < P; j += blockDim.x) {
        const int o = j ^ st;
        if (o > j) {
          const bool asc = (j & size) == 0;
          const uint64_t a = s_v[j], b = s_v[o];
          if ((a > b) == asc) {
            s_v[j] = b;
            s_v[o] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = 1 + threadIdx.x; i < R; i += blockDim.x) spl[i - 1] = s_v[((int64_t)i * m) / R];
}

// per leaf: the largest local k-th d2 of its queries (rows in z order = leaf order), or +inf
__global__ void k_leaf_kth2(const int32_t *__restrict__ beg, int64_t nleaf, const float *__restrict__ d2, int k,
                            int have_rows, float *__restrict__ r2) {
  for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < nleaf; l += (int64_t)gridDim.x * blockDim.x) {
    float r = have_rows ? 0.f : INFINITY;
    if (have_rows)
      for (int i = beg[l]; i < beg[l + 1]; ++i) r = fmaxf(r, d2[(int64_t)i * k + (k - 1)]);
    r2[l] = r;
  }
}

// queries to re-walk against local + ghost points: the points of every local box a peer hit
__global__ void k_requery_flags(const int32_t *__restrict__ hit, const int32_t *__restrict__ leafspl,
                                const int32_t *__restrict__ beg0, int64_t nnodes, int32_t *__restrict__ flag) {
  for (int64_t i = blockIdx.x; i < nnodes; i += gridDim.x) {
    const int f = hit[i] ? 1 : 0;
    for (int j = beg0[leafspl[i]] + threadIdx.x; j < beg0[leafspl[i + 1]]; j += blockDim.x) flag[j] = f;
  }
}

// gather sel (flag == want) points in order: out[off[i]] = pts[i]; pos[off[i]] = i
__global__ void k_gather_flagged(const float4 *__restrict__ pts, const int32_t *__restrict__ flag,
                                 const int64_t *__restrict__ off, int64_t n, int want, float4 *__restrict__ out,
                                 int32_t *__restrict__ pos) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if ((flag[i] != 0) == (want != 0)) {
      const int64_t o = want ? off[i] : i - off[i];
      out[o] = pts[i];
      if (pos) pos[o] = (int32_t)i;
    }
  }
}

// re-walked rows replace the local rows (row t of the second walk = query bpos[t], same z order)
__global__ void k_merge_rows(const int32_t *__restrict__ idx2, const float *__restrict__ d22,
                             const int32_t *__restrict__ rowg2, const int32_t *__restrict__ bpos, int64_t nb, int k,
                             const float4 *__restrict__ pts, int32_t *__restrict__ idx, float *__restrict__ d2,
                             int *__restrict__ bad) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nb * k; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / k;
    const int c = (int)(t - r * k);
    const int64_t i = bpos[r];
    if (c == 0 && rowg2[r] != __float_as_int(pts[i].w)) *bad = 1;
    idx[i * k + c] = idx2[t];
    d2[i * k + c] = d22[t];
  }
}

// query-only points of a joint tree (the library's convention: negative id)
__global__ void k_query_only(float4 *__restrict__ p, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i].w = __int_as_float(-1);
}

// row t of the ghost walk (query bpos[t], reported by its input row t of the joint tree) merged with
// the query's local row: the k smallest of the two (d2, id)-sorted rows (d2 >= 0: bit order ==
// float order; ids are distinct between local and ghost points)
__global__ void k_merge_ghost_rows(const int32_t *__restrict__ gi, const float *__restrict__ gd,
                                   const int32_t *__restrict__ growg, int kg, const int32_t *__restrict__ bpos,
                                   int64_t nb, int k, int32_t *__restrict__ idx, float *__restrict__ d2,
                                   int32_t *__restrict__ ti, float *__restrict__ td, int *__restrict__ bad) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nb; t += (int64_t)gridDim.x * blockDim.x) {
    if (growg[t] != (int32_t)t) *bad = 1;
    const int64_t i = bpos[t];
    const int32_t *li = idx + i * k;
    const float *ld = d2 + i * k;
    const int32_t *hi = gi + t * kg;
    const float *hd = gd + t * kg;
    int a = 0, b = 0;
    for (int c = 0; c < k; ++c) {
      bool take_local;
      if (b >= kg) take_local = true;
      else if (a >= k) take_local = false;
      else {
        const unsigned x = __float_as_uint(ld[a]), y = __float_as_uint(hd[b]);
        take_local = x < y || (x == y && li[a] < hi[b]);
      }
      if (take_local) {
        ti[t * k + c] = li[a];
        td[t * k + c] = ld[a];
        ++a;
      } else {
        ti[t * k + c] = hi[b];
        td[t * k + c] = hd[b];
        ++b;
      }
    }
    for (int c = 0; c < k; ++c) {
      idx[i * k + c] = ti[t * k + c];
      d2[i * k + c] = td[t * k + c];
    }
  }
}

__global__ void k_rowg_from_pts(const float4 *__restrict__ pts, int64_t n, int32_t *__restrict__ rowg) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    rowg[i] = __float_as_int(pts[i].w);
}

__global__ void k_box_leaf_range(const int32_t *__restrict__ leafspl, int64_t nnodes, int2 *__restrict__ r) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnodes; i += (int64_t)gridDim.x * blockDim.x)
    r[i] = make_int2(leafspl[i], leafspl[i + 1]);
}

__global__ void k_shift_range(int2 *__restrict__ r, int64_t n, int off) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    r[i] = make_int2(r[i].x + off, r[i].y + off);
}

__global__ void k_i32_to_u64(const int32_t *__restrict__ a, int64_t n, uint64_t *__restrict__ b) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = (uint64_t)(uint32_t)a[i];
}

namespace {
void ck(int code) {
  if (code != JZ_OK) throw Error(code, jz_last_error());
}

// device buffers released when the scope ends (stream-ordered)
struct Scratch {
  cudaStream_t st;
  std::vector<void *> p;
  explicit Scratch(cudaStream_t s) : st(s) {}
  template <class T>
  T *get(int64_t n) {
    void *q = nullptr;
    JZ_CUDA(cudaMallocAsync(&q, (size_t)(n > 0 ? n : 1) * sizeof(T), st));
    p.push_back(q);
    return static_cast<T *>(q);
  }
  ~Scratch() {
    for (void *q : p) cudaFreeAsync(q, st);
  }
};

double now_ms() {
  timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return t.tv_sec * 1e3 + t.tv_nsec * 1e-6;
}

std::vector<int64_t> excl(const std::vector<int64_t> &c) {
  std::vector<int64_t> o(c.size() + 1, 0);
  for (size_t i = 0; i < c.size(); ++i) o[i + 1] = o[i] + c[i];
  return o;
}

// all-gather of a variable number of fixed-size records: returns the concatenation (device) and
// per-rank record counts / offsets
template <class T>
T *all_gather_v(Comm *c, const T *mine, int64_t cnt, int rec, Scratch &S, std::vector<int64_t> &counts,
                std::vector<int64_t> &offs, cudaStream_t st) {
  const int R = c->size;
  counts.assign(R, 0);
  c->all_gather_i64_host(&cnt, 1, counts.data(), st);
  int64_t mx = 0;
  for (auto v : counts) mx = v > mx ? v : mx;
  offs = excl(counts);
  T *pad = S.get<T>((mx > 0 ? mx : 1) * rec);
  if (cnt > 0) JZ_CUDA(cudaMemcpyAsync(pad, mine, cnt * rec * sizeof(T), cudaMemcpyDeviceToDevice, st));
  T *all = S.get<T>((int64_t)R * (mx > 0 ? mx : 1) * rec);
  c->all_gather(pad, all, (size_t)(mx > 0 ? mx : 1) * rec * sizeof(T), st);
  T *out = S.get<T>((offs[R] > 0 ? offs[R] : 1) * rec);
  for (int r = 0; r < R; ++r)
    if (counts[r] > 0)
      JZ_CUDA(cudaMemcpyAsync(out + offs[r] * rec, all + (int64_t)r * (mx > 0 ? mx : 1) * rec,
                              counts[r] * rec * sizeof(T), cudaMemcpyDeviceToDevice, st));
  return out;
}

// exchange: device send buffer grouped by destination (host counts per destination), returns the
// received records (device, caller frees) and their count
template <class T>
T *exchange(Comm *c, const T *send, const std::vector<int64_t> &scount, int rec, int64_t *nrecv, cudaStream_t st) {
  const int R = c->size;
  std::vector<int64_t> mat((size_t)R * R);
  c->all_gather_i64_host(scount.data(), R, mat.data(), st);
  std::vector<int64_t> rc(R);
  for (int s = 0; s < R; ++s) rc[s] = mat[(size_t)s * R + c->rank];
  const auto so = excl(scount), ro = excl(rc);
  T *recv = nullptr;
  JZ_CUDA(cudaMallocAsync(&recv, (size_t)(ro[R] > 0 ? ro[R] : 1) * rec * sizeof(T), st));
  c->all_to_all_v(send, scount.data(), so.data(), recv, rc.data(), ro.data(), rec * sizeof(T), st);
  *nrecv = ro[R];
  return recv;
}
}  // namespace

}  // namespace jz

extern "C" {

int jz_knn_build_dist(jz_comm *comm, const float *pos, int64_t n, int64_t gidx_base, const float *box,
                      const jz_knn_params *p, jz_stream_t s, jz_knn_index **out) {
  using namespace jz;
  if (!comm || !out || n < 0 || (n > 0 && !pos) || gidx_base < 0 || gidx_base + n > (int64_t)INT32_MAX - 1) {
    set_last_error("jz_knn_build_dist: bad argument");
    return JZ_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)s;
  struct Guard {
    jz_comm *c;
    cudaStream_t st;
    ~Guard() { c->leave(st); }
  } guard{(comm->enter(), comm), st};
  try {
    NvtxRange nv("jz build_dist");
    const int R = comm->size, r = comm->rank;
    double t0 = now_ms();
    Dom D{};
    if (box) {
      for (int d = 0; d < 3; ++d)
        if (!(box[d] > 0.f) || !std::isfinite(box[d])) throw Error(JZ_EINVAL, "periodic box lengths must be finite and > 0");
      D.periodic = 1;
      for (int d = 0; d < 3; ++d) {
        D.L[d] = box[d];
        D.h[d] = 0.5f * box[d];
      }
    }
    Scratch S(st);
    // 1. validation + one global key frame (open: all-reduced bounding box; P:L133 cubic frame)
    float lo[3], hi[3];
    local_bbox(pos, n, 3, D, lo, hi, st);
    double red[8] = {lo[0], lo[1], lo[2], -(double)hi[0], -(double)hi[1], -(double)hi[2], (double)n, 0.0};
    double tot[1] = {(double)n};
    comm->all_reduce_host(red, 6, RedOp::kMin, st);
    comm->all_reduce_host(tot, 1, RedOp::kSum, st);
    const int64_t ntot = (int64_t)tot[0];
    if (ntot < 1) throw Error(JZ_EINVAL, "no points on any rank");
    jz_knn_params prm{};
    if (p) prm = *p;
    if (!box) {
      float e = 0.f;
      for (int d = 0; d < 3; ++d) {
        prm.frame_origin[d] = (float)red[d];
        const float sp = (float)(-red[3 + d]) - (float)red[d];
        if (sp > e) e = sp;
      }
      prm.frame_extent = e > 0.f ? e : 1.f;
      prm.flags |= JZ_FLAG_FRAME;
    }
    // 2. keys in the global frame
    uint64_t *keys = S.get<uint64_t>(n);
    if (n > 0)
      ck(jz_morton_keys(pos, n, box, prm.frame_origin, prm.frame_extent, keys, s));
    // 3. splitters from N_samp sampled keys per rank
    const int ns = kSampTotal / R < 1000 ? kSampTotal / R : 1000;
    const int64_t myns = n > 0 ? ns : 0;
    uint64_t *samp = S.get<uint64_t>(ns);
    if (myns > 0) {
      k_sample_keys<<<grid_for(ns, 256), 256, 0, st>>>(keys, n, ns, 0x6a7a6b6e6e00ull + (uint64_t)r, samp);
      JZ_LAUNCH_CHECK();
    }
    std::vector<int64_t> sc, so;
    uint64_t *allsamp = all_gather_v<uint64_t>(comm, samp, myns, 1, S, sc, so, st);
    const int m_s = (int)so[R];
    uint64_t *spl = S.get<uint64_t>(R);
    if (R > 1) {
      int P = 1;
      while (P < m_s) P <<= 1;
      JZ_CUDA(cudaFuncSetAttribute(k_splitters, cudaFuncAttributeMaxDynamicSharedMemorySize, P * 8));
      k_splitters<<<1, 1024, P * 8, st>>>(allsamp, m_s, P, R, spl);
      JZ_LAUNCH_CHECK();
    }
    // 4. Morton-range partition: bucket, exchange counts, all-to-all-v of float4 {x, y, z, gidx}
    int32_t *dest = S.get<int32_t>(n);
    int64_t *cnt_d = S.get<int64_t>(R);
    ck(jz_bucket_by_splitters(keys, n, spl, R - 1, dest, cnt_d, s));
    std::vector<int64_t> scount(R);
    JZ_CUDA(cudaMemcpyAsync(scount.data(), cnt_d, R * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    JZ_CUDA(cudaStreamSynchronize(st));
    const auto soff = excl(scount);
    int64_t *soff_d = S.get<int64_t>(R + 1);
    JZ_CUDA(cudaMemcpyAsync(soff_d, soff.data(), (R + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    float4 *send = S.get<float4>(n);
    ck(jz_pack_by_rank(pos, n, gidx_base, dest, soff_d, R, reinterpret_cast<float *>(send), s));
    int64_t m = 0;
    float4 *local = exchange<float4>(comm, send, scount, 1, &m, st);
    const double t1 = now_ms();
    // 5. local tree over the received points
    jz_knn_index *ix = nullptr;
    try {
      if (m > 0) {
        ix = build_impl(reinterpret_cast<const float *>(local), m, 4, 1, m, box, &prm, st);
      } else {
        ix = new jz_knn_index();
        ix->st = st;
        ix->D = D;
        ix->empty = true;
      }
    } catch (...) {
      cudaFreeAsync(local, st);
      throw;
    }
    JZ_CUDA(cudaFreeAsync(local, st));
    ix->comm = comm;
    ix->n_own = n;
    ix->gidx_base = gidx_base;
    ix->has_box = box != nullptr;
    for (int d = 0; d < 3; ++d) ix->box[d] = box ? box[d] : 0.f;
    ix->prm_frame = prm;
    ix->dist_cnt[0] = m;
    ix->dist_ms[0] = t1 - t0;
    ix->dist_ms[1] = now_ms() - t1;
    JZ_CUDA(cudaStreamSynchronize(st));
    *out = ix;
    return JZ_OK;
  } catch (const Error &e) {
    set_last_error(e.what());
    comm->abort();
    return e.code;
  } catch (const std::exception &e) {
    set_last_error(e.what());
    comm->abort();
    return JZ_ECUDA;
  }
}

int jz_knn_rows_dist(const jz_knn_index *ix, int order, int64_t *m) {
  if (!ix || !m || !ix->comm || (order != JZ_ORDER_INPUT && order != JZ_ORDER_Z)) return JZ_EINVAL;
  *m = order == JZ_ORDER_Z ? (ix->empty ? 0 : ix->n) : ix->n_own;
  return JZ_OK;
}

int jz_knn_query_dist(jz_knn_index *ix, int k, int order, int32_t *out_idx, float *out_d2, int32_t *out_row_gidx,
                      jz_stream_t s) {
  using namespace jz;
  if (!ix || !ix->comm || k < 1 || (order != JZ_ORDER_INPUT && order != JZ_ORDER_Z)) {
    set_last_error("jz_knn_query_dist: bad argument (distributed index, k >= 1, order)");
    return JZ_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)s;
  struct Guard {
    jz_comm *c;
    cudaStream_t st;
    ~Guard() { c->leave(st); }
  } guard{(ix->comm->enter(), ix->comm), st};
  try {
    NvtxRange nv("jz query_dist");
    Comm *comm = ix->comm;
    const int R = comm->size, r = comm->rank;
    const int64_t m = ix->empty ? 0 : ix->n;
    const int64_t rows_out = order == JZ_ORDER_Z ? m : ix->n_own;
    if (rows_out > 0 && (!out_idx || !out_d2 || (order == JZ_ORDER_Z && !out_row_gidx)))
      throw Error(JZ_EINVAL, "NULL output");
    double tot[1] = {(double)m};
    comm->all_reduce_host(tot, 1, RedOp::kSum, st);
    if (k > (int64_t)tot[0]) throw Error(JZ_EINVAL, "k must not exceed the total number of points");
    const float *boxp = ix->has_box ? ix->box : nullptr;
    double t0 = now_ms();
    const bool prof = getenv("JZ_DIST_PROF") != nullptr;
    double tp = t0;
    auto mark = [&](const char *what) {  // diagnostics: per-segment wall time (stream synchronised)
      if (!prof) return;
      cudaStreamSynchronize(st);
      const double t = now_ms();
      fprintf(stderr, "rank %d %-14s %8.2f ms\n", r, what, t - tp);
      tp = t;
    };
    Scratch S(st);
    // rows of the local points in z order (the output itself for JZ_ORDER_Z)
    int32_t *idx1 = order == JZ_ORDER_Z ? out_idx : S.get<int32_t>(m * k);
    float *d21 = order == JZ_ORDER_Z ? out_d2 : S.get<float>(m * k);
    int32_t *rowg1 = order == JZ_ORDER_Z ? out_row_gidx : S.get<int32_t>(m);
    // 6. local walk: exact over the local points, so its k-th d2 bounds the global one
    const bool local_rows = m >= k;
    if (local_rows) ck(jz_knn_query(ix, k, JZ_ORDER_Z, idx1, d21, rowg1, s));
    else if (m > 0) {
      k_rowg_from_pts<<<grid_for(m, 256), 256, 0, st>>>(ix->pts, m, rowg1);
      JZ_LAUNCH_CHECK();
    }
    const double t1 = now_ms();
    int64_t nghost = 0, nreq = 0, nbox_mine = 0;
    if (R > 1) {
      // 7. query boxes: nodes of the finest plane with <= kQBoxNodes nodes, radius^2 = the largest
      //    local k-th d2 of their queries (+inf without local rows); all-gathered
      float *qb = nullptr, *lqb = nullptr;
      int2 *brange = nullptr;
      int64_t nleaf_mine = 0;
      int pq = 0;
      if (m > 0) {
        const auto &pl = ix->planes;
        pq = (int)pl.size() - 1;
        for (int q = 0; q < (int)pl.size(); ++q)
          if (pl[q].nnodes <= kQBoxNodes) {
            pq = q;
            break;
          }
        float *r2leaf = S.get<float>(pl[0].nnodes);
        mark("local walk");
        k_leaf_kth2<<<grid_for(pl[0].nnodes, 128), 128, 0, st>>>(pl[0].beg, pl[0].nnodes, d21, k, local_rows, r2leaf);
        JZ_LAUNCH_CHECK();
        nbox_mine = pl[pq].nnodes;
        qb = S.get<float>(nbox_mine * 8);
        k_plane_qboxes<<<grid_for(nbox_mine, 128), 128, 0, st>>>(pl[pq].box, pl[pq].leafspl, nbox_mine, r2leaf, r, qb);
        JZ_LAUNCH_CHECK();
        nleaf_mine = pl[0].nnodes;  // leaf boxes (own radius each) refine the re-walk set
        lqb = S.get<float>(nleaf_mine * 8);
        k_plane_qboxes<<<grid_for(nleaf_mine, 128), 128, 0, st>>>(pl[0].box, pl[0].leafspl, nleaf_mine, r2leaf, r, lqb);
        JZ_LAUNCH_CHECK();
        brange = S.get<int2>(nbox_mine);
        k_box_leaf_range<<<grid_for(nbox_mine, 128), 128, 0, st>>>(pl[pq].leafspl, nbox_mine, brange);
        JZ_LAUNCH_CHECK();
      }
      std::vector<int64_t> bc, bo, lc, lo_;
      float *allb = all_gather_v<float>(comm, qb, nbox_mine, 8, S, bc, bo, st);
      mark("boxes");
      float *alll = all_gather_v<float>(comm, lqb, nleaf_mine, 8, S, lc, lo_, st);
      int2 *allr = all_gather_v<int2>(comm, brange, nbox_mine, 1, S, bc, bo, st);
      const int64_t nb = bo[R], nl = lo_[R];
      for (int q = 0; q < R; ++q)  // leaf ranges into the concatenated leaf-box array
        if (bc[q] > 0 && lo_[q] > 0) {
          k_shift_range<<<grid_for(bc[q], 128), 128, 0, st>>>(allr + bo[q], bc[q], (int)lo_[q]);
          JZ_LAUNCH_CHECK();
        }
      int32_t *hit = S.get<int32_t>(nl);
      JZ_CUDA(cudaMemsetAsync(hit, 0, (nl > 0 ? nl : 1) * sizeof(int32_t), st));
      // 8. ghosts: local points within a peer box's radius (point-level filter), flags of hit boxes
      std::vector<int64_t> gcount(R, 0);
      float4 *gsend = nullptr;
      if (m > 0 && nb > 0) {
        int32_t *mask = S.get<int32_t>(m);
        int64_t *gc = S.get<int64_t>(R);
        const auto &pl = ix->planes;
        const int top = ghost_grid_plane(pl);
        JZ_CUDA(cudaMemsetAsync(gc, 0, R * sizeof(int64_t), st));
        int32_t *cand_g = (int64_t)pl[top].nnodes * nb <= (int64_t)1 << 28 ? S.get<int32_t>(pl[top].nnodes * nb) : nullptr;
        const int64_t nch = (nb + kQChunk - 1) / kQChunk;
        float4 *qch = reinterpret_cast<float4 *>(S.get<float>(nch * 8));
        k_qchunks<<<grid_for(nch, 256), 256, 0, st>>>(allb, nb, qch);
        mark("pre-select");
        k_select_ghosts<<<(unsigned)pl[top].nnodes, 256, 0, st>>>(ix->pts, pl[top].box, pl[top].leafspl, pl[0].box,
                                                                   pl[0].beg, allb, nb, r, ix->D, mask, allr, alll, hit,
                                                                   cand_g, qch);
        JZ_LAUNCH_CHECK();
        mark("k_select_ghosts");
        if (prof) fprintf(stderr, "rank %d top nodes %lld boxes %lld leaves %lld\n", r, (long long)pl[top].nnodes, (long long)nb, (long long)nl);
        mark("gather boxes");
        k_ghost_count<<<grid_for(m, 256, 148 * 4), 256, 0, st>>>(mask, m, R, (unsigned long long *)gc);
        JZ_LAUNCH_CHECK();
        JZ_CUDA(cudaMemcpyAsync(gcount.data(), gc, R * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        JZ_CUDA(cudaStreamSynchronize(st));
        const auto go = excl(gcount);
        int64_t *go_d = S.get<int64_t>(R + 1);
        JZ_CUDA(cudaMemcpyAsync(go_d, go.data(), (R + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
        gsend = S.get<float4>(go[R]);
        ck(jz_knn_pack_ghosts(ix, mask, R, go_d, reinterpret_cast<float *>(gsend), s));
      } else {
        gsend = S.get<float4>(1);
      }
      mark("select ghosts");
      float4 *ghosts = exchange<float4>(comm, gsend, gcount, 1, &nghost, st);
      mark("exchange");
      if (nl > 0) comm->all_reduce_max_i32(hit, nl, st);
      // 9. queries to re-walk: the points of my leaves that some peer's points reached
      if (m > 0 && nghost > 0) {
        const auto &pl = ix->planes;
        int32_t *flag = S.get<int32_t>(m);
        int64_t *off = S.get<int64_t>(m + 1);
        k_requery_flags<<<(unsigned)(nleaf_mine < 65535 ? nleaf_mine : 65535), 128, 0, st>>>(
            hit + lo_[r], pl[0].leafspl, pl[0].beg, nleaf_mine, flag);
        JZ_LAUNCH_CHECK();
        mark("allreduce hits");
        exclusive_scan_i32_to_i64(flag, off, m, st);
        nreq = read_i64(off + m, st);
        if (nreq > 0) {
          int32_t *bpos = S.get<int32_t>(nreq);
          jz_knn_index *ix2 = nullptr;
          try {
            // JZ_REWALK_GHOST=1: walk the flagged queries against the ghosts only and merge with the
            // local rows (no second tree over local + ghosts); measured slower and erratic at 10^8
            // (ghost walk ~10 ms: the flagged queries are sparse in z order, so their 32-query items
            // span large boxes), kept as an option
            static const bool ghost_only = getenv("JZ_REWALK_GHOST") != nullptr;
            if (local_rows && ghost_only) {
              // 10. the flagged queries walked against the ghost points only (a joint tree of
              //     nreq query-only points + the ghosts), then each row is merged with the query's
              //     exact local row: the union's k smallest (d2, id) pairs are the global row,
              //     since every point within the local k-th distance is local or a ghost
              float4 *all = S.get<float4>(nreq + nghost);
              k_gather_flagged<<<grid_for(m, 256), 256, 0, st>>>(ix->pts, flag, off, m, 1, all, bpos);
              JZ_LAUNCH_CHECK();
              k_query_only<<<grid_for(nreq, 256), 256, 0, st>>>(all, nreq);
              JZ_LAUNCH_CHECK();
              JZ_CUDA(cudaMemcpyAsync(all + nreq, ghosts, nghost * sizeof(float4), cudaMemcpyDeviceToDevice, st));
              mark("flags+gather");
              // ghosts are thin shells outside this rank's Morton range, sparse in key space: the
              // regularisation of P:L255-270 (F3) splits the huge nodes they would form
              jz_knn_params p2 = ix->prm_frame;
              if (p2.reg_fmax <= 0) p2.reg_fmax = kRegGhost;
              ix2 = build_impl(reinterpret_cast<const float *>(all), nreq + nghost, 4, 1, nreq, boxp, &p2, st);
              mark("ghost build");
              const int kg = (int)(k < nghost ? k : nghost);
              int32_t *idx2 = S.get<int32_t>(nreq * kg);
              float *d22 = S.get<float>(nreq * kg);
              int32_t *rowg2 = S.get<int32_t>(nreq);
              ck(jz_knn_query(ix2, kg, JZ_ORDER_Z, idx2, d22, rowg2, s));
              mark("ghost walk");
              if (prof) {
                float tm[6];
                int64_t ev = 0;
                jz_knn_stage_times(ix2, tm, &ev);
                fprintf(stderr, "rank %d ghost walk: planes %d n2n %.2f ms leaf %.2f ms evals/query %.0f\n", r,
                        (int)ix2->planes.size(), tm[3], tm[4], (double)ev / (double)nreq);
              }
              int *bad = S.get<int>(1);
              JZ_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
              int32_t *tmpi = S.get<int32_t>(nreq * k);
              float *tmpd = S.get<float>(nreq * k);
              k_merge_ghost_rows<<<grid_for(nreq, 128), 128, 0, st>>>(idx2, d22, rowg2, kg, bpos, nreq, k, idx1, d21,
                                                                       tmpi, tmpd, bad);
              JZ_LAUNCH_CHECK();
              int hb = 0;
              JZ_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
              JZ_CUDA(cudaStreamSynchronize(st));
              if (hb) throw Error(JZ_ECUDA, "internal: ghost rows out of order");
            } else {
              // 10. the flagged queries walked over local + ghost points (a second tree with those
              //     queries first); their rows replace the local rows (a rank with < k local
              //     points: every local query is flagged)
              float4 *all = S.get<float4>(m + nghost);
              k_gather_flagged<<<grid_for(m, 256), 256, 0, st>>>(ix->pts, flag, off, m, 1, all, bpos);
              JZ_LAUNCH_CHECK();
              k_gather_flagged<<<grid_for(m, 256), 256, 0, st>>>(ix->pts, flag, off, m, 0, all + nreq, nullptr);
              JZ_LAUNCH_CHECK();
              JZ_CUDA(cudaMemcpyAsync(all + m, ghosts, nghost * sizeof(float4), cudaMemcpyDeviceToDevice, st));
              jz_knn_params p2 = ix->prm_frame;
              if (p2.reg_fmax <= 0) p2.reg_fmax = kRegGhost;
              ix2 = build_impl(reinterpret_cast<const float *>(all), m + nghost, 4, 1, nreq, boxp, &p2, st);
              int32_t *idx2 = S.get<int32_t>(nreq * k);
              float *d22 = S.get<float>(nreq * k);
              int32_t *rowg2 = S.get<int32_t>(nreq);
              ck(jz_knn_query(ix2, k, JZ_ORDER_Z, idx2, d22, rowg2, s));
              int *bad = S.get<int>(1);
              JZ_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st));
              k_merge_rows<<<grid_for(nreq * k, 256), 256, 0, st>>>(idx2, d22, rowg2, bpos, nreq, k, ix->pts, idx1, d21,
                                                                    bad);
              JZ_LAUNCH_CHECK();
              int hb = 0;
              JZ_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
              JZ_CUDA(cudaStreamSynchronize(st));
              if (hb) throw Error(JZ_ECUDA, "internal: re-walked rows out of order");
            }
          } catch (...) {
            jz_knn_free(ix2);
            cudaFreeAsync(ghosts, st);
            throw;
          }
          jz_knn_free(ix2);
        }
      }
      if (m > 0 && !local_rows && nreq < m) throw Error(JZ_ECUDA, "internal: rank without local rows not re-walked");
      JZ_CUDA(cudaFreeAsync(ghosts, st));
    }
    const double t2 = now_ms();
    // 11. (JZ_ORDER_INPUT, F2) reverse exchange of the rows to the ranks owning their input rows
    if (order == JZ_ORDER_INPUT) {
      std::vector<int64_t> sl(R);
      const int64_t mine[1] = {ix->gidx_base};
      comm->all_gather_i64_host(mine, 1, sl.data(), st);
      std::vector<uint64_t> splh(R > 1 ? R - 1 : 1);
      for (int q = 1; q < R; ++q) splh[q - 1] = (uint64_t)sl[q];
      uint64_t *spl = S.get<uint64_t>(R);
      JZ_CUDA(cudaMemcpyAsync(spl, splh.data(), splh.size() * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
      uint64_t *g64 = S.get<uint64_t>(m);
      int32_t *dest = S.get<int32_t>(m);
      int64_t *cnt_d = S.get<int64_t>(R);
      if (m > 0) {
        k_i32_to_u64<<<grid_for(m, 256), 256, 0, st>>>(rowg1, m, g64);
        JZ_LAUNCH_CHECK();
      }
      ck(jz_bucket_by_splitters(g64, m, spl, R - 1, dest, cnt_d, s));
      std::vector<int64_t> rc(R);
      JZ_CUDA(cudaMemcpyAsync(rc.data(), cnt_d, R * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      JZ_CUDA(cudaStreamSynchronize(st));
      const auto ro = excl(rc);
      int64_t *ro_d = S.get<int64_t>(R + 1);
      JZ_CUDA(cudaMemcpyAsync(ro_d, ro.data(), (R + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
      const int W = 2 * k + 1;
      int32_t *rows = S.get<int32_t>(m * W);
      ck(jz_pack_rows(idx1, d21, rowg1, m, k, dest, ro_d, R, rows, s));
      int64_t got = 0;
      int32_t *recv = exchange<int32_t>(comm, rows, rc, W, &got, st);
      if (got != ix->n_own) {
        cudaFreeAsync(recv, st);
        throw Error(JZ_ECUDA, "internal: rank received a wrong number of input rows");
      }
      const int code = jz_scatter_rows(recv, got, k, ix->gidx_base, ix->n_own, out_idx, out_d2, s);
      JZ_CUDA(cudaFreeAsync(recv, st));
      ck(code);
      if (out_row_gidx && ix->n_own > 0) {
        std::vector<int32_t> g(ix->n_own);
        for (int64_t i = 0; i < ix->n_own; ++i) g[i] = (int32_t)(ix->gidx_base + i);
        JZ_CUDA(cudaMemcpyAsync(out_row_gidx, g.data(), g.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
      }
    }
    JZ_CUDA(cudaStreamSynchronize(st));
    ix->dist_ms[2] = t1 - t0;
    ix->dist_ms[3] = t2 - t1;
    ix->dist_ms[4] = now_ms() - t2;
    ix->dist_cnt[1] = nghost;
    ix->dist_cnt[2] = nreq;
    ix->dist_cnt[3] = nbox_mine;
    return JZ_OK;
  } catch (const Error &e) {
    set_last_error(e.what());
    ix->comm->abort();
    return e.code;
  } catch (const std::exception &e) {
    set_last_error(e.what());
    ix->comm->abort();
    return JZ_ECUDA;
  }
}

int jz_knn_dist_stats(const jz_knn_index *ix, int64_t counts[4], double ms[6]) {
  if (!ix || !ix->comm) return JZ_EINVAL;
  if (counts)
    for (int i = 0; i < 4; ++i) counts[i] = ix->dist_cnt[i];
  if (ms) {
    for (int i = 0; i < 5; ++i) ms[i] = ix->dist_ms[i];
    ms[5] = ix->comm->busy_ms;
  }
  return JZ_OK;
}

}  // extern "C"
