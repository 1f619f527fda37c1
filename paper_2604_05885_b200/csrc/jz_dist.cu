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
#include <vector>

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

__global__ void k_pack(const float *__restrict__ pos, int64_t n, int64_t gbase, const int32_t *__restrict__ dest,
                       const int64_t *__restrict__ off, unsigned long long *__restrict__ cursor,
                       float4 *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = dest[i];
    const unsigned long long p = warp_slot(cursor, r);
    out[off[r] + (int64_t)p] = make_float4(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], __int_as_float((int)(gbase + i)));
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
constexpr int kGhostHit = 16;  // query boxes per leaf kept for the point-level filter

// one CTA per node of the top plane: candidate peer boxes, then its leaves
__global__ void __launch_bounds__(256) k_select_ghosts(const float4 *__restrict__ pts,
                                                       const NodeBox *__restrict__ topbox,
                                                       const int32_t *__restrict__ top_leafspl,
                                                       const NodeBox *__restrict__ leafbox,
                                                       const int32_t *__restrict__ leafbeg, const float *__restrict__ qb,
                                                       int64_t nqb, int self, Dom D, int32_t *__restrict__ mask) {
  __shared__ int s_cand[kGhostCand];
  __shared__ int s_n;
  __shared__ int s_over;
  const int64_t T = blockIdx.x;
  if (threadIdx.x == 0) {
    s_n = 0;
    s_over = 0;
  }
  __syncthreads();
  const NodeBox tb = topbox[T];
  for (int64_t j = threadIdx.x; j < nqb; j += blockDim.x) {
    float r2;
    int rk;
    const NodeBox b = qbox_at(qb, j, &r2, &rk);
    if (rk == self) continue;
    if (box_dlow2(tb, b, D) <= r2) {
      int p = atomicAdd(&s_n, 1);
      if (p < kGhostCand) s_cand[p] = (int)j;
      else s_over = 1;
    }
  }
  __syncthreads();
  const int nc = s_n;
  if (nc == 0) {
    // no peer reaches this node: clear its points' masks
    for (int l = top_leafspl[T]; l < top_leafspl[T + 1]; ++l)
      for (int i = leafbeg[l] + threadIdx.x; i < leafbeg[l + 1]; i += blockDim.x) mask[i] = 0;
    return;
  }
  const bool over = s_over;
  for (int l = top_leafspl[T] + threadIdx.x; l < top_leafspl[T + 1]; l += blockDim.x) {
    const NodeBox lb = leafbox[l];
    int m = 0;
    int hit[kGhostHit];  // query boxes reaching this leaf (point-level filter below)
    int nh = 0;
    const int64_t lim = over ? nqb : nc;
    for (int64_t c = 0; c < lim; ++c) {
      const int64_t j = over ? c : s_cand[c];
      float r2;
      int rk;
      const NodeBox b = qbox_at(qb, j, &r2, &rk);
      if (rk == self || rk < 0 || rk > 31) continue;
      if (box_dlow2(lb, b, D) <= r2) {
        m |= 1 << rk;
        if (nh < kGhostHit) hit[nh] = (int)j;
        ++nh;
      }
    }
    if (m == 0 || nh > kGhostHit) {  // nothing, or too many boxes: leaf granularity
      for (int i = leafbeg[l]; i < leafbeg[l + 1]; ++i) mask[i] = m;
      continue;
    }
    // point granularity: a point goes to rank r only if one of r's boxes reaches the point itself
    // (exact point-box bound, the same test as the box test with a degenerate box)
    for (int i = leafbeg[l]; i < leafbeg[l + 1]; ++i) {
      const float4 p = pts[i];
      NodeBox pb;
      pb.lo = make_float4(p.x, p.y, p.z, 0.f);
      pb.hi = pb.lo;
      int pm = 0;
      for (int h = 0; h < nh; ++h) {
        float r2;
        int rk;
        const NodeBox b = qbox_at(qb, hit[h], &r2, &rk);
        if (!((pm >> rk) & 1) && box_dlow2(pb, b, D) <= r2) pm |= 1 << rk;
      }
      mask[i] = pm;
    }
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
      jz::k_pack<<<jz::grid_for(n, 256), 256, 0, st>>>(pos, n, gidx_base, dest, offsets, cur, (float4 *)out4);
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
    const int top = (int)pl.size() - 1;
    JZ_CUDA(cudaMemsetAsync(counts, 0, nranks * sizeof(int64_t), st));
    if (nbox > 0) {
      jz::k_select_ghosts<<<(unsigned)pl[top].nnodes, 256, 0, st>>>(v.pts, pl[top].box, pl[top].leafspl, pl[0].box,
                                                                     pl[0].beg, boxes, nbox, self_rank, v.D, mask);
      JZ_LAUNCH_CHECK();
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
