// jz_leaf.cu -- LeafToLeaf (Alg. 1 line 6 L321, L386, L398).
//
// One warp per (query leaf, chunk of 32 queries); one query point per lane. The warp
// walks its leaf's interaction list in r_low order; before each entry it takes the warp max of
// the lanes' current k-th squared distance and stops once r_low exceeds it (P:L398 early exit,
// "maximum current estimate ... across all threads"). The source leaf's float4 points
// {x, y, z, bits(gidx)} are staged in the warp's shared-memory slot with coalesced 16-byte
// loads and read back as broadcasts. Each lane keeps a sorted register top-k of 64-bit keys
// (d2_bits << 32 | gidx + 1): unsigned order == (d2, index) lexicographic order since d2 >= 0,
// so ties go to the lower global index (R2). The list starts full of sentinels at
// the leaf's R_max^2, which bounds every contained query's true k-th distance, so candidates
// beyond it are never inserted. Periodic boxes: per (query leaf, source leaf) pair each axis is
// classified from the two AABBs as "all pairs wrap by -L / +L / none" (then the shift is one
// exact FADD) or "straddles" (per-pair select); both reproduce the definition bit for bit.
// The epilogue writes each row straight to its final place (input order or z-order), so there
// is no separate reorder pass.
#include "jz_common.cuh"
#include "jz_internal.h"

namespace jz {

constexpr int kLeafWarps = 4;

template <int K>
__device__ __forceinline__ void topk_insert(unsigned long long (&a)[K], unsigned long long key) {
#pragma unroll
  for (int j = K - 1; j > 0; --j) {
    const bool mv = key < a[j - 1];
    const bool here = !mv && key < a[j];
    a[j] = mv ? a[j - 1] : (here ? key : a[j]);
  }
  if (key < a[0]) a[0] = key;
}

struct LeafK {
  const float4 *pts;
  const int32_t *leaf_beg;
  const NodeBox *leaf_box;
  const int64_t *ispl;
  const int32_t *isrc;
  const float *rlow;
  const float *rmax2;
  const int32_t *perm;
  const int32_t *zrow;
  int64_t nleaf;
  int64_t n_query;
  int k;
  int order;
  int nmax0;
  int chunks;
  int early;
  int sorted;
  int32_t *out_idx;
  float *out_d2;
  int32_t *out_row_gidx;
  unsigned long long *evals;
};

template <int K, bool PER>
__global__ void __launch_bounds__(kLeafWarps * 32) k_leaf2leaf(LeafK a, Dom D) {
  extern __shared__ float4 s_pts[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float4 *sp = s_pts + warp * a.nmax0;
  const int64_t item = (int64_t)blockIdx.x * kLeafWarps + warp;
  const int64_t leaf = item / a.chunks;
  const int chunk = (int)(item % a.chunks);
  if (leaf >= a.nleaf) return;
  const int qb = a.leaf_beg[leaf], qe = a.leaf_beg[leaf + 1];
  const int q0 = qb + chunk * 32;
  if (q0 >= qe) return;
  const int qi = q0 + lane;
  bool act = qi < qe;
  float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
  int inpos = 0;
  if (act) {
    q = a.pts[qi];
    inpos = a.perm[qi];
    act = inpos < a.n_query;
  }
  if (!__any_sync(0xffffffffu, act)) return;

  // top-k: slots [0, K-k) hold 0 (below every real key), [K-k, K) start at the sentinel (R_max^2, max)
  const float R = a.rmax2[leaf];
  unsigned long long tk[K];
  const unsigned long long sentinel = ((unsigned long long)__float_as_uint(R) << 32) | 0xffffffffull;
#pragma unroll
  for (int j = 0; j < K; ++j) tk[j] = (j < K - a.k) ? 0ull : sentinel;
  float kth = R;

  const NodeBox qbox = a.leaf_box[leaf];
  const int64_t eb = a.ispl[leaf], ee = a.ispl[leaf + 1];
  unsigned long long nev = 0;
  for (int64_t e = eb; e < ee; ++e) {
    const int s = a.isrc[e];
    if (a.early) {
      const float rl = a.rlow[e];
      const unsigned m = __reduce_max_sync(0xffffffffu, act ? __float_as_uint(kth) : 0u);
      if (rl > __uint_as_float(m)) {
        if (a.sorted) break;
        continue;
      }
    }
    const int sb = a.leaf_beg[s], se = a.leaf_beg[s + 1];
    const int m = se - sb;
    __syncwarp();
    for (int t = lane; t < m; t += 32) sp[t] = a.pts[sb + t];
    __syncwarp();
    // periodic shift classes (uniform over the warp: all lanes share the query leaf)
    float sh[3] = {0.f, 0.f, 0.f};
    bool straddle = false, shifted = false;
    if (PER) {
      const NodeBox sbx = a.leaf_box[s];
      const float qlo[3] = {qbox.lo.x, qbox.lo.y, qbox.lo.z}, qhi[3] = {qbox.hi.x, qbox.hi.y, qbox.hi.z};
      const float slo[3] = {sbx.lo.x, sbx.lo.y, sbx.lo.z}, shi[3] = {sbx.hi.x, sbx.hi.y, sbx.hi.z};
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const float tmin = __fsub_rn(qlo[d], shi[d]), tmax = __fsub_rn(qhi[d], slo[d]);
        if (tmin >= D.h[d]) {
          sh[d] = -D.L[d];
          shifted = true;
        } else if (tmax < -D.h[d]) {
          sh[d] = D.L[d];
          shifted = true;
        } else if (!(tmin >= -D.h[d] && tmax < D.h[d])) {
          straddle = true;
        }
      }
    }
    if (act) {
      nev += (unsigned)m;
      if (!PER || (!straddle && !shifted)) {
        for (int j = 0; j < m; ++j) {
          const float4 sv = sp[j];
          const float d2 = canon_d2_open(q.x, q.y, q.z, sv.x, sv.y, sv.z);
          if (d2 <= kth) {
            const unsigned long long key =
                ((unsigned long long)__float_as_uint(d2) << 32) | (unsigned)(__float_as_int(sv.w) + 1);
            if (key < tk[K - 1]) {
              topk_insert<K>(tk, key);
              kth = __uint_as_float((unsigned)(tk[K - 1] >> 32));
            }
          }
        }
      } else if (!straddle) {
        for (int j = 0; j < m; ++j) {
          const float4 sv = sp[j];
          const float tx = __fadd_rn(__fsub_rn(q.x, sv.x), sh[0]);
          const float ty = __fadd_rn(__fsub_rn(q.y, sv.y), sh[1]);
          const float tz = __fadd_rn(__fsub_rn(q.z, sv.z), sh[2]);
          const float d2 = __fmaf_rn(tz, tz, __fmaf_rn(ty, ty, __fmul_rn(tx, tx)));
          if (d2 <= kth) {
            const unsigned long long key =
                ((unsigned long long)__float_as_uint(d2) << 32) | (unsigned)(__float_as_int(sv.w) + 1);
            if (key < tk[K - 1]) {
              topk_insert<K>(tk, key);
              kth = __uint_as_float((unsigned)(tk[K - 1] >> 32));
            }
          }
        }
      } else {
        for (int j = 0; j < m; ++j) {
          const float4 sv = sp[j];
          const float d2 = canon_d2_per(q.x, q.y, q.z, sv.x, sv.y, sv.z, D);
          if (d2 <= kth) {
            const unsigned long long key =
                ((unsigned long long)__float_as_uint(d2) << 32) | (unsigned)(__float_as_int(sv.w) + 1);
            if (key < tk[K - 1]) {
              topk_insert<K>(tk, key);
              kth = __uint_as_float((unsigned)(tk[K - 1] >> 32));
            }
          }
        }
      }
    }
  }
  if (a.evals) {
    unsigned long long tot = nev;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if (lane == 0 && tot) atomicAdd(a.evals, tot);
  }
  if (act) {
    const int64_t row = a.order == JZ_ORDER_INPUT ? (int64_t)inpos : (a.zrow ? (int64_t)a.zrow[qi] : (int64_t)qi);
    int32_t *oi = a.out_idx + row * a.k;
    float *od = a.out_d2 + row * a.k;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      if (j >= K - a.k) {
        oi[j - (K - a.k)] = (int32_t)((unsigned)(tk[j] & 0xffffffffu) - 1u);
        od[j - (K - a.k)] = __uint_as_float((unsigned)(tk[j] >> 32));
      }
    }
    if (a.out_row_gidx) a.out_row_gidx[row] = __float_as_int(q.w);
  }
}

template <int K>
static void launch_k(const LeafK &la, const Dom &D, unsigned blocks, size_t smem, cudaStream_t st) {
  if (D.periodic) k_leaf2leaf<K, true><<<blocks, kLeafWarps * 32, smem, st>>>(la, D);
  else k_leaf2leaf<K, false><<<blocks, kLeafWarps * 32, smem, st>>>(la, D);
}

void leaf_to_leaf(const LeafArgs &a, const Dom &D, cudaStream_t st) {
  LeafK la;
  la.pts = a.pts;
  la.leaf_beg = a.leaf_beg;
  la.leaf_box = a.leaf_box;
  la.ispl = a.il->ispl;
  la.isrc = a.il->isrc;
  la.rlow = a.il->rlow;
  la.rmax2 = a.rmax2;
  la.perm = a.perm;
  la.zrow = a.zrow;
  la.nleaf = a.nleaf;
  la.n_query = a.n_query;
  la.k = a.k;
  la.order = a.order;
  la.nmax0 = a.nmax0;
  la.chunks = (int)ceil_div(a.nmax0, 32);
  la.early = !(a.flags & JZ_FLAG_NO_EARLY_EXIT);
  la.sorted = !(a.flags & JZ_FLAG_NO_SEGSORT);
  la.out_idx = a.out_idx;
  la.out_d2 = a.out_d2;
  la.out_row_gidx = a.out_row_gidx;
  la.evals = a.evals;
  const int64_t items = a.nleaf * la.chunks;
  const unsigned blocks = (unsigned)ceil_div(items, kLeafWarps);
  const size_t smem = (size_t)kLeafWarps * a.nmax0 * sizeof(float4);
  if (blocks == 0) return;
  if (a.k <= 8) launch_k<8>(la, D, blocks, smem, st);
  else if (a.k <= 16) launch_k<16>(la, D, blocks, smem, st);
  else launch_k<32>(la, D, blocks, smem, st);
  JZ_LAUNCH_CHECK();
}

}  // namespace jz
